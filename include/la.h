/*
 * la.h -- C ABI of the B200-native GAP-LA layer-assignment hot path.
 *
 * Paper: "GAP-LA: GPU-Accelerated Performance-Driven Layer Assignment",
 * arXiv 2507.13375 (cited below as PAPER l.<line of PAPER.md>).
 *
 * The calls follow the paper's problem statement: layer assignment "takes a
 * GCell grid graph with GCell edge capacity, a netlist and an optimized 2D
 * global routing solution as input and assigns each 2D routing segment to a
 * certain layer to generate a 3D global routing solution" whose projection is
 * the input (PAPER §II-B l.132-133, §II-D l.150-152).  The per-batch loop is
 * Alg. 2 (l.335-354): for every batch, bottom-up getSubtreeCandidate (Alg. 3,
 * l.355-411) then top-down traceBackSolution (Alg. 4, l.418-435); demand is the
 * Alg. 2 input "demand map D and capacity map C" (l.343), committed between
 * batches (§III-A l.224-226).  Net delay is Elmore on the pi-model RC tree
 * (§II-C l.146, §III-D l.443-444).  Exact operand-level definitions: DESIGN.md
 * §3 (= SURVEY.md §8(c) c.3, O1-O9), readings of garbled / silent passages:
 * DESIGN.md §4.
 *
 * Conventions (all calls):
 *  - Return la_status: LA_OK (0) or a negative error; no exception crosses the
 *    ABI.  la_last_error() returns a thread-local message (net id / segment
 *    index for route errors).
 *  - Every input pointer is caller-owned HOST memory, read only during the call
 *    (the library copies what it needs).  The library owns all device memory
 *    and the context.  Output pointers are caller-allocated HOST buffers.
 *  - Results are in input net / pin order, never in batch order.
 *  - Units: kOhm, fF, ps (kOhm x fF = ps); GCell pitch = 1.
 *  - Call order: la_init_grid -> la_load_nets -> for k = 0..n_batches-1:
 *    la_assign_batch(k), la_commit_demand(k) -> la_eval_timing / la_get_*.
 *    Violations return LA_ESTATE.  LA_ECUDA / LA_ENCCL poison the context:
 *    every later call except la_destroy returns LA_ESTATE.
 *  - la_assign_batch / la_commit_demand / la_assign_all only ENQUEUE work on
 *    the context's stream (no host synchronisation); la_sync, la_eval_timing,
 *    la_get_* synchronise.  Asynchronous CUDA faults surface at the next
 *    synchronising call.
 *  - Multi-GPU (world > 1): one process and one context per GPU.
 *    la_load_nets, la_commit_demand, la_eval_timing and la_get_solution are
 *    collective (every rank calls them with the same arguments).
 *  - Nothing on the compute path runs on the host: if the CUDA device or the
 *    kernels are unavailable the calls fail (LA_ECUDA); there is no CPU
 *    fallback.
 */
#ifndef GAPLA_LA_H
#define GAPLA_LA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct la_ctx la_ctx;

typedef enum {
    LA_OK = 0,
    LA_EINVAL = -1,  /* bad descriptor field or invalid route (see la_init_grid / la_load_nets) */
    LA_ESTATE = -2,  /* call-order violation, or context poisoned by an earlier CUDA/NCCL error */
    LA_ENOMEM = -3,  /* device or host allocation failed                                        */
    LA_ECUDA = -4,   /* CUDA runtime error (context poisoned)                                    */
    LA_ENCCL = -5,   /* NCCL error (context poisoned)                                            */
    LA_ERANGE = -6   /* batch index out of range, or an output buffer too small                  */
} la_status;

/* Grid, technology and weights.  Alg. 2 inputs. */
typedef struct {
    int32_t X, Y, L;            /* GCells along x and y; metal layers, 2 <= L <= 16; X, Y <= 65535   */
    const uint8_t *dir;         /* [L] 0 = H (wires along x), 1 = V                                   */
    const uint8_t *routable;    /* [L] 0/1; each direction needs >= 1 routable layer                  */
    const double *r, *c;        /* [L] wire R (kOhm) and C (fF) per GCell pitch        */
    const double *vr;           /* [L-1] via R (kOhm) of the cut between layer k and k+1 (l.340)     */
    const double *ofw;          /* [L] Eq. (3) overflow weight ofw(l) (l.182)                          */
    double s_pos, s_zero;       /* Eq. (3) exponent: 0.5 if c > 0, 1.5 if c = 0 (l.182)               */
    const int32_t *wire_cap;    /* wire-edge capacity, API layout: layers l = 0..L-1 concatenated;   */
                                /* within layer l the edges keyed by their lower endpoint (x, y),    */
                                /* row-major [y][x]: (X-1)*Y entries if H, X*(Y-1) if V               */
    const int32_t *via_cap;     /* via-cut capacity [(L-1)][Y][X], cut k between layers k and k+1    */
    const int32_t *wire_dem0;   /* initial wire demand, same layout; NULL = all 0                     */
    const int32_t *via_dem0;    /* initial via-cut demand, same layout; NULL = all 0                  */
    double W_D, W_CAP, W_CONG;  /* Alg. 2 weights w^d, w^cap, w^cong (l.338)                           */
    double W_VIA;               /* per-via-cut cost inside ViaCong (Alg. 3 l.377; reading R11)         */
    double r_avg;               /* look-ahead unit R (l.452); NaN = mean of routable r                 */
    double logit_k, logit_b;    /* Eq. (4): k = 10, b = 0.3 (l.314)                                    */
    double w_floor;             /* pin weight used when WNS >= 0 (reading R2)                          */
    int32_t delta_lo, delta_hi; /* Eq. (3) marginal-table domain for d - c (reading R20)               */
    int32_t device;             /* CUDA device ordinal of this process                                 */
    int32_t rank, world;        /* this process's rank, number of ranks (1..8)                          */
    const void *nccl_id;        /* 128-byte ncclUniqueId created by rank 0; NULL when world == 1, or
                                   with world > 1 for the host transport (la_get/put_decisions)      */
    void *stream;               /* cudaStream_t to enqueue on; NULL = library-owned stream             */
} la_grid_desc;

/* Netlist pins and the 2D routing solution. */
typedef struct {
    int64_t n_nets;
    const int64_t *pin_ptr;     /* [n_nets+1] CSR over pins; pin 0 of each net is its driver          */
    const int32_t *pin_x, *pin_y;   /* GCell of each pin                                              */
    const uint8_t *pin_layer;   /* < L                                                                  */
    const double *pin_cap;      /* fF (driver entry ignored)                                            */
    const double *pin_slack;    /* ps (driver entry ignored), Eq. (4) input                             */
    const int64_t *seg_ptr;     /* [n_nets+1] CSR into seg_xy                                            */
    const int32_t *seg_xy;      /* [n_segs][4] x1 y1 x2 y2, axis-aligned 2D segments (may overlap)       */
    const double *r_drv;        /* [n_nets] kOhm, ur(root) seed (reading R6); NULL = 0                   */
    const int64_t *order_key;   /* [n_nets] priority, smaller = earlier, ties by net index; NULL = index */
    double wns;                 /* design WNS (ps), Eq. (4)                                              */
} la_net_desc;

/* Counters of the loaded instance (exact, from the built forest). */
typedef struct {
    int64_t n_nets, n_pins, n_nodes, n_sinks;
    int64_t wirelength;         /* unit 2D edges over all nets                                          */
    int64_t footprint;          /* (element, net) pairs sorted by the batching pass                      */
    int32_t n_batches, max_height;
    int64_t max_batch_nets, max_net_nodes;
    int64_t via_cuts;           /* after assignment (valid once la_get_solution / la_eval_timing ran)  */
    int64_t launches;           /* kernels launched by la_assign_* / la_commit_demand / la_eval_timing */
    double load_ms;             /* host tree build + upload inside la_load_nets                         */
    double batch_ms;            /* GPU batching pass (sort + Kahn layering) inside la_load_nets         */
    int64_t wire_state_words;   /* sum over LA-tree edges of len x (#legal layers of the edge direction) */
    int64_t via_state_words;    /* n_nodes x (L - 1)                                                      */
    int64_t h2d_bytes, d2h_bytes;   /* host<->device bytes copied by the library since init             */
} la_stats;

/* Per-kernel device time, from CUDA events recorded on the context stream
 * around every launch while profiling is enabled (la_set_profiling). */
typedef struct {
    int64_t assign_launches, commit_launches, elmore_launches, reconcile_calls;
    double assign_ms, commit_ms, elmore_ms, reconcile_ms;
    int64_t eval_launches;
    double eval_ms;
    int64_t pretime_launches, order_calls;   /* la_pre_timing kernels; la_paper_batches calls          */
    double pretime_ms, order_ms;             /* order_ms: the whole call (host->device copies included) */
    double order_kernel_ms;                  /* la_paper_batches' kernels and sorts alone                */
} la_profile;

/* Evaluation of a 3D solution (la_eval_overflow).
 * Overflow of a GCell edge e on layer l with demand d and capacity c:
 *   Eq. (3) (PAPER §II-E l.178-182): of = ofw(l) * e^{s (d - c)}, s = s_pos (0.5) if
 *   c > 0 else s_zero (1.5), summed over every wire edge of every layer: tof_wire
 *   (the paper's "total overflow of all the GCell edges", l.169);
 *   Eq. (2) (l.175-177): of = max{0, d - c}: legacy_wire (exact integer).
 * The via-cut grid of reading R11 is evaluated the same way with ofw of the
 * cut's lower layer (R36): tof_via, legacy_via.  Exactness: every element is
 * binned by (layer, c == 0, d - c) with integer counts on the GPU; the host
 * then sums count * ofw(l) * exp(s * (d - c)) per layer in a fixed order, so the
 * result is deterministic and within a few ulps times the element count of the
 * exactly rounded sum (DESIGN §5 "k_eval").  d - c outside [delta_lo, delta_hi]
 * is clamped (reading R20) and counted in out_of_domain.  wirelength[l] = unit
 * wire edges the solution assigns to layer l, via_cuts = sum over via stacks of
 * (t - b), wire_cap = sum_l c[l] * wirelength[l] (fF; the power term of R27). */
typedef struct {
    double tof_wire, tof_via;
    int64_t legacy_wire, legacy_via;
    int64_t wirelength[16];
    int64_t via_cuts;
    double wire_cap;
    int64_t out_of_domain;
} la_eval;

/* Create a context: validate the grid, allocate the packed device demand
 * planes, build the Eq. (3) marginal tables and the via-R table, set up NCCL
 * when world > 1 and nccl_id is given.  Device memory comes from the device's
 * default stream-ordered pool (cudaMallocAsync); the library raises the pool's
 * release threshold, so memory freed by la_destroy stays reserved for the next
 * context of the process.
 * Errors: LA_EINVAL when L < 2 or L > 16, X or Y <= 1 or > 65535, 3 X Y >= 2^32
 * (footprint element ids of the batching pass are 32-bit), any r, c,
 * vr, ofw, W_*, s_pos, s_zero or capacity negative, delta_lo > delta_hi, a
 * direction without a routable layer, bad rank/world; LA_ECUDA / LA_ENCCL on
 * device errors; LA_ENOMEM. */
la_status la_init_grid(const la_grid_desc *g, la_ctx **out);

/* Build the LA directed trees (PAPER §III-B; DESIGN §3 O1), weights Eq.(4)/(5)
 * (O2) and upstream-R estimates (O3) on the host, upload the batch-major
 * forest, and run the GPU conflict-free batching pass (DESIGN §5 K1/K2).
 * Writes the number of batches.  Collective when world > 1.
 * Errors: LA_EINVAL for a pin layer >= L, a pin or segment outside the grid,
 * a non-axis-aligned segment, a route that is not a tree, a pin GCell not on
 * the route, a net without pins, a net with more than 65534 LA-tree nodes or
 * sinks (message names the net); LA_ESTATE if nets were already loaded. */
la_status la_load_nets(la_ctx *ctx, const la_net_desc *n, int32_t *n_batches);

/* Alg. 3 + Alg. 4 for batch k on this rank's shard of the batch: bottom-up
 * candidate DP with look-ahead, then backtrack.  Enqueue only.
 * With conflict-free batches the demand commit of this rank's nets of batch k is FUSED
 * into this call's kernel (each net commits as soon as it is backtracked; nets of one
 * batch never share a footprint element, so this cannot change another net's reads), so
 * la_get_demand between la_assign_batch(k) and la_commit_demand(k) already sees those
 * commits; la_commit_demand(k) adds the other ranks' nets (world > 1).  With snapshot
 * batches every commit happens in la_commit_demand.
 * Errors: LA_ERANGE (k out of range), LA_ESTATE (k is not the next batch). */
la_status la_assign_batch(la_ctx *ctx, int32_t batch);

/* Commit batch k's chosen wires and via cuts into the demand grid (integer
 * atomics).  On a context with an NCCL communicator (nccl_id given; world 1 included,
 * which runs the same path on one GPU) first reconcile every rank's decisions and net
 * costs for batch k (one sum all-reduce each over the batch's packed decisions, others'
 * slots 0), so every replica holds every decision; then replay the OTHER ranks' nets
 * (k_commit over the batch's node ranges outside this rank's two shards: its own nets
 * committed inside la_assign_batch), or the whole batch with snapshot batches.
 * Collective.  Enqueue only.  Errors: LA_ESTATE unless batch k was just assigned. */
la_status la_commit_demand(la_ctx *ctx, int32_t batch);

/* Host transport of the multi-GPU reconcile: a context created
 * with world > 1 and nccl_id == NULL does not use NCCL; after la_assign_batch(k) the caller
 * takes every rank's packed decisions (u32 per node of batch k: layer | b << 8 | t << 16 |
 * 1 << 24 on the rank's own nets, 0 elsewhere) and net costs (f64 per net of batch k, 0 on
 * other ranks' nets) with la_get_decisions, sums them element-wise over the ranks (a sum of
 * disjoint slots: exact), hands the sums to every rank with la_put_decisions, then calls
 * la_commit_demand(k).  Same results as the NCCL path; used to test the sharded path on
 * one GPU and to reconcile over any other transport.  la_batch_extent gives the slot counts
 * (nodes, nets) of batch k.  Errors: LA_ESTATE outside that sequence or on an NCCL or
 * single-rank context; LA_ERANGE for a bad batch. */
la_status la_batch_extent(la_ctx *ctx, int32_t batch, int64_t *nodes, int64_t *nets);
la_status la_get_decisions(la_ctx *ctx, int32_t batch, uint32_t *dec, double *net_cost);
la_status la_put_decisions(la_ctx *ctx, int32_t batch, const uint32_t *dec, const double *net_cost);

/* Every remaining batch (the whole Alg. 2 loop), enqueued.  Collective.
 * LA_SCHED_BATCH: la_assign_batch + la_commit_demand for every remaining batch,
 * one k_assign launch per batch in which every CTA first takes the batch's big
 * nets, then its small nets.  LA_SCHED_DATAFLOW (one rank, no batch assigned
 * since the last load / la_reset): ONE persistent launch in which each net
 * starts as soon as every earlier-priority net sharing a footprint element with
 * it has committed.  Without la_set_schedule the library picks
 * DATAFLOW when the design has at most as many nets as resident warps (one wave,
 * latency-bound) and BATCH otherwise.  Both are bit-identical to sequential
 * assignment. */
la_status la_assign_all(la_ctx *ctx);

/* Paper-style snapshot batches (PAPER §III-A l.224-226 "nets in a
 * subset are assigned in parallel", Alg. 1 l.257-260, Alg. 2 l.345; reading R31).  Call
 * before la_load_nets.  batch_of[n_nets] (>= 0, input net order) replaces the conflict-free
 * batching: batches run in ascending id, every net of a batch reads the demand at the
 * start of its batch, and the batch's commits are applied after it (k_commit), so results
 * are deterministic but may differ from sequential assignment when nets of one batch
 * share GCell edges (the paper's "minimal quality degradation").  batch_of == NULL restores
 * conflict-free batching.  Forces LA_SCHED_BATCH.  Errors: LA_ESTATE after la_load_nets,
 * LA_EINVAL for a negative count; a negative id or a count that differs from the net
 * descriptor's is reported by la_load_nets (LA_EINVAL). */
la_status la_set_snapshot_batches(la_ctx *ctx, const int32_t *batch_of, int64_t n_nets);

/* Alg. 1 lines 3-10 on the GPU (PAPER §III-A l.213-262):
 * critical-net-analysis based ordering and batching, given what Alg. 1 lines 1-2 (STA)
 * produce.  Inputs: the net descriptor (its pin slacks, segments and wns), criticality[n_nets]
 * = number of critical paths through each net (l.208), alpha (semi-critical ratio, 0.7,
 * l.216-218) and th (3, l.215).  Steps:
 *   Divide (l.3): critical nets N_c: criticality > th; semi-critical N_s: the rest with net
 *     slack (minimum over the net's sink slacks, l.217) < alpha * wns; non-critical N_n.
 *   PartitionAndSort(N_c) (l.4, l.228): bands [C, C], [C/2, C), [C/4, C/2), ... of
 *     criticality (C = the maximum); inside a band criticality descending, net slack
 *     ascending, net index.
 *   PartitionAndSort(N_s) (l.5, l.229, reading R33): bands slack == wns, then
 *     (f_{k-1} wns, f_k wns] with f_k = 1 - 0.01 k^2 (1, 0.99, 0.96, 0.91, ...; reading R42)
 *     down to alpha * wns; inside a band net slack ascending, net index.
 *   Sort(N_n) (l.6, l.230 "congestion-driven"; reading R43): 2D wirelength (sum of the
 *     segments' lengths) ascending, index.
 *   GetBatches (l.7-9, reading R31): every band (and N_n) cut in its order into batches of
 *     at most max_batch nets; Concat (l.10): N_c's, then N_s's, then N_n's.
 * Runs on ctx's device and stream (any state after la_init_grid; the context's nets are not
 * used or changed): the descriptor's pin_ptr, pin_slack, seg_ptr, seg_xy and criticality are
 * copied to the device, per-net keys and bands are formed by hand-written kernels, two stable
 * radix passes (CUB) order the nets and a scan forms the batches.  Output: batch_of[n_nets]
 * (input order, caller-owned host memory), *n_batches; feed them to la_set_snapshot_batches.
 * Errors: LA_EINVAL on NULL arrays, alpha <= 0, th < 0, max_batch < 1, a negative criticality
 * or n_nets >= 2^31; LA_ECUDA (poisons the context). */
la_status la_paper_batches(la_ctx *ctx, const la_net_desc *n, const int32_t *criticality, double alpha, int32_t th,
                           int64_t max_batch, int32_t *batch_of, int32_t *n_batches);

/* Pre-assignment timing on the 2D LA trees (PAPER §III-B l.283-286:
 * "For horizontal (vertical) wire connections, we calculate resistance (capacitance) using
 * the average per-unit-length resistance (capacitance) of all horizontal (vertical) wires ...
 * the widely adopted pi-model"; Alg. 1 inputs r_avg, c_avg l.240-241; reading R44).  Every
 * LA-tree edge of direction t and length len is a pi section R = r_t len, C = c_t len (C/2 at
 * each end); sinks hang on their node through zero-resistance edges (l.284).  Outputs (either
 * may be NULL): sink_delay[n_pins] = the Elmore wire delay from the driver's node to the
 * sink's node (ps, input pin order, driver slots 0) and net_cap[n_nets] = the net's total load
 * capacitance (wires + sinks, fF) — the parasitics the STA of Alg. 1 line 1 consumes (the STA
 * is out of scope).  r_h, r_v (kOhm per GCell), c_h, c_v (fF per GCell): per-direction unit
 * values; NaN = the mean of r (c) over the routable layers of that direction (R44).
 * Requires la_load_nets (runs on the resident forest; independent of the batching and of any
 * assignment).  Synchronises.  Not collective: every rank evaluates every net.  Errors:
 * LA_ESTATE before la_load_nets, LA_EINVAL for a negative unit value. */
la_status la_pre_timing(la_ctx *ctx, double r_h, double r_v, double c_h, double c_v, double *sink_delay,
                        double *net_cap);

/* Schedule used by la_assign_all on one rank; automatic until set. */
enum { LA_SCHED_DATAFLOW = 0, LA_SCHED_BATCH = 1 };
la_status la_set_schedule(la_ctx *ctx, int32_t schedule);   /* LA_EINVAL for an unknown value */

/* Elmore delay / downstream capacitance over the 3D RC trees of every net
 * (DESIGN §3 O9).  Outputs (any may be NULL): sink_delay[n_pins] in input pin
 * order (driver slots 0), net_cap[n_nets] (wire + sink C, fF), net_rc[n_nets]
 * (sum over resistors of R x downstream C, ps).  Requires every batch
 * committed.  Synchronises.  Collective.  With world > 1 each rank evaluates only
 * the nets it assigned (its shards of every batch) and leaves the others' values 0;
 * with NCCL the three arrays are then summed over the ranks (an all-gather: every
 * value has exactly one nonzero contributor, x + 0 == x), so every rank returns the
 * complete outputs; with the host transport the caller sums them. */
la_status la_eval_timing(la_ctx *ctx, double *sink_delay, double *net_cap, double *net_rc);

/* The 3D solution in input net order (Alg. 2 output GRS-3D, l.344).  Pass
 * NULL arrays to query the counts.  Per net, wires [x1 y1 x2 y2 layer] with
 * x1 <= x2, y1 <= y2 sorted lexicographically, one per LA-tree edge; vias
 * [x y b t] (t > b) sorted, one per via stack; net_cost[i] = f[root][p_drv]
 * (Alg. 4 l.426).  wire_ptr / via_ptr are CSR offsets [n_nets+1].
 * Synchronises.  Collective. */
la_status la_get_solution(la_ctx *ctx, int64_t *n_wires, int64_t *n_vias,
                          int64_t *wire_ptr, int32_t *wires,
                          int64_t *via_ptr, int32_t *vias, double *net_cost);

/* Current demand in the API layout of la_grid_desc (either may be NULL).  Includes the
 * commits enqueued so far (see la_assign_batch for the fused world == 1 commit). */
la_status la_get_demand(la_ctx *ctx, int32_t *wire_dem, int32_t *via_dem);

/* Conflict-free batch id of every net, input order. */
la_status la_get_batches(la_ctx *ctx, int32_t *batch_of);

/* Restore the initial demand and rewind to batch 0 (keeps the loaded forest),
 * so the hot path can be re-run on the same input. */
la_status la_reset(la_ctx *ctx);

la_status la_get_stats(la_ctx *ctx, la_stats *out);

/* Enable (1) / disable (0) CUDA-event timing of every kernel launch. */
la_status la_set_profiling(la_ctx *ctx, int32_t enable);

/* Accumulated per-kernel device times since the last reset (synchronises).
 * reset != 0 clears the accumulators after reading. */
la_status la_get_profile(la_ctx *ctx, la_profile *out, int32_t reset);

/* Overflow, via count and wire capacitance of the current solution and demand
 * (la_eval above; k_eval_plane / k_eval_nodes).  Requires every batch committed
 * (LA_ESTATE otherwise).  Synchronises.  Collective when world > 1 (every rank
 * holds the full demand and evaluates it; results are identical). */
la_status la_eval_overflow(la_ctx *ctx, la_eval *out);

/* Diagnostics: enable (1) / disable (0) per-net timestamps in k_assign (device
 * %globaltimer, ns).  While enabled every k_assign launch records, for each net
 * it runs, [0] the time its warp took the net, [1] the time its predecessors
 * were all committed (dataflow mode; = [0] otherwise), [2] the end of the
 * gather, [3] the end of its commit, [4] the SM it ran on.  la_get_trace copies
 * them to out[n_nets][5] in INPUT net order (synchronises); LA_ESTATE when
 * tracing was never enabled.  Tracing adds one 40-byte store per net. */
la_status la_set_tracing(la_ctx *ctx, int32_t enable);
la_status la_get_trace(la_ctx *ctx, int64_t *out);

/* Create an ncclUniqueId (128 bytes) on rank 0, to be broadcast to every rank
 * and passed as la_grid_desc.nccl_id. */
la_status la_nccl_unique_id(void *out128);

/* Measurement aid (bench.py): the FP64 vector pipe's peak on `device`, in
 * lane operations per second (one DADD = 1 op), from a kernel of independent DADD chains on
 * every SM (the DP's fp64 work is DADD / DMUL, no FMA: --fmad=false).  Synchronous; writes
 * *ops_per_s; LA_ECUDA on a CUDA error. */
la_status la_fp64_peak(int32_t device, double *ops_per_s);

/* Wait for all enqueued work; surfaces asynchronous CUDA errors. */
la_status la_sync(la_ctx *ctx);

void la_destroy(la_ctx *ctx);

/* Thread-local message of the last error (never NULL). */
const char *la_last_error(void);

/* Contiguous shard [*beg, *end) of n items for `rank` of `world` (host-only
 * helper; the split used for every batch). */
void la_shard_range(int64_t n, int32_t world, int32_t rank, int64_t *beg, int64_t *end);

#ifdef __cplusplus
}
#endif
#endif /* GAPLA_LA_H */
