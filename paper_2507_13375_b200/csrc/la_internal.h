// Internal declarations of the GAP-LA B200 library (host C++ <-> CUDA kernels).
// Not part of the ABI: include/la.h is.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/la.h"

namespace gapla {

// Device allocations of the library go through the stream-ordered allocator's default pool
// (cudaMallocAsync on the legacy stream, then a sync so any stream may use the memory); the
// pool keeps freed memory (release threshold raised in la_init_grid), so a new context for
// the next design does not pay the driver's page mapping again.
template <class T>
inline cudaError_t dmalloc(T **p, size_t bytes) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(p), bytes ? bytes : 16, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    return e;
}
inline cudaError_t dfree(void *p) { return p ? cudaFreeAsync(p, 0) : cudaSuccess; }

constexpr int MAXL = 16;                      // layers supported by the kernels
constexpr int MAXKIDS = 4;                    // a GCell has 4 neighbours -> <= 4 children
constexpr int MAXPAIRS = MAXL * (MAXL + 1) / 2;
constexpr uint8_t NO_DIR = 255;               // edir of a root

// Small per-layer tables staged into shared memory by every kernel CTA.
struct TechTab {
    double r[MAXL], c[MAXL], vr[MAXL], ofw[MAXL];
    double VR[MAXL * MAXL];                   // VR[a][b] = sum_{k=min}^{max-1} vr[k], ascending k
};

// Device view of the grid state.  Demand state is packed: one int32 word per
// (unit edge or via cut, layer) = ((d - c) << 1) | (c == 0).  A commit adds 2.
// Wire H plane [y][x][h] (x < X-1, h = index among H layers), V plane
// [x][y][v] (y < Y-1): one straight run's words on all its legal layers are one
// contiguous block.  Via plane [y][x][k], k < L-1.
struct DevGrid {
    int32_t X, Y, L, LH, LV;
    int8_t lidx[MAXL];                        // index of layer l inside its direction plane
    uint8_t dir[MAXL], routable[MAXL];
    int32_t delta_lo, delta_hi;
    double W_D, W_CAP, W_CONG, W_VIA;
    int32_t *wH, *wV, *via;
    const double *Mpos, *Mzero;               // Eq. (3) marginal tables over [delta_lo, delta_hi]
    const TechTab *tab;
};

// Batch-major forest.  Nets of one conflict-free batch are contiguous; the
// nodes of one net are contiguous, ordered by height (leaves first, root last).
struct DevForest {
    int64_t n_nets, n_nodes, n_sinks;
    const uint32_t *xy;                       // x | y << 16
    const int32_t *kid;                       // [n_nodes][4] global child ids (E, W, N, S order), -1
    const int32_t *len;                       // parent-edge length (unit edges)
    const uint8_t *edir;                      // direction parent -> node (0 E, 1 W, 2 N, 3 S); NO_DIR at root
    const uint8_t *nkid, *nl, *nh;            // #children; lowest / highest pin layer (driver incl.); nl=255 if none
    const uint16_t *height;                   // height (leaves 0)
    const int32_t *sink0;                     // first sink (pin arrays) of the node
    const uint16_t *nsink;
    const double *wd, *ur;                    // W_D * w_n (Eq. 5), ur (O3)
    const uint8_t *p_layer;                   // sinks, grouped by node, input order
    const double *p_cap, *p_w;                // C_q; weight of the pin-via delay term
    const int64_t *p_orig;                    // input pin index
    const int64_t *net_node0;                 // [n_nets+1] first node of each net (batch-major)
    const int64_t *net_id;                    // input net index
    const uint8_t *net_pdrv;                  // driver pin layer
};

// The trees as built (input-order chunks, net-local child ids and sink offsets), indexed by the
// batch-major position p through src_node0 / src_sink0; dst_sink0 = first sink of position p.
struct ForestSrc {
    const uint32_t *xy;
    const int32_t *kid, *len, *sink0;
    const uint8_t *edir, *nkid, *nl, *nh, *p_layer;
    const uint16_t *nsink, *height;
    const double *wd, *ur, *p_cap, *p_w;
    const int64_t *p_orig;
    const int64_t *src_node0, *src_sink0, *dst_sink0;   // [n_nets] / [n_nets] / [n_nets + 1]
};

// Default capacities of k_assign's shared-memory net slot: a net whose LA tree has
// at most NS nodes and at most NP sinks is "small" and keeps all its DP state in
// its warp's slot; a larger ("big") net is run by a whole CTA.
constexpr int NS_DEFAULT = 28;              // replaced at load time by the SLOT_BYTES fit
constexpr int NP_DEFAULT = 48;
constexpr int SLOT_BYTES = 4096;            // shared memory per warp's net slot (4 warps per CTA, 6-7 CTAs per SM)
constexpr int ASSIGN_WARPS = 4;
#ifndef ASSIGN_CTAS_LAT
#define ASSIGN_CTAS_LAT 6                   // k_assign CTAs per SM, latency-bound launches (80 registers)
#endif
// k_assign_g: 4 CTAs of 4 warps per SM (128 registers: the group path's per-slot cost' values
// stay in registers) and a 13 KB shared-memory arena per warp (measured: 6-7 CTAs/SM spill and
// run cfg5 at 103-119 ms, 5 at 94 ms, 4 at 87 ms, 3 at 99 ms; profiles/r02_*)
#ifndef G_CTAS_LAT
#define G_CTAS_LAT 4                        // k_assign_g CTAs per SM, latency-bound launches
#endif
#ifndef G_CTAS_THR
#define G_CTAS_THR 4                        // k_assign_g CTAs per SM, throughput-bound launches
#endif
#ifndef G_WARP_ARENA
#define G_WARP_ARENA 13312                  // k_assign_g shared-memory bytes per warp
#endif
#ifndef ASSIGN_CTAS_THR
#define ASSIGN_CTAS_THR 7                   // k_assign CTAs per SM, throughput-bound launches (72 registers)
#endif

struct DevScratch {
    double *froot;                            // [n_nets] f[root][p_drv]
    uint8_t *lay, *sb, *st;                   // decisions per node: entry layer, span (b, t)
    uint32_t *dec;                            // packed decisions for the multi-GPU reconcile
    double *Cd, *rcv, *Tin;                   // Elmore per node
    double *sink_delay, *net_cap, *net_rc;    // outputs (input order)
};

// Kernel launchers (la_kernels.cu).  All enqueue on `s`.
cudaError_t launch_pack_state(const DevGrid &G, const int32_t *wcap, const int32_t *wdem, const int32_t *vcap,
                              const int32_t *vdem, const int64_t *wire_off, cudaStream_t s);
cudaError_t launch_unpack_demand(const DevGrid &G, const int32_t *wcap, const int32_t *vcap, int32_t *wdem,
                                 int32_t *vdem, const int64_t *wire_off, cudaStream_t s);
// One k_assign launch.  Nets are named by forest position through two lists in
// topological (forest) order: big nets (more than NS nodes or NP sinks), run by
// the first n_big_ctas CTAs, one whole CTA per net, and small nets, run by the
// other CTAs, one 8-lane group per net.  wait == nullptr: batch mode.
struct AssignLaunch {
    const int4 *big_pos, *small_pos;          // per net: {forest position, first node, nodes | sinks << 16, first sink}
    int64_t big_beg, big_end;                 // this launch's range of big_pos
    int64_t small_beg, small_end;             // this launch's range of small_pos
    int32_t n_big_ctas;                       // CTAs [0, n_big_ctas) take big nets
    int32_t hybrid;                           // batch mode: every CTA takes big nets first, then small
    int32_t big_split;                        // big nets by half-CTAs (throughput) or whole CTAs (latency)
    unsigned long long *ticket;               // [0] small, [1] big; zeroed before the launch
    int32_t *wait;                            // dataflow mode: unfinished predecessors per net
    const int64_t *succ_off;                  // [n_nets+1] successor CSR (forest order)
    const int32_t *succ;
    char *gscratch;                           // big nets that do not fit a CTA's shared memory:
    int64_t gslot_bytes;                      //   one global slot per big CTA
    int32_t NS, NP;                           // shared-memory slot capacities of a small net
    int32_t LD;                               // max(#H layers, #V layers): layer slots per direction
    int32_t commit;                           // fuse the demand commit (K8) into the kernel
    int64_t *trace;                           // diagnostics: [n_nets][5] per-net timestamps, or nullptr
    // k_assign_g (batch mode): jobs of up to four small nets, one 8-lane group per net
    const int4 *jobs;                         // {first small_pos index, count, off1 | off2 << 16, off3}
    int64_t job_beg, job_end;
    int32_t warp_arena;                       // shared-memory bytes per warp (group arena)
    int32_t *glock;                           // lock per pooled global slot of a big net
    int32_t n_gslots;
};
size_t assign_smem_bytes(int L, int LD, int NS, int NP);
size_t assign_group_net_bytes(int nodes, int sinks, int L, int LD);   // one net's state on the group path
size_t assign_warp_arena_bytes(int L, int LD);                         // per-warp shared memory of k_assign_g
size_t assign_team_net_bytes(int nodes, int sinks, int L, int LD);    // a big net's state on k_assign_g (upper bound)
cudaError_t assign_g_resident_ctas(int L, int LD, int *per_sm_lat, int *per_sm_thr);
cudaError_t launch_assign_g(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a, int grid,
                            bool throughput, cudaStream_t s);
size_t assign_net_bytes(int nodes, int sinks, int L, int LD);
int assign_nets_per_cta();
size_t assign_cta_net_bytes(int L, int LD, int NS, int NP);   // shared memory a big net may use
cudaError_t assign_resident_ctas(int L, int LD, int NS, int NP, int *per_sm_lat, int *per_sm_thr, int *n_sm);
cudaError_t launch_assign(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a, int grid,
                          bool throughput, cudaStream_t s);
cudaError_t fp64_peak(double *ops_per_s);   // la_fp64_peak (la_kernels.cu), current device
cudaError_t launch_permute_forest(const DevForest &F, const ForestSrc &src, cudaStream_t s);
cudaError_t launch_commit(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t node_beg,
                          int64_t node_end, cudaStream_t s);
cudaError_t launch_pack_decisions(const DevScratch &S, int64_t node_beg, int64_t node_end, cudaStream_t s);
cudaError_t launch_unpack_decisions(const DevScratch &S, int64_t node_beg, int64_t node_end, cudaStream_t s);
// k_elmore over the nets [net_beg, net_end) of `list` (forest positions), or over the positions
// [net_beg, net_end) themselves when list is null: la_tree.cu (launch_elmore), the round-1 kernel
// in la_kernels.cu (launch_elmore_v1, A/B only).
cudaError_t launch_elmore(const DevForest &F, const DevScratch &S, const TechTab *tab, int L, int64_t net_beg,
                          int64_t net_end, const int32_t *list, cudaStream_t s);
cudaError_t launch_elmore_v1(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t net_beg,
                             int64_t net_end, const int32_t *list, cudaStream_t s);

// Chunked tree passes (la_tree.cu): a chunk is a run of consecutive forest positions
// run by one warp — whole nets with at most CHUNK_NODES nodes and CHUNK_SINKS sinks together
// (lane = node), or one bigger net.  Record {first position, first node, first sink,
// nets | sinks << 6 | nodes << 13}, or {position, first node, first sink, 1 << 31} for a bigger net.
constexpr int CHUNK_NODES = 32;
constexpr int CHUNK_SINKS = 64;
// Pre-assignment pi-model parasitics per direction (0 = H, 1 = V): unit R (kOhm), unit C (fF).
struct PreRC { double rd[2], cd[2]; };
// Cd / Dg: per-node scratch [n_nodes] for nets beyond a chunk.
cudaError_t launch_pre_timing(const DevForest &F, const int4 *chunks, int64_t n_chunks, const PreRC &P, double *Cd,
                              double *Dg, double *sink_delay, double *net_cap, cudaStream_t s);
// Alg. 1 lines 3-10 (la_order.cu): device inputs; batch_of [n_nets] device output.
struct OrderIn {
    int64_t n_nets;
    const int64_t *pin_ptr, *seg_ptr;
    const double *pin_slack;
    const int32_t *seg_xy, *crit;
    double wns, alpha;
    int32_t th;
    int64_t max_batch;
};
cudaError_t gpu_paper_batches(const OrderIn &in, int32_t *batch_of, int32_t *n_batches, cudaStream_t s,
                              int64_t *launches);

// A large copy between pageable host memory and the device through the pinned pipeline of
// la_host.cpp (copy_many): returns once the bytes have landed.
cudaError_t pinned_copy(void *dst, const void *src, size_t bytes, cudaMemcpyKind kind);

// la_get_solution on the GPU (la_solution.cu): sol_count fills wcnt / vcnt [N+1] (input net order),
// their exclusive sums wptr / vptr [N+1], cost [N] = f[root] and *vcuts; temp == nullptr queries
// the CUB scratch size.  sol_fill writes each net's wires (5 x int32) and via stacks (4 x int32)
// at its offsets, ascending.
cudaError_t sol_count(const DevForest &F, const DevScratch &S, int64_t *wcnt, int64_t *vcnt, int64_t *wptr,
                      int64_t *vptr, double *cost, unsigned long long *vcuts, void *temp, size_t *temp_bytes,
                      cudaStream_t s);
cudaError_t sol_fill(const DevForest &F, const DevScratch &S, const int64_t *wptr, const int64_t *vptr, int32_t *wires,
                     int32_t *vias, cudaStream_t s);

// Evaluator (la_kernels.cu): histogram of (layer, c == 0, clamp(d - c)) over one packed
// plane with `slots` layers per element group (slot -> layer via layer_of), exact
// legacy sum of max(0, d - c) per layer, and the out-of-domain count.
struct EvalDev {
    unsigned long long *hist;                 // [MAXL][2][nbins], nbins = delta_hi - delta_lo + 1
    unsigned long long *legacy;               // [MAXL]
    unsigned long long *oob;                  // [1]
    unsigned long long *wl;                   // [MAXL] unit wire edges per layer (k_eval_nodes)
    unsigned long long *vcuts;                // [1]
};
cudaError_t launch_eval_plane(const int32_t *words, int64_t n, int slots, const int8_t *layer_of_slot, EvalDev E,
                              int delta_lo, int delta_hi, cudaStream_t s);
cudaError_t launch_eval_nodes(const DevForest &F, const DevScratch &S, EvalDev E, cudaStream_t s);

// GPU conflict-free batching (la_batch.cu): keys = (element << 32) | rank,
// returns batch id per rank (host vector) and the number of batches.  The
// predecessor DAG (successor CSR over ranks, in-degrees) stays on the device in
// `dag` until gpu_dag_to_positions re-indexes it into forest order.
struct DagDev {
    int64_t n = 0, n_edges = 0;
    int64_t *off = nullptr;                   // [n+1]
    int32_t *succ = nullptr;                  // [n_edges]
    int32_t *indeg = nullptr;                 // [n]
    void release();
    DagDev() = default;
    DagDev(const DagDev &) = delete;
    DagDev &operator=(const DagDev &) = delete;
    ~DagDev() { release(); }
};
// keys: host (h_keys) or device (d_keys, not owned) array of n_keys.
cudaError_t gpu_conflict_batches(const uint64_t *h_keys, const uint64_t *d_keys, int64_t n_keys, int elem_bits,
                                 int64_t n_nets, std::vector<int32_t> &batch_of_rank, int32_t &n_batches,
                                 cudaStream_t s, int64_t *launches, DagDev *dag);
// k_fp_keys: keys[j] = fp[j] << 32 | rank[net] for j in [start[net], start[net + 1]), nets [0, n).
cudaError_t launch_fp_keys(const uint64_t *fp, const int64_t *start, const int32_t *rank, int64_t n, uint64_t *keys,
                           cudaStream_t s);
// pos_of_rank / rank_of_pos: host arrays [n].  Outputs (device, caller frees
// with cudaFree): off_p [n+1], succ_p [n_edges], indeg_p [n], all in positions.
cudaError_t gpu_dag_to_positions(DagDev &dag, const int64_t *h_rank_of_pos, int64_t **off_p, int32_t **succ_p,
                                 int32_t **indeg_p, cudaStream_t s, int64_t *launches);

}  // namespace gapla
