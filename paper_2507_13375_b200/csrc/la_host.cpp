// Host side of the GAP-LA B200 library: the C ABI of include/la.h.
//
// Responsibilities: validate inputs, build the Eq. (3) marginal and
// via-R tables (host libm, reading R20), build every net's layer-assignment
// directed tree (PAPER §III-B l.264-281), its Eq. (4)/(5) weights (§III-C
// l.307-320) and upstream-R estimates (§III-D l.452) with a thread pool, lay the
// forest out batch-major after the GPU conflict-free batching pass, upload, and
// drive the kernels batch by batch (Alg. 2, l.345-352).  No step of the hot path
// (DP, backtrack, commit, reconcile, Elmore) runs here.
//
// Compiled with -ffp-contract=off: the host-computed fp64 inputs of the DP
// (weights, ur, tables) follow DESIGN §3 O2-O4 operand by operand.
#include <algorithm>
#include <array>
#include <limits>
#include <type_traits>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <sys/mman.h>

#include <nccl.h>

#include "la_internal.h"

using namespace gapla;

namespace {

thread_local std::string g_err = "";

la_status set_err(la_status st, const std::string &msg) {
    g_err = msg;
    return st;
}

const double INF = std::numeric_limits<double>::infinity();
enum { DIR_E = 0, DIR_W = 1, DIR_N = 2, DIR_S = 3 };
const int DX[4] = {1, -1, 0, 0}, DY[4] = {0, 0, 1, -1};
const int OPP[4] = {DIR_W, DIR_E, DIR_S, DIR_N};

}  // namespace

namespace gapla {
// Host staging vectors without the serial zero-fill of value-initialisation.  Large buffers
// (>= 32 MB: the forest staging, footprint keys) are 2 MB-aligned and madvise'd for transparent
// huge pages, so the threads that first touch them take ~500x fewer page faults.
template <class T>
struct default_init_alloc : std::allocator<T> {
    template <class U> struct rebind { using other = default_init_alloc<U>; };
    using std::allocator<T>::allocator;
    static constexpr size_t HUGE_MIN = (size_t)32 << 20, HUGE_ALIGN = (size_t)2 << 20;
    T *allocate(size_t n) {
        const size_t bytes = n * sizeof(T);
        if (bytes < HUGE_MIN) return std::allocator<T>::allocate(n);
        void *p = std::aligned_alloc(HUGE_ALIGN, (bytes + HUGE_ALIGN - 1) & ~(HUGE_ALIGN - 1));
        if (!p) throw std::bad_alloc();
        madvise(p, bytes, MADV_HUGEPAGE);   // advisory: ignored where THP is off
        return static_cast<T *>(p);
    }
    void deallocate(T *p, size_t n) {
        if (n * sizeof(T) < HUGE_MIN) std::allocator<T>::deallocate(p, n);
        else std::free(p);
    }
    template <class U> void construct(U *p) { ::new ((void *)p) U; }
    template <class U, class... A> void construct(U *p, A &&...a) { ::new ((void *)p) U(std::forward<A>(a)...); }
};
template <class T> using hvec = std::vector<T, default_init_alloc<T>>;

}  // namespace gapla
using gapla::hvec;

struct la_ctx {
    int device = 0, rank = 0, world = 1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool poisoned = false;
    bool loaded = false;
    int32_t next_batch = 0;
    bool pending_commit = false;

    int X = 0, Y = 0, L = 0, LH = 0, LV = 0;
    std::vector<uint8_t> dir, routable;
    std::vector<double> r, c, vr, ofw;
    double s_pos = 0, s_zero = 0, W_D = 0, W_CAP = 0, W_CONG = 0, W_VIA = 0, r_avg = 0;
    double logit_k = 0, logit_b = 0, w_floor = 0;
    int32_t delta_lo = 0, delta_hi = 0;
    std::vector<int64_t> wire_off;            // [L+1] API layout offsets
    int64_t n_wire_api = 0, n_via_api = 0, n_wire_packed = 0;
    TechTab tab;

    // device grid
    int32_t *d_wH = nullptr, *d_wV = nullptr, *d_via = nullptr;
    int32_t *d_wH0 = nullptr, *d_wV0 = nullptr, *d_via0 = nullptr;
    int32_t *d_wcap = nullptr, *d_vcap = nullptr;
    int64_t *d_wire_off = nullptr;
    double *d_Mpos = nullptr, *d_Mzero = nullptr;
    TechTab *d_tab = nullptr;
    DevGrid G{};

    // forest (host copies needed for outputs)
    int64_t n_nets = 0, n_pins = 0, n_nodes = 0, n_sinks = 0;
    hvec<int64_t> h_net_node0, h_net_id;
    std::vector<int64_t> batch_net0;          // [n_batches+1] first net (batch-major) of each batch
    int32_t LD = 0;                           // layer slots per direction
    int32_t NS = NS_DEFAULT, NP = NP_DEFAULT; // small-path capacities of k_assign
    int32_t grid = 0;                         // resident k_assign CTAs (persistent grid), latency variant
    int32_t grid_thr = 0;                     // the same, throughput variant (more CTAs per SM)
    int32_t assign_variant = -1;              // -1: per launch; GAPLA_ASSIGN_VARIANT=0 latency / 1 throughput
    int32_t thr_nets_per_warp = 12;           // throughput variant above this many nets per resident warp
    int32_t schedule = -1;                    // -1: automatic (la_assign_all); else LA_SCHED_*
    bool flow_dirty = false;                  // tickets / wait counters consumed since the last reset
    bool fuse_commit = true;
    bool host_xport = false;                  // world > 1 without NCCL: la_get_decisions / la_put_decisions
    bool nccl = false;                        // an NCCL communicator (any world, 1 included): reconcile by all-reduce
    // la_get_solution: decisions copied to the host and the per-net counts, kept between the count
    // query and the fill call until the next assignment or reset
    bool sol_valid = false;
    int64_t *d_sol_w = nullptr;               // [4][N+1] wire / via counts and offsets (la_solution.cu)
    double *d_sol_cost = nullptr;             // [N] f[root] in input order
    unsigned long long *d_sol_vc = nullptr;   // via cuts
    char *d_sol_temp = nullptr;               // CUB scan scratch
    size_t sol_temp_bytes = 0;
    int64_t sol_nw_total = 0, sol_nv_total = 0;
    int32_t *d_sol_rows = nullptr;            // wires (5 x int32) then via stacks (4 x int32), in dev_allocs
    int32_t *d_own_pos = nullptr;             // world > 1: this rank's nets (forest positions), every batch
    int64_t n_own = 0;
    int32_t put_batch = -1;                   // host transport: batch whose reconciled decisions arrived
    int64_t *d_trace = nullptr;               // la_set_tracing: [n_nets][5] (forest order)
    unsigned long long *d_eval = nullptr;     // la_eval_overflow buffers (lazy)
    int8_t *d_eval_lay = nullptr;             // [3][MAXL] slot -> layer for the H, V and via planes
    bool eval0_done = false;                  // Σ(d - c) per layer of the initial planes (la_eval_overflow)
    std::vector<long long> eval0_wire, eval0_via;
    int64_t eval0_oob = 0;
    std::vector<int64_t> batch_big0, batch_small0;   // [n_batches+1] per-batch ranges of the role lists
    // role lists as packed per-net records (position, node0, nodes | sinks << 16, sink0): one
    // 16-byte load per net instead of a chain of dependent loads in k_assign
    int4 *d_big_pos = nullptr, *d_small_pos = nullptr;               // batch order
    int4 *d_flow_big_pos = nullptr, *d_flow_small_pos = nullptr;     // dataflow priority order
    hvec<int64_t> h_net_sink0;                                       // [n_nets+1] first sink per position
    int32_t n_big_ctas = 0;
    std::vector<int32_t> snap_batch;          // la_set_snapshot_batches (input order); empty: conflict-free
    bool hybrid = true;                       // batch-mode launches: all CTAs take big nets first
    int32_t big_split = -1;                   // -1: per launch (launch_grid); GAPLA_BIG_SPLIT=0/1 forces
    bool tracing = false;
    // tickets and the dataflow DAG (device)
    unsigned long long *d_ticket = nullptr;   // [n_batches + 1]: [0] dataflow, [1 + b] batch b
    int64_t *d_succ_off = nullptr;
    int32_t *d_succ = nullptr, *d_indeg = nullptr, *d_wait = nullptr;
    char *d_gscratch = nullptr;
    int64_t gslot_bytes = 0;
    int32_t *d_glock = nullptr;               // lock per pooled global slot
    int32_t n_gslots = 0;
    int32_t warp_arena = 0;                   // k_assign_g shared memory per warp
    int32_t grid_g = 0, grid_g_thr = 0;       // resident k_assign_g CTAs (latency / throughput variant)
    bool group_path = true;                   // batch mode on k_assign_g (GAPLA_GROUP=0: k_assign)
    std::vector<int4> h_jobs;                 // this rank's jobs (k_assign_g), batch by batch
    std::vector<int64_t> batch_job0;          // [n_batches+1]
    int4 *d_jobs = nullptr;
    int4 *d_chunks = nullptr;                 // chunks of the tree passes (build_chunks), in dev_allocs
    int64_t n_chunks = 0;
    int64_t n_flow_big = 0, n_flow_small = 0; // dataflow role lists (k_assign's NS / NP roles)
    int32_t n_big_ctas_flow = 0;              // big-net CTAs of the dataflow launch
    std::vector<int32_t> batch_of_net;        // input order
    std::vector<int32_t> h_big_pos, h_small_pos;
    DevForest F{};
    DevScratch S{};
    std::vector<void *> dev_allocs;           // forest + scratch

    la_stats stats{};
    ncclComm_t comm = nullptr;

    // CUDA-event profiling of kernel launches
    struct Span { int kind; cudaEvent_t a, b; };
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<Span> spans;
    la_profile acc{};
    cudaEvent_t ev_get() {
        if (!ev_pool.empty()) { cudaEvent_t e = ev_pool.back(); ev_pool.pop_back(); return e; }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }

    std::thread free_thr;                     // releases la_load_nets' host staging in the background
    ~la_ctx() {
        if (free_thr.joinable()) free_thr.join();
        if (stream) cudaStreamSynchronize(stream);   // frees are ordered on the legacy stream
        cudaDeviceSynchronize();
        for (void *p : dev_allocs) dfree(p);
        void *gp[] = {d_wH, d_wV, d_via, d_wH0, d_wV0, d_via0, d_wcap, d_vcap, d_wire_off, d_Mpos, d_Mzero, d_tab,
                      d_ticket, d_trace, d_eval, d_eval_lay, d_succ_off, d_succ, d_indeg, d_wait, d_gscratch,
                      d_glock};
        for (void *p : gp) if (p) dfree(p);
        if (comm) ncclCommDestroy(comm);
        for (auto &sp : spans) { cudaEventDestroy(sp.a); cudaEventDestroy(sp.b); }
        for (auto e : ev_pool) cudaEventDestroy(e);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
};

namespace {

la_status cuda_fail(la_ctx *ctx, cudaError_t e, const char *where) {
    if (ctx) ctx->poisoned = true;
    return set_err(LA_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                                    \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);    \
    } while (0)

#define NK(call)                                                                          \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess) {                                                          \
            ctx->poisoned = true;                                                         \
            return set_err(LA_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
        }                                                                                 \
    } while (0)

template <class T>
la_status dev_upload(la_ctx *ctx, T **dst, const T *src, size_t n) {
    void *p = nullptr;
    cudaError_t e = dmalloc(&p, std::max<size_t>(n * sizeof(T), 16));
    if (e != cudaSuccess) {
        ctx->poisoned = true;
        return set_err(e == cudaErrorMemoryAllocation ? LA_ENOMEM : LA_ECUDA,
                       std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    ctx->dev_allocs.push_back(p);
    *dst = static_cast<T *>(p);
    if (src && n) {
        CK(cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
        ctx->stats.h2d_bytes += (int64_t)(n * sizeof(T));
    }
    return LA_OK;
}

enum { K_ASSIGN = 0, K_COMMIT = 1, K_ELMORE = 2, K_RECONCILE = 3, K_EVAL = 4, K_PRETIME = 5, K_ORDER = 6,
       K_ORDER_KERNELS = 7 };

// Profiling brackets: record a CUDA event before / after a launch on the context stream.
int prof_begin(la_ctx *ctx, int kind) {
    if (!ctx->prof) return -1;
    la_ctx::Span sp{kind, ctx->ev_get(), ctx->ev_get()};
    cudaEventRecord(sp.a, ctx->stream);
    ctx->spans.push_back(sp);
    return (int)ctx->spans.size() - 1;
}
void prof_end(la_ctx *ctx, int i) {
    if (i >= 0) cudaEventRecord(ctx->spans[i].b, ctx->stream);
}

template <class T>
la_status dev_alloc(la_ctx *ctx, T **dst, size_t n) {
    return dev_upload<T>(ctx, dst, nullptr, n);
}

#define TRY(x)                          \
    do {                                \
        la_status s_ = (x);             \
        if (s_ != LA_OK) return s_;     \
    } while (0)

// Run f(i) for i in [0, n) on up to nthr threads (contiguous blocks).
template <class F>
void par_for(int64_t n, unsigned nthr, F f) {
    if (n <= 0) return;
    nthr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nthr, n / 2048 + 1));
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nthr; t++)
        th.emplace_back([&, t] { for (int64_t i = n * t / nthr; i < n * (t + 1) / nthr; i++) f(i); });
    for (int64_t i = 0; i < n / nthr; i++) f(i);
    for (auto &x : th) x.join();
}

// Host <-> device copies of pageable host memory, pipelined: the ranges are cut into pieces that
// worker threads copy into pinned double buffers (a process-wide pool, allocated on first use and
// kept like the device pool) while the DMA of the previous piece runs on the worker's own stream.
// Returns once every piece has landed.  (A pageable cudaMemcpyAsync stages through one driver
// buffer serially: ~7 GB/s measured for the forest upload.)
struct Xfer {
    void *dst;
    const void *src;
    size_t bytes;
};
constexpr int PIN_WORKERS = 8;
constexpr size_t PIN_PIECE = (size_t)16 << 20;
struct PinnedPool {
    std::mutex m;
    char *buf[PIN_WORKERS][2] = {};
    bool ok = false;
};
PinnedPool g_pin;

cudaError_t copy_many(const std::vector<Xfer> &xs, int device, cudaMemcpyKind kind) {
    std::lock_guard<std::mutex> lock(g_pin.m);
    if (!g_pin.ok) {
        for (int w = 0; w < PIN_WORKERS; w++)
            for (int b = 0; b < 2; b++) {
                cudaError_t e = cudaHostAlloc((void **)&g_pin.buf[w][b], PIN_PIECE, cudaHostAllocPortable);
                if (e != cudaSuccess) return e;
            }
        g_pin.ok = true;
    }
    struct Piece { const Xfer *x; size_t off, len; };
    std::vector<Piece> pieces;
    for (const Xfer &x : xs)
        for (size_t off = 0; off < x.bytes; off += PIN_PIECE) pieces.push_back({&x, off, std::min(PIN_PIECE, x.bytes - off)});
    if (pieces.empty()) return cudaSuccess;
    std::atomic<size_t> next{0};
    std::atomic<int> err{(int)cudaSuccess};
    const bool h2d = kind == cudaMemcpyHostToDevice;
    auto worker = [&](int w) {
        cudaError_t e = cudaSetDevice(device);
        cudaStream_t st = nullptr;
        cudaEvent_t ev[2] = {nullptr, nullptr};
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        for (int b = 0; b < 2 && e == cudaSuccess; b++) e = cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming);
        bool used[2] = {false, false};
        const Piece *pend[2] = {nullptr, nullptr};   // D2H: piece waiting in buffer b
        int b = 0;
        for (size_t i; e == cudaSuccess && (i = next.fetch_add(1)) < pieces.size(); b ^= 1) {
            const Piece &pc = pieces[i];
            if (used[b]) {
                e = cudaEventSynchronize(ev[b]);
                if (e == cudaSuccess && !h2d && pend[b])
                    std::memcpy((char *)pend[b]->x->dst + pend[b]->off, g_pin.buf[w][b], pend[b]->len);
            }
            if (e != cudaSuccess) break;
            if (h2d) {
                std::memcpy(g_pin.buf[w][b], (const char *)pc.x->src + pc.off, pc.len);
                e = cudaMemcpyAsync((char *)pc.x->dst + pc.off, g_pin.buf[w][b], pc.len, kind, st);
            } else {
                e = cudaMemcpyAsync(g_pin.buf[w][b], (const char *)pc.x->src + pc.off, pc.len, kind, st);
                pend[b] = &pc;
            }
            if (e == cudaSuccess) e = cudaEventRecord(ev[b], st);
            used[b] = true;
        }
        for (int k = 0; k < 2 && e == cudaSuccess; k++)
            if (used[k]) {
                e = cudaEventSynchronize(ev[k]);
                if (e == cudaSuccess && !h2d && pend[k])
                    std::memcpy((char *)pend[k]->x->dst + pend[k]->off, g_pin.buf[w][k], pend[k]->len);
            }
        for (int k = 0; k < 2; k++) if (ev[k]) cudaEventDestroy(ev[k]);
        if (st) cudaStreamDestroy(st);
        if (e != cudaSuccess) err.store((int)e);
    };
    const int nw = (int)std::min<size_t>(PIN_WORKERS, pieces.size());
    std::vector<std::thread> th;
    for (int w = 1; w < nw; w++) th.emplace_back(worker, w);
    worker(0);
    for (auto &t : th) t.join();
    return (cudaError_t)err.load();
}

}  // namespace

namespace gapla {
cudaError_t pinned_copy(void *dst, const void *src, size_t bytes, cudaMemcpyKind kind) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    return copy_many({{dst, src, bytes}}, dev, kind);
}
}  // namespace gapla

namespace {

// Run f(t, begin, end) on nthr threads over contiguous blocks [n*t/nthr, n*(t+1)/nthr).
template <class F>
void par_chunks(int64_t n, unsigned nthr, F f) {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nthr; t++) th.emplace_back([&, t] { f(t, n * t / nthr, n * (t + 1) / nthr); });
    f(0, 0, n / nthr);
    for (auto &x : th) x.join();
}

// In-place inclusive prefix sum of a[0, n) on nthr threads: each block sums its range, then adds
// the sum of the blocks before it (integer: exact, the serial loop's result).
template <class T>
void par_prefix(T *a, int64_t n, unsigned nthr) {
    if (n < ((int64_t)1 << 20) || nthr <= 1) {
        for (int64_t i = 1; i < n; i++) a[i] += a[i - 1];
        return;
    }
    std::vector<T> part(nthr, 0), off(nthr, 0);
    par_chunks(n, nthr, [&](unsigned t, int64_t lo, int64_t hi) {
        T s = 0;
        for (int64_t i = lo; i < hi; i++) { s += a[i]; a[i] = s; }
        part[t] = s;
    });
    for (unsigned t = 1; t < nthr; t++) off[t] = off[t - 1] + part[t - 1];
    par_chunks(n, nthr, [&](unsigned t, int64_t lo, int64_t hi) {
        if (t) for (int64_t i = lo; i < hi; i++) a[i] += off[t];
    });
}

// Sort v by cmp on nthr threads: sorted blocks, then pairwise merges in parallel.
template <class T, class C>
void par_sort(std::vector<T> &v, C cmp, unsigned nthr) {
    const int64_t n = (int64_t)v.size();
    unsigned k = 1;
    while (k * 2 <= nthr && n / (k * 2) >= 65536) k *= 2;
    if (k == 1) { std::sort(v.begin(), v.end(), cmp); return; }
    std::vector<int64_t> b(k + 1);
    for (unsigned i = 0; i <= k; i++) b[i] = n * i / k;
    {
        std::vector<std::thread> th;
        for (unsigned i = 0; i < k; i++) th.emplace_back([&, i] { std::sort(v.begin() + b[i], v.begin() + b[i + 1], cmp); });
        for (auto &x : th) x.join();
    }
    std::vector<T> tmp(n);
    std::vector<T> *src = &v, *dst = &tmp;
    for (unsigned w = 1; w < k; w *= 2) {
        std::vector<std::thread> th;
        for (unsigned i = 0; i < k; i += 2 * w)
            th.emplace_back([&, i, w] {
                const int64_t a = b[i], m = b[std::min(k, i + w)], e = b[std::min(k, i + 2 * w)];
                std::merge(src->begin() + a, src->begin() + m, src->begin() + m, src->begin() + e, dst->begin() + a, cmp);
            });
        for (auto &x : th) x.join();
        std::swap(src, dst);
    }
    if (src != &v) v.swap(*src);
}

bool ok_nonneg(const double *a, int n) {
    for (int i = 0; i < n; i++)
        if (!(a[i] >= 0.0)) return false;
    return true;
}

// ------------------------------------------------------------ tree builder ---
// One net's layer-assignment directed tree (DESIGN §3 O1).  Nodes: pin GCells,
// GCells of degree != 2, and bends; edges are maximal straight runs; root = the
// driver GCell; children ordered E, W, N, S; sinks keep input order.
struct BuiltNet {
    // per node, final order (height ascending, then preorder)
    hvec<uint32_t> xy;
    hvec<int32_t> kid;      // 4 per node, local final ids, -1
    hvec<int32_t> len;
    hvec<uint8_t> edir, nkid, nl, nh;
    hvec<int32_t> sink0;    // local sink offset
    hvec<uint16_t> nsink;
    hvec<double> wd, ur;
    hvec<uint16_t> height;
    // sinks grouped by node in final node order
    hvec<uint8_t> p_layer;
    hvec<double> p_cap, p_w;
    hvec<int64_t> p_orig;
    hvec<uint64_t> fp;      // footprint elements
    int64_t wl = 0;                // unit edges (summed over the nets appended)
    int64_t wsw = 0;               // sum over tree edges of len x #legal layers of the edge direction
};

// Section timers of Builder::build for the CPU harness (tools/hostbench); no-ops in the library.
#ifdef GAPLA_BUILD_PROF
inline uint64_t bprof_now() { return __builtin_ia32_rdtsc(); }
thread_local uint64_t bprof_acc[16], bprof_t;
#define BPROF(k) do { const uint64_t t_ = bprof_now(); bprof_acc[k] += t_ - bprof_t; bprof_t = t_; } while (0)
#define BPROF_START() (bprof_t = bprof_now())
#else
#define BPROF(k) do {} while (0)
#define BPROF_START() do {} while (0)
#endif

struct Builder {
    const la_ctx *ctx;
    const la_net_desc *nd;
    int nlegal[2] = {0, 0};        // routable layers per direction
    // scratch
    std::vector<uint64_t> ek;      // edge keys: gcell * 2 + t  (t = 0 H (x,y)-(x+1,y), 1 V (x,y)-(x,y+1))
    std::vector<uint64_t> vs;      // vertex gcells
    std::vector<uint8_t> mask;     // neighbour bits per vertex (1 << dir)
    std::vector<int32_t> vnode;    // vertex -> preorder node id, -1
    std::vector<int32_t> stack;
    // preorder tree
    std::vector<int32_t> px, py, ppar, plen, pedir, pheight, pnl, pnh;
    std::vector<std::array<int32_t, 4>> pkids;     // children per preorder node (E, W, N, S order)
    std::vector<uint8_t> pnk;                       // number of children
    std::vector<int32_t> sink_cnt, sink_beg;        // sinks per node: CSR over sink_list
    std::vector<int64_t> sink_list, pin_node;       // input pin indices, grouped by node in input order
    std::vector<double> w, ur, pwq;                 // pwq: Eq. (4) weight per pin of the net
    std::vector<int32_t> order, finalid, pre, vof, hcnt;
    int last_height = 0;                            // height of the last built net's root
    std::vector<uint8_t> seen, isn;                 // isn: vertex is a tree node
    std::vector<int32_t> nbr, pin_v;                 // [4 per vertex] neighbour; vertex of each pin

    // GCell -> vertex index: open-addressing hash over vs (built once per net)
    std::vector<uint64_t> hkey;
    std::vector<int32_t> hval;
    uint64_t hmask = 0;
    int hshift = 0;
    void hinit(size_t maxn) {                     // empty table for up to maxn GCells
        int bits = 4;
        while (((size_t)1 << bits) < 2 * maxn) bits++;
        hkey.assign((size_t)1 << bits, ~0ull);
        hval.resize((size_t)1 << bits);
        hmask = ((uint64_t)1 << bits) - 1;
        hshift = 64 - bits;
        vs.clear();
    }
    int32_t hinsert(uint64_t g) {                 // vertex of GCell g, added if new
        uint64_t h = (g * 0x9E3779B97F4A7C15ull) >> hshift;
        while (hkey[h] != ~0ull) {
            if (hkey[h] == g) return hval[h];
            h = (h + 1) & hmask;
        }
        hkey[h] = g;
        hval[h] = (int32_t)vs.size();
        vs.push_back(g);
        return hval[h];
    }
    int64_t vfind(uint64_t g) const {
        uint64_t h = (g * 0x9E3779B97F4A7C15ull) >> hshift;
        while (hkey[h] != ~0ull) {
            if (hkey[h] == g) return hval[h];
            h = (h + 1) & hmask;
        }
        return -1;
    }

    double pin_weight(double slack) const {      // Eq. (4), reading R1/R2
        if (!(nd->wns < 0.0)) return ctx->w_floor;
        double x = slack / nd->wns;
        return 1.0 / (1.0 + std::exp(-ctx->logit_k * (x - ctx->logit_b)));
    }

    // returns empty string on success, else the error message
    std::string build(int64_t net, BuiltNet &out) {
        const int X = ctx->X, Y = ctx->Y, L = ctx->L;
        const int64_t p0 = nd->pin_ptr[net], p1 = nd->pin_ptr[net + 1];
        const int64_t s0 = nd->seg_ptr[net], s1 = nd->seg_ptr[net + 1];
        char buf[200];
        if (p1 <= p0) return "net " + std::to_string(net) + ": no pins";
        for (int64_t p = p0; p < p1; p++) {
            if (nd->pin_x[p] < 0 || nd->pin_y[p] < 0 || nd->pin_x[p] >= X || nd->pin_y[p] >= Y) {
                std::snprintf(buf, sizeof buf, "net %lld: pin %lld outside the grid", (long long)net, (long long)p);
                return buf;
            }
            if (nd->pin_layer[p] >= L) {
                std::snprintf(buf, sizeof buf, "net %lld: pin %lld layer >= L", (long long)net, (long long)p);
                return buf;
            }
        }
        BPROF_START();
        ek.clear();
        for (int64_t s = s0; s < s1; s++) {
            const int32_t *q = nd->seg_xy + 4 * s;
            int x1 = q[0], y1 = q[1], x2 = q[2], y2 = q[3];
            if (x1 < 0 || y1 < 0 || x2 < 0 || y2 < 0 || x1 >= X || x2 >= X || y1 >= Y || y2 >= Y) {
                std::snprintf(buf, sizeof buf, "net %lld: segment %lld outside the grid", (long long)net,
                              (long long)(s - s0));
                return buf;
            }
            if (x1 != x2 && y1 != y2) {
                std::snprintf(buf, sizeof buf, "net %lld: segment %lld not axis-aligned", (long long)net,
                              (long long)(s - s0));
                return buf;
            }
            if (y1 == y2) {
                for (int x = std::min(x1, x2); x < std::max(x1, x2); x++) ek.push_back(((uint64_t)y1 * X + x) * 2);
            } else {
                for (int y = std::min(y1, y2); y < std::max(y1, y2); y++) ek.push_back(((uint64_t)y * X + x1) * 2 + 1);
            }
        }
        BPROF(0);   // pin checks + unit edges
        std::sort(ek.begin(), ek.end());
        ek.erase(std::unique(ek.begin(), ek.end()), ek.end());
        const uint64_t g_drv = (uint64_t)nd->pin_y[p0] * X + nd->pin_x[p0];
        // vertices: the edges' endpoints, deduplicated on insertion into the GCell -> vertex hash
        // (numbered in first-seen order: the numbering is internal), with each vertex's
        // neighbour bits and neighbour vertex per direction filled in the same pass
        const size_t vmax = 2 * ek.size() + 1;
        hinit(vmax);
        mask.assign(vmax, 0);
        nbr.resize(4 * vmax);                        // neighbour vertex per direction (where mask has it)
        for (uint64_t k : ek) {                      // both endpoints of every unit edge
            const uint64_t g = k >> 1;
            const int32_t a = hinsert(g);
            if (k & 1) {
                const int32_t b = hinsert(g + X);
                mask[a] |= 1 << DIR_N; nbr[4 * a + DIR_N] = b;
                mask[b] |= 1 << DIR_S; nbr[4 * b + DIR_S] = a;
            } else {
                const int32_t b = hinsert(g + 1);
                mask[a] |= 1 << DIR_E; nbr[4 * a + DIR_E] = b;
                mask[b] |= 1 << DIR_W; nbr[4 * b + DIR_W] = a;
            }
        }
        if (ek.empty()) hinsert(g_drv);
        BPROF(1);   // sort / unique edges, vertices and neighbours
        pin_v.resize(p1 - p0);
        for (int64_t p = p0; p < p1; p++) {
            const int64_t v = vfind((uint64_t)nd->pin_y[p] * X + nd->pin_x[p]);
            if (v < 0) {
                std::snprintf(buf, sizeof buf, "net %lld: pin %lld GCell not on the route", (long long)net, (long long)p);
                return buf;
            }
            pin_v[p - p0] = (int32_t)v;
        }
        const size_t nv = vs.size();
        if (nv != ek.size() + 1) {
            std::snprintf(buf, sizeof buf, "net %lld: route is not a tree (cycle or disconnected)", (long long)net);
            return buf;
        }
        BPROF(2);   // pin lookups
        BPROF(3);   // neighbour masks
        BPROF(4);   // (connectivity: checked by the DFS below)
        // tree nodes (O1): pin GCells, GCells of degree != 2 and bends
        isn.assign(nv, 0);
        for (int64_t p = p0; p < p1; p++) isn[pin_v[p - p0]] = 1;
        for (size_t vi = 0; vi < nv; vi++) {
            const uint8_t m = mask[vi];
            if (__builtin_popcount(m) != 2 || !(m == ((1 << DIR_E) | (1 << DIR_W)) || m == ((1 << DIR_N) | (1 << DIR_S))))
                isn[vi] = 1;
        }
        BPROF(5);   // pin cells
        // preorder DFS from the root, children E, W, N, S
        px.clear(); py.clear(); ppar.clear(); plen.clear(); pedir.clear(); pkids.clear(); pnk.clear();
        vnode.assign(nv, -1);
        auto add = [&](int x, int y, int par, int ln, int ed, int64_t vi) {
            px.push_back(x); py.push_back(y); ppar.push_back(par); plen.push_back(ln); pedir.push_back(ed);
            pkids.push_back({-1, -1, -1, -1}); pnk.push_back(0);
            vnode[vi] = (int32_t)px.size() - 1;
            return (int32_t)px.size() - 1;
        };
        pre.clear();
        // every vertex is walked exactly once from the driver iff the route is a tree (nv = edges + 1
        // was checked): a vertex met twice closes a cycle, fewer than nv walked leaves a component out
        seen.assign(nv, 0);
        size_t walked = 1;
        {
            const int32_t rv = pin_v[0];
            seen[rv] = 1;
            add((int)(g_drv % X), (int)(g_drv / X), -1, 0, -1, rv);
            stack.assign(1, 0);
            vof.assign(1, (int32_t)rv);
            while (!stack.empty()) {
                int32_t n = stack.back();
                stack.pop_back();
                pre.push_back(n);
                int32_t kids[4];
                int nk = 0;
                for (int d = 0; d < 4; d++) {
                    if (ppar[n] >= 0 && d == OPP[pedir[n]]) continue;
                    if (!(mask[vof[n]] >> d & 1)) continue;
                    int cx = px[n] + DX[d], cy = py[n] + DY[d], ln = 1;
                    int32_t vi = nbr[4 * vof[n] + d];
                    for (;;) {                         // straight through non-nodes: the run continues in d
                        if (seen[vi]) {
                            std::snprintf(buf, sizeof buf, "net %lld: route is not a tree (cycle or disconnected)",
                                          (long long)net);
                            return buf;
                        }
                        seen[vi] = 1;
                        walked++;
                        if (isn[vi]) break;
                        cx += DX[d]; cy += DY[d]; ln++;
                        vi = nbr[4 * vi + d];
                    }
                    int32_t k = add(cx, cy, n, ln, d, vi);
                    vof.push_back((int32_t)vi);
                    pkids[n][pnk[n]++] = k;
                    kids[nk++] = k;
                }
                for (int i = nk - 1; i >= 0; i--) stack.push_back(kids[i]);
            }
        }
        if (walked != nv) {
            std::snprintf(buf, sizeof buf, "net %lld: route is not a tree (cycle or disconnected)", (long long)net);
            return buf;
        }
        BPROF(6);   // preorder DFS (run walks)
        const size_t nn = px.size();
        // pins: nl/nh over all pins (driver included); sinks in input order
        pnl.assign(nn, 255);
        pnh.assign(nn, -1);
        sink_cnt.assign(nn + 1, 0);
        pin_node.resize(p1 - p0);
        pwq.resize(p1 - p0);
        for (int64_t p = p0; p < p1; p++) {
            int32_t n = vnode[pin_v[p - p0]];
            pin_node[p - p0] = n;
            pnl[n] = std::min<int32_t>(pnl[n], nd->pin_layer[p]);
            pnh[n] = std::max<int32_t>(pnh[n], nd->pin_layer[p]);
            if (p != p0) {
                sink_cnt[n + 1]++;
                pwq[p - p0] = pin_weight(nd->pin_slack[p]);
            }
        }
        sink_beg.assign(nn + 1, 0);
        for (size_t n = 0; n < nn; n++) sink_beg[n + 1] = sink_beg[n] + sink_cnt[n + 1];
        sink_list.resize(sink_beg[nn]);
        for (size_t n = 0; n < nn; n++) sink_cnt[n] = sink_beg[n];     // fill cursors
        for (int64_t p = p0 + 1; p < p1; p++) sink_list[sink_cnt[pin_node[p - p0]]++] = p;   // input order per node
        BPROF(7);   // pins -> nodes, Eq. (4) weights, sink lists
        // heights; subtree max sink weight (Eq. 5, reading R3); 0 without sinks (R39)
        pheight.assign(nn, 0);
        w.assign(nn, 0.0);
        for (auto it = pre.rbegin(); it != pre.rend(); ++it) {
            int32_t n = *it;
            int h = 0;
            double m = 0.0;
            for (int32_t q = sink_beg[n]; q < sink_beg[n + 1]; q++) m = std::max(m, pwq[sink_list[q] - p0]);
            for (int k = 0; k < pnk[n]; k++) { h = std::max(h, pheight[pkids[n][k]] + 1); m = std::max(m, w[pkids[n][k]]); }
            pheight[n] = h;
            w[n] = m;
        }
        // ur (reading R6): ur(root) = r_drv, ur(n) = ur(parent) + r_avg * len
        ur.assign(nn, 0.0);
        for (int32_t n : pre)
            ur[n] = (ppar[n] < 0) ? (nd->r_drv ? nd->r_drv[net] : 0.0) : ur[ppar[n]] + ctx->r_avg * plen[n];
        BPROF(8);   // heights, w, ur
        // final order: height ascending, then preorder
        // (counting sort by height, stable in preorder; the root has the largest height)
        hcnt.assign((size_t)pheight[pre[0]] + 2, 0);
        for (int32_t n : pre) hcnt[pheight[n] + 1]++;
        for (size_t h = 1; h < hcnt.size(); h++) hcnt[h] += hcnt[h - 1];
        order.resize(nn);
        for (int32_t n : pre) order[hcnt[pheight[n]]++] = n;
        finalid.assign(nn, -1);
        for (size_t i = 0; i < nn; i++) finalid[order[i]] = (int32_t)i;
        BPROF(9);   // final order
        // appended to the chunk's arrays (node ids and sink offsets stay net-local)
        // (default-initialising vectors: one resize per array per net, every element written below)
        const size_t b0 = out.xy.size(), q0 = out.p_layer.size(), nq = (size_t)sink_beg[nn];
        out.xy.resize(b0 + nn); out.kid.resize((b0 + nn) * 4); out.len.resize(b0 + nn); out.edir.resize(b0 + nn);
        out.nkid.resize(b0 + nn); out.nl.resize(b0 + nn); out.nh.resize(b0 + nn); out.sink0.resize(b0 + nn);
        out.nsink.resize(b0 + nn); out.wd.resize(b0 + nn); out.ur.resize(b0 + nn); out.height.resize(b0 + nn);
        out.p_layer.resize(q0 + nq); out.p_cap.resize(q0 + nq); out.p_w.resize(q0 + nq); out.p_orig.resize(q0 + nq);
        size_t qo = q0;
        for (size_t j = 0; j < nn; j++) {
            const size_t i = b0 + j;
            int32_t n = order[j];
            out.xy[i] = (uint32_t)px[n] | ((uint32_t)py[n] << 16);
            for (int k = 0; k < 4; k++) out.kid[i * 4 + k] = k < pnk[n] ? finalid[pkids[n][k]] : -1;
            out.len[i] = plen[n];
            out.edir[i] = ppar[n] < 0 ? NO_DIR : (uint8_t)pedir[n];
            out.nkid[i] = pnk[n];
            out.nl[i] = (uint8_t)pnl[n];
            out.nh[i] = (uint8_t)(pnh[n] < 0 ? 255 : pnh[n]);
            out.wd[i] = ctx->W_D * w[n];
            out.ur[i] = ur[n];
            out.height[i] = (uint16_t)std::min(pheight[n], 65535);
            out.sink0[i] = (int32_t)(qo - q0);
            out.nsink[i] = (uint16_t)(sink_beg[n + 1] - sink_beg[n]);
            for (int32_t qi = sink_beg[n]; qi < sink_beg[n + 1]; qi++, qo++) {
                const int64_t q = sink_list[qi];
                out.p_layer[qo] = nd->pin_layer[q];
                out.p_cap[qo] = nd->pin_cap[q];
                // pin-via delay weight: w^d_{n->par} for a non-root node (Alg. 3 l.6), W_D * w_q at the root (R13)
                out.p_w[qo] = ppar[n] < 0 ? ctx->W_D * pwq[q - p0] : ctx->W_D * w[n];
                out.p_orig[qo] = q;
            }
        }
        BPROF(10);  // output arrays
        // footprint = unit edges U node GCells (disjoint element spaces)
        const size_t f0 = out.fp.size();
        out.fp.resize(f0 + ek.size() + nn);
        std::memcpy(out.fp.data() + f0, ek.data(), sizeof(uint64_t) * ek.size());
        const uint64_t gbase = (uint64_t)2 * X * Y;
        for (size_t n = 0; n < nn; n++) out.fp[f0 + ek.size() + n] = gbase + (uint64_t)py[n] * X + px[n];
        out.wl += (int64_t)ek.size();
        for (size_t n = 0; n < nn; n++)
            if (ppar[n] >= 0) out.wsw += (int64_t)plen[n] * nlegal[(pedir[n] == DIR_E || pedir[n] == DIR_W) ? 0 : 1];
        BPROF(11);  // footprint
        last_height = pheight[pre[0]];
        return "";
    }
};

// Flat per-thread storage of built nets (input-order chunk).
struct Chunk {
    int64_t beg = 0, end = 0;
    std::vector<int64_t> node_off, sink_off, fp_off;   // per net, size n+1
    BuiltNet acc;                                      // concatenated arrays
    std::string err;
    int64_t err_net = -1;
    int max_height = 0;
};

// Reserve a chunk's arrays once from upper bounds (nodes <= pins + 2 segments: every tree node is
// a pin GCell or an endpoint of a segment; unit edges <= the summed segment lengths; sinks = pins
// - nets), so they never regrow: no reallocation copies, and pages are touched (faulted) once --
// reserved but untouched virtual memory costs nothing, and default_init_alloc backs buffers of
// 32 MB and more with transparent huge pages.
void reserve_chunk(Chunk &ch, const la_net_desc *nd) {
    const int64_t P = nd->pin_ptr[ch.end] - nd->pin_ptr[ch.beg];
    const int64_t s0 = nd->seg_ptr[ch.beg], s1 = nd->seg_ptr[ch.end];
    int64_t len = 0;
    for (int64_t s = s0; s < s1; s++) {
        const int32_t *q = nd->seg_xy + 4 * s;
        len += std::abs((int64_t)q[2] - q[0]) + std::abs((int64_t)q[3] - q[1]);
    }
    const int64_t nodes = P + 2 * (s1 - s0) + 1, sinks = std::max<int64_t>(0, P - (ch.end - ch.beg));
    BuiltNet &a = ch.acc;
    a.xy.reserve(nodes); a.kid.reserve(4 * nodes); a.len.reserve(nodes); a.edir.reserve(nodes);
    a.nkid.reserve(nodes); a.nl.reserve(nodes); a.nh.reserve(nodes); a.sink0.reserve(nodes);
    a.nsink.reserve(nodes); a.wd.reserve(nodes); a.ur.reserve(nodes); a.height.reserve(nodes);
    a.p_layer.reserve(sinks); a.p_cap.reserve(sinks); a.p_w.reserve(sinks); a.p_orig.reserve(sinks);
    a.fp.reserve(len + nodes);
    ch.node_off.reserve(ch.end - ch.beg + 1);
    ch.sink_off.reserve(ch.end - ch.beg + 1);
    ch.fp_off.reserve(ch.end - ch.beg + 1);
}

}  // namespace

// =============================================================== C ABI ======
extern "C" {

const char *la_last_error(void) { return g_err.c_str(); }

void la_shard_range(int64_t n, int32_t world, int32_t rank, int64_t *beg, int64_t *end) {
    if (world <= 0) world = 1;
    int64_t q = n / world, r = n % world;
    *beg = rank * q + std::min<int64_t>(rank, r);
    *end = *beg + q + (rank < r ? 1 : 0);
}

la_status la_init_grid(const la_grid_desc *g, la_ctx **out) {
    if (!g || !out) return set_err(LA_EINVAL, "null argument");
    *out = nullptr;
    if (g->L < 2 || g->L > MAXL) return set_err(LA_EINVAL, "L must be in [2, 16]");
    if (g->X <= 1 || g->Y <= 1 || g->X > 65535 || g->Y > 65535) return set_err(LA_EINVAL, "X, Y must be in [2, 65535]");
    // conflict-free batching sorts (element << 32 | rank) keys over 3 X Y footprint elements
    // (unit H edges, unit V edges, GCells): the element id must fit in 32 bits
    if ((uint64_t)3 * (uint64_t)g->X * (uint64_t)g->Y >= ((uint64_t)1 << 32))
        return set_err(LA_EINVAL, "grid too large: 3 X Y must be < 2^32 (footprint element ids)");
    if (!g->dir || !g->routable || !g->r || !g->c || !g->vr || !g->ofw || !g->wire_cap || !g->via_cap)
        return set_err(LA_EINVAL, "null grid array");
    const int L = g->L;
    if (!ok_nonneg(g->r, L) || !ok_nonneg(g->c, L) || !ok_nonneg(g->vr, L - 1) || !ok_nonneg(g->ofw, L))
        return set_err(LA_EINVAL, "negative (or NaN) r, c, vr or ofw");
    double ws[] = {g->W_D, g->W_CAP, g->W_CONG, g->W_VIA, g->s_pos, g->s_zero, g->w_floor};
    if (!ok_nonneg(ws, 7)) return set_err(LA_EINVAL, "negative (or NaN) weight or exponent");
    if (g->delta_lo > g->delta_hi) return set_err(LA_EINVAL, "delta_lo > delta_hi");
    if (g->world < 1 || g->world > 64 || g->rank < 0 || g->rank >= g->world) return set_err(LA_EINVAL, "bad rank/world");
    bool hasH = false, hasV = false;
    for (int l = 0; l < L; l++) {
        if (g->dir[l] > 1) return set_err(LA_EINVAL, "dir must be 0 or 1");
        if (g->routable[l]) (g->dir[l] == 0 ? hasH : hasV) = true;
    }
    if (!hasH || !hasV) return set_err(LA_EINVAL, "each direction needs a routable layer");

    la_ctx *ctx = new la_ctx();
    ctx->device = g->device;
    ctx->rank = g->rank;
    ctx->world = g->world;
    ctx->X = g->X; ctx->Y = g->Y; ctx->L = L;
    ctx->dir.assign(g->dir, g->dir + L);
    ctx->routable.assign(g->routable, g->routable + L);
    ctx->r.assign(g->r, g->r + L);
    ctx->c.assign(g->c, g->c + L);
    ctx->vr.assign(g->vr, g->vr + L - 1);
    ctx->ofw.assign(g->ofw, g->ofw + L);
    ctx->s_pos = g->s_pos; ctx->s_zero = g->s_zero;
    ctx->W_D = g->W_D; ctx->W_CAP = g->W_CAP; ctx->W_CONG = g->W_CONG; ctx->W_VIA = g->W_VIA;
    ctx->logit_k = g->logit_k; ctx->logit_b = g->logit_b; ctx->w_floor = g->w_floor;
    ctx->delta_lo = g->delta_lo; ctx->delta_hi = g->delta_hi;
    // r_avg (reading R6): mean of routable r, summed in ascending layer order
    if (std::isnan(g->r_avg)) {
        double s = 0.0;
        int cnt = 0;
        for (int l = 0; l < L; l++)
            if (g->routable[l]) { s = s + g->r[l]; cnt++; }
        ctx->r_avg = s / (double)cnt;
    } else {
        ctx->r_avg = g->r_avg;
    }
    ctx->wire_off.assign(L + 1, 0);
    for (int l = 0; l < L; l++) {
        int64_t n = g->dir[l] == 0 ? (int64_t)(g->X - 1) * g->Y : (int64_t)g->X * (g->Y - 1);
        ctx->wire_off[l + 1] = ctx->wire_off[l] + n;
        if (g->dir[l] == 0) ctx->LH++; else ctx->LV++;
    }
    ctx->n_wire_api = ctx->wire_off[L];
    ctx->n_via_api = (int64_t)(L - 1) * g->X * g->Y;
    {   // capacities >= 0, checked on the host threads (one pass over each array)
        const unsigned nthr = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        auto any_neg = [&](const int32_t *a, int64_t n) {
            std::atomic<bool> bad{false};
            par_chunks(n, n < (1 << 20) ? 1u : nthr, [&](unsigned, int64_t lo, int64_t hi) {
                int32_t m = 0;
                for (int64_t i = lo; i < hi; i++) m |= a[i];   // sign bit of any element
                if (m < 0) bad = true;
            });
            return bad.load();
        };
        if (any_neg(g->wire_cap, ctx->n_wire_api)) { delete ctx; return set_err(LA_EINVAL, "negative wire capacity"); }
        if (any_neg(g->via_cap, ctx->n_via_api)) { delete ctx; return set_err(LA_EINVAL, "negative via capacity"); }
    }

    // technology tables (O4): VR[a][b] ascending sums; Eq. (3) marginals with host libm
    std::memset(&ctx->tab, 0, sizeof(TechTab));
    for (int l = 0; l < L; l++) {
        ctx->tab.r[l] = g->r[l];
        ctx->tab.c[l] = g->c[l];
        ctx->tab.ofw[l] = g->ofw[l];
        if (l < L - 1) ctx->tab.vr[l] = g->vr[l];
    }
    for (int a = 0; a < L; a++)
        for (int b = 0; b < L; b++) {
            double s = 0.0;
            for (int k = std::min(a, b); k < std::max(a, b); k++) s = s + g->vr[k];
            ctx->tab.VR[a * MAXL + b] = s;
        }
    const int nd = g->delta_hi - g->delta_lo + 1;
    std::vector<double> Mpos(nd), Mzero(nd);
    for (int i = 0; i < nd; i++) {
        double d = (double)(g->delta_lo + i);
        Mpos[i] = std::exp(g->s_pos * (d + 1.0)) - std::exp(g->s_pos * d);
        Mzero[i] = std::exp(g->s_zero * (d + 1.0)) - std::exp(g->s_zero * d);
    }

    cudaError_t e = cudaSetDevice(g->device);
    if (e != cudaSuccess) { delete ctx; return cuda_fail(nullptr, e, "cudaSetDevice"); }
    {   // keep freed device memory in the default pool for the next context (see dmalloc)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    if (g->stream) {
        ctx->stream = static_cast<cudaStream_t>(g->stream);
    } else {
        e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) { delete ctx; return cuda_fail(nullptr, e, "cudaStreamCreate"); }
        ctx->own_stream = true;
    }
    auto fail = [&](la_status st) { delete ctx; return st; };
    auto up = [&](auto **dst, const auto *src, size_t n) -> la_status {
        using T = std::remove_const_t<std::remove_reference_t<decltype(*src)>>;
        void *p = nullptr;
        cudaError_t ee = dmalloc(&p, std::max<size_t>(n * sizeof(T), 16));
        if (ee != cudaSuccess) return set_err(ee == cudaErrorMemoryAllocation ? LA_ENOMEM : LA_ECUDA,
                                              std::string("cudaMalloc: ") + cudaGetErrorString(ee));
        *dst = static_cast<T *>(p);
        if (src && n) {
            ee = cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream);
            if (ee != cudaSuccess) return set_err(LA_ECUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(ee));
            ctx->stats.h2d_bytes += (int64_t)(n * sizeof(T));
        }
        return LA_OK;
    };
    la_status st;
    ctx->n_wire_packed = (int64_t)(g->X - 1) * g->Y * ctx->LH + (int64_t)g->X * (g->Y - 1) * ctx->LV;
    if ((st = up(&ctx->d_wH, (const int32_t *)nullptr, (size_t)(g->X - 1) * g->Y * ctx->LH)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_wV, (const int32_t *)nullptr, (size_t)g->X * (g->Y - 1) * ctx->LV)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_via, (const int32_t *)nullptr, (size_t)ctx->n_via_api)) != LA_OK) return fail(st);
    // capacities (and initial demand) through the pinned pipeline (copy_many), not pageable copies
    if ((st = up(&ctx->d_wcap, (const int32_t *)nullptr, (size_t)ctx->n_wire_api)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_vcap, (const int32_t *)nullptr, (size_t)ctx->n_via_api)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_wire_off, ctx->wire_off.data(), (size_t)L + 1)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_Mpos, Mpos.data(), (size_t)nd)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_Mzero, Mzero.data(), (size_t)nd)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_tab, &ctx->tab, 1)) != LA_OK) return fail(st);
    int32_t *d_wdem0 = nullptr, *d_vdem0 = nullptr;
    if (g->wire_dem0 && (st = up(&d_wdem0, (const int32_t *)nullptr, (size_t)ctx->n_wire_api)) != LA_OK) return fail(st);
    if (g->via_dem0 && (st = up(&d_vdem0, (const int32_t *)nullptr, (size_t)ctx->n_via_api)) != LA_OK) return fail(st);
    {
        std::vector<Xfer> xs{{ctx->d_wcap, g->wire_cap, sizeof(int32_t) * (size_t)ctx->n_wire_api},
                             {ctx->d_vcap, g->via_cap, sizeof(int32_t) * (size_t)ctx->n_via_api}};
        if (d_wdem0) xs.push_back({d_wdem0, g->wire_dem0, sizeof(int32_t) * (size_t)ctx->n_wire_api});
        if (d_vdem0) xs.push_back({d_vdem0, g->via_dem0, sizeof(int32_t) * (size_t)ctx->n_via_api});
        e = cudaStreamSynchronize(ctx->stream);   // the small table uploads above are on ctx->stream
        if (e == cudaSuccess) e = copy_many(xs, g->device, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            if (d_wdem0) dfree(d_wdem0);
            if (d_vdem0) dfree(d_vdem0);
            delete ctx;
            return cuda_fail(nullptr, e, "grid upload");
        }
        for (const Xfer &x : xs) ctx->stats.h2d_bytes += (int64_t)x.bytes;
    }

    DevGrid &G = ctx->G;
    G.X = g->X; G.Y = g->Y; G.L = L; G.LH = ctx->LH; G.LV = ctx->LV;
    int ih = 0, iv = 0;
    for (int l = 0; l < MAXL; l++) {
        G.dir[l] = l < L ? g->dir[l] : 0;
        G.routable[l] = l < L ? g->routable[l] : 0;
        G.lidx[l] = l < L ? (int8_t)(g->dir[l] == 0 ? ih++ : iv++) : 0;
    }
    G.delta_lo = g->delta_lo; G.delta_hi = g->delta_hi;
    G.W_D = g->W_D; G.W_CAP = g->W_CAP; G.W_CONG = g->W_CONG; G.W_VIA = g->W_VIA;
    G.wH = ctx->d_wH; G.wV = ctx->d_wV; G.via = ctx->d_via;
    G.Mpos = ctx->d_Mpos; G.Mzero = ctx->d_Mzero; G.tab = ctx->d_tab;
    e = launch_pack_state(G, ctx->d_wcap, d_wdem0, ctx->d_vcap, d_vdem0, ctx->d_wire_off, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (d_wdem0) dfree(d_wdem0);
    if (d_vdem0) dfree(d_vdem0);
    if (e != cudaSuccess) { delete ctx; return cuda_fail(nullptr, e, "pack initial state"); }
    // pristine copy of the initial packed state for la_reset
    size_t bH = sizeof(int32_t) * (size_t)(g->X - 1) * g->Y * ctx->LH;
    size_t bV = sizeof(int32_t) * (size_t)g->X * (g->Y - 1) * ctx->LV;
    size_t bVia = sizeof(int32_t) * (size_t)ctx->n_via_api;
    if ((st = up(&ctx->d_wH0, (const int32_t *)nullptr, bH / 4)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_wV0, (const int32_t *)nullptr, bV / 4)) != LA_OK) return fail(st);
    if ((st = up(&ctx->d_via0, (const int32_t *)nullptr, bVia / 4)) != LA_OK) return fail(st);
    e = cudaMemcpyAsync(ctx->d_wH0, ctx->d_wH, bH, cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->d_wV0, ctx->d_wV, bV, cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->d_via0, ctx->d_via, bVia, cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) { delete ctx; return cuda_fail(nullptr, e, "snapshot initial state"); }

    ctx->host_xport = g->world > 1 && !g->nccl_id;   // ranks reconciled by the caller (la_get/put_decisions)
    ctx->nccl = g->nccl_id != nullptr;                // world 1 with an id: the NCCL reconcile on one GPU
    if (g->nccl_id) {
        ncclUniqueId id;
        std::memcpy(&id, g->nccl_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&ctx->comm, g->world, id, g->rank);
        if (r != ncclSuccess) {
            delete ctx;
            return set_err(LA_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
    }
    *out = ctx;
    return LA_OK;
}

static std::vector<int4> pack_nets(const la_ctx *ctx, const std::vector<int32_t> &pos);

la_status la_load_nets(la_ctx *ctx, const la_net_desc *n, int32_t *n_batches) {
    if (!ctx || !n) return set_err(LA_EINVAL, "null argument");
    if (ctx->poisoned) return set_err(LA_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    if (ctx->loaded) return set_err(LA_ESTATE, "nets already loaded");
    if (n->n_nets < 0) return set_err(LA_EINVAL, "bad net descriptor");
    if (n->n_nets > 0) {
        if (!n->pin_ptr || !n->seg_ptr || !n->pin_x || !n->pin_y || !n->pin_layer || !n->pin_cap || !n->pin_slack)
            return set_err(LA_EINVAL, "bad net descriptor: null array");
        if (!n->seg_xy && n->seg_ptr[n->n_nets] > 0) return set_err(LA_EINVAL, "bad net descriptor: null seg_xy");
    }
    if (n->n_nets >= ((int64_t)1 << 31)) return set_err(LA_EINVAL, "too many nets");
    CK(cudaSetDevice(ctx->device));
    auto t0 = std::chrono::steady_clock::now();
    const bool verbose = getenv("GAPLA_VERBOSE") != nullptr;   // phase times of la_load_nets to stderr
    auto tph = t0;
    auto phase = [&](const char *what) {
        if (!verbose) return;
        auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[gapla load] %-28s %9.1f ms\n", what, std::chrono::duration<double, std::milli>(t - tph).count());
        tph = t;
    };
    const int64_t N = n->n_nets;
    ctx->n_nets = N;
    ctx->n_pins = N > 0 ? n->pin_ptr[N] : 0;

    // ---- build every net's tree in parallel (input-order chunks)
    unsigned nthr = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (N < 4096) nthr = 1;
    const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(N, (int64_t)nthr * 8));
    std::vector<Chunk> chunks(nchunks);
    for (int64_t c = 0; c < nchunks; c++) {
        chunks[c].beg = N * c / nchunks;
        chunks[c].end = N * (c + 1) / nchunks;
    }
    std::atomic<int64_t> next{0};
    auto worker = [&]() {
        Builder B{ctx, n};
        for (int l = 0; l < ctx->L; l++) if (ctx->routable[l]) B.nlegal[ctx->dir[l]]++;
        for (;;) {
            int64_t c = next.fetch_add(1);
            if (c >= nchunks) break;
            Chunk &ch = chunks[c];
            reserve_chunk(ch, n);
            ch.node_off.assign(1, 0);
            ch.sink_off.assign(1, 0);
            ch.fp_off.assign(1, 0);
            for (int64_t net = ch.beg; net < ch.end; net++) {
                BuiltNet &a = ch.acc;                        // the net's tree is appended to the chunk
                std::string err = B.build(net, a);
                if (!err.empty()) { ch.err = err; ch.err_net = net; break; }
                ch.node_off.push_back((int64_t)a.xy.size());
                ch.sink_off.push_back((int64_t)a.p_layer.size());
                ch.fp_off.push_back((int64_t)a.fp.size());
                ch.max_height = std::max<int>(ch.max_height, B.last_height);
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned i = 1; i < nthr; i++) th.emplace_back(worker);
        worker();
        for (auto &t : th) t.join();
    }
    phase("  build threads");
    for (auto &ch : chunks)
        if (ch.err_net >= 0) return set_err(LA_EINVAL, ch.err);

    // per-net index: chunk and local position; flat per-net node and sink counts
    hvec<int32_t> chunk_of(N);                // (default-initialised: every element is written)
    for (int64_t c = 0; c < nchunks; c++)
        for (int64_t i = chunks[c].beg; i < chunks[c].end; i++) chunk_of[i] = (int32_t)c;
    hvec<int32_t> nn_of(N), ns_of(N);
    par_for(N, nthr, [&](int64_t net) {
        const Chunk &ch = chunks[chunk_of[net]];
        const int64_t i = net - ch.beg;
        nn_of[net] = (int32_t)std::min<int64_t>(ch.node_off[i + 1] - ch.node_off[i], INT32_MAX);
        ns_of[net] = (int32_t)std::min<int64_t>(ch.sink_off[i + 1] - ch.sink_off[i], INT32_MAX);
    });
    auto nnodes_of = [&](int64_t net) { return (int64_t)nn_of[net]; };
    auto nsinks_of = [&](int64_t net) { return (int64_t)ns_of[net]; };
    // nets whose whole DP state fits a group's shared-memory slot (SLOT_BYTES) stay
    // on chip; the slot's node capacity NS follows from the layer count
    ctx->LD = std::max(ctx->LH, ctx->LV);
    {
        int64_t budget = SLOT_BYTES;
        if (const char *e = getenv("GAPLA_SLOT_BYTES")) budget = std::max(512, atoi(e));
        int ns = 1;
        while (assign_net_bytes(ns + 1, ctx->NP, ctx->L, ctx->LD) <= (size_t)budget) ns++;
        ctx->NS = ns;
    }
    if (const char *e = getenv("GAPLA_NS")) ctx->NS = std::max(1, std::min(1024, atoi(e)));   // tuning knobs
    if (const char *e = getenv("GAPLA_NP")) ctx->NP = std::max(1, std::min(4096, atoi(e)));
    // batch mode (k_assign_g): a net is "big" when its group-path state does not fit a warp's
    // arena; the dataflow kernel (k_assign) re-classifies by its own slot (NS, NP)
    ctx->warp_arena = (int32_t)assign_warp_arena_bytes(ctx->L, ctx->LD);
    if (const char *e = getenv("GAPLA_GROUP")) ctx->group_path = atoi(e) != 0;
    auto is_big_flow = [&](int64_t net) { return nnodes_of(net) > ctx->NS || nsinks_of(net) > ctx->NP; };
    // small nets (one 8-lane group each, four per warp) up to nmax nodes; larger nets run
    // level-parallel on a team of groups (DESIGN §5 "group path").  nmax is per batch: a batch
    // with many nets per resident warp is throughput-bound and keeps nets up to group_nmax_thr
    // nodes on the (more efficient) group path; a smaller batch is bound by its slowest net and
    // sends nets above group_nmax_lat nodes to the (lower-latency) team path.
    int64_t group_nmax_lat = 8, group_nmax_thr = 24;
    if (const char *e = getenv("GAPLA_GROUP_NMAX")) group_nmax_lat = group_nmax_thr = std::max(1, std::min(65535, atoi(e)));
    if (const char *e = getenv("GAPLA_GROUP_NMAX_LAT")) group_nmax_lat = std::max(1, std::min(65535, atoi(e)));
    if (const char *e = getenv("GAPLA_GROUP_NMAX_THR")) group_nmax_thr = std::max(1, std::min(65535, atoi(e)));
    std::vector<int32_t> nmax_of_batch;       // filled once the batches are known
    // nets whose group-path state exceeds a warp arena, once per net (in parallel)
    std::vector<uint8_t> over_arena(N, 0);
    if (ctx->group_path)
        par_for(N, nthr, [&](int64_t net) {
            over_arena[net] = assign_group_net_bytes((int)nnodes_of(net), (int)nsinks_of(net), ctx->L, ctx->LD) >
                              (size_t)ctx->warp_arena;
        });
    auto is_big = [&](int64_t net, int32_t b) {
        if (!ctx->group_path) return is_big_flow(net);
        return nnodes_of(net) > nmax_of_batch[b] || over_arena[net] != 0;
    };
    for (int64_t net = 0; net < N; net++)
        if (nnodes_of(net) >= 65535 || nsinks_of(net) >= 65535)
            return set_err(LA_EINVAL, "net " + std::to_string(net) + ": more than 65534 LA-tree nodes or sinks");

    phase("tree build");
    std::vector<int64_t> cnode(nchunks + 1, 0), csink(nchunks + 1, 0), cfp(nchunks + 1, 0);
    for (int64_t c = 0; c < nchunks; c++) {
        cnode[c + 1] = cnode[c] + (int64_t)chunks[c].acc.xy.size();
        csink[c + 1] = csink[c] + (int64_t)chunks[c].acc.p_layer.size();
        cfp[c + 1] = cfp[c] + (int64_t)chunks[c].acc.fp.size();
    }
    uint64_t *d_fp_raw = nullptr;   // the footprints as built (input order), for the GPU keys
    // ---- upload the trees as built (input-order chunks) on a background thread while the host
    // orders and batches the nets: the copies depend on the build only (k_permute_forest lays the
    // forest out batch-major once the order is known).  The thread owns its allocations until the
    // join below; every return path between here and the join joins it first (UpJoin).
    ForestSrc src{};
    std::vector<void *> raw;                                // input-order device copies, freed below
    cudaError_t up_err = cudaSuccess;
    int64_t up_bytes = 0;
    std::thread up_thr([&]() {
        std::vector<Xfer> xfers;
        auto raw_up = [&](auto member, const std::vector<int64_t> &base, int per, auto **dst) -> cudaError_t {
            using T = typename std::remove_reference<decltype(chunks[0].acc.*member)>::type::value_type;
            T *d = nullptr;
            cudaError_t e = dmalloc(&d, sizeof(T) * std::max<int64_t>(base[nchunks] * per, 1));
            if (e != cudaSuccess) return e;
            raw.push_back(d);
            for (int64_t c = 0; c < nchunks; c++) {
                const auto &v = chunks[c].acc.*member;
                if (v.empty()) continue;
                xfers.push_back({d + base[c] * per, v.data(), sizeof(T) * v.size()});
                up_bytes += (int64_t)(sizeof(T) * v.size());
            }
            *dst = d;
            return cudaSuccess;
        };
        cudaError_t e = cudaSetDevice(ctx->device);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::xy, cnode, 1, &src.xy);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::kid, cnode, 4, &src.kid);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::len, cnode, 1, &src.len);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::sink0, cnode, 1, &src.sink0);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::edir, cnode, 1, &src.edir);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::nkid, cnode, 1, &src.nkid);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::nl, cnode, 1, &src.nl);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::nh, cnode, 1, &src.nh);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::nsink, cnode, 1, &src.nsink);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::height, cnode, 1, &src.height);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::wd, cnode, 1, &src.wd);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::ur, cnode, 1, &src.ur);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::p_layer, csink, 1, &src.p_layer);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::p_cap, csink, 1, &src.p_cap);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::p_w, csink, 1, &src.p_w);
        if (e == cudaSuccess) e = raw_up(&BuiltNet::p_orig, csink, 1, &src.p_orig);
        if (e == cudaSuccess && ctx->snap_batch.empty()) e = raw_up(&BuiltNet::fp, cfp, 1, &d_fp_raw);
        if (e == cudaSuccess) e = copy_many(xfers, ctx->device, cudaMemcpyHostToDevice);
        up_err = e;
    });
    struct UpJoin {
        std::thread &t;
        std::vector<void *> &raw;
        ~UpJoin() {
            if (t.joinable()) {   // an early return: wait for the copies, then free their buffers
                t.join();
                for (void *p : raw) dfree(p);
            }
        }
    } up_join{up_thr, raw};
    // ---- priority order (order_key, index) and footprint keys (element << 32 | rank)
    hvec<int64_t> by_rank(N);
    // key range of order_key: a small range (priorities, wirelengths) is ordered by a parallel
    // counting sort, stable in input order -- the same (key, index) order as the comparison sort
    int64_t kmin = 0, kmax = -1;
    if (n->order_key && N > 0) {
        const unsigned nt = std::max(1u, nthr);
        std::vector<int64_t> lo(nt, INT64_MAX), hi(nt, INT64_MIN);
        par_chunks(N, nt, [&](unsigned t, int64_t a, int64_t b) {
            for (int64_t i = a; i < b; i++) { lo[t] = std::min(lo[t], n->order_key[i]); hi[t] = std::max(hi[t], n->order_key[i]); }
        });
        kmin = *std::min_element(lo.begin(), lo.end());
        kmax = *std::max_element(hi.begin(), hi.end());
    }
    const uint64_t span = (uint64_t)kmax - (uint64_t)kmin;    // no signed overflow for any key range
    const unsigned nt_c = (unsigned)std::max<int64_t>(1, std::min<int64_t>(std::max(1u, nthr), N / 65536 + 1));
    bool permutation = false;                           // keys kmin .. kmin+N-1, each once: rank = key - kmin
    if (n->order_key && N > 0 && span == (uint64_t)(N - 1)) {
        par_for(N, nthr, [&](int64_t r) { by_rank[r] = -1; });
        par_for(N, nthr, [&](int64_t i) { by_rank[n->order_key[i] - kmin] = i; });
        std::atomic<bool> full{true};
        par_chunks(N, nt_c, [&](unsigned, int64_t a, int64_t b) {
            for (int64_t r = a; r < b; r++) if (by_rank[r] < 0) { full = false; break; }
        });
        permutation = full;                             // N writes fill N slots only if no key repeats
        if (permutation) phase("  priority order (permutation)");
    }
    const bool counting = !permutation && n->order_key && N > 0 &&
                          span < (uint64_t)std::min<int64_t>(N + 1024, ((int64_t)1 << 23) / nt_c);   // <= 64 MB of counters
    if (counting) {
        const int64_t R = kmax - kmin + 1;
        const unsigned nt = nt_c;
        std::vector<std::vector<int64_t>> cnt(nt, std::vector<int64_t>(R, 0));
        par_chunks(N, nt, [&](unsigned t, int64_t a, int64_t b) {
            for (int64_t i = a; i < b; i++) cnt[t][n->order_key[i] - kmin]++;
        });
        int64_t run = 0;                                    // exclusive offsets, key-major, then thread (input) order
        for (int64_t k = 0; k < R; k++)
            for (unsigned t = 0; t < nt; t++) { const int64_t c = cnt[t][k]; cnt[t][k] = run; run += c; }
        par_chunks(N, nt, [&](unsigned t, int64_t a, int64_t b) {
            for (int64_t i = a; i < b; i++) by_rank[cnt[t][n->order_key[i] - kmin]++] = i;
        });
        phase("  priority sort (counting)");
    } else if (permutation) {
    } else if (n->order_key) {
        // sort (key, index) pairs in place of indices: contiguous keys, no indirection in the comparator
        std::vector<std::pair<int64_t, int64_t>> kv(N);
        par_for(N, nthr, [&](int64_t i) { kv[i] = {n->order_key[i], i}; });
        par_sort(kv, [](const std::pair<int64_t, int64_t> &a, const std::pair<int64_t, int64_t> &b) { return a < b; },
                 nthr);
        par_for(N, nthr, [&](int64_t r) { by_rank[r] = kv[r].second; });
        phase("  priority sort");
    } else {
        for (int64_t i = 0; i < N; i++) by_rank[i] = i;
    }
    // footprint keys (element << 32 | rank) are formed on the GPU from the as-built footprints
    // (k_fp_keys, one thread per input net, in place: the radix sort makes the order irrelevant)
    hvec<int64_t> fp_start(N + 1);
    fp_start[0] = 0;
    par_for(N, nthr, [&](int64_t net) {
        const Chunk &ch = chunks[chunk_of[net]];
        const int64_t i = net - ch.beg;
        fp_start[net + 1] = ch.fp_off[i + 1] - ch.fp_off[i];
    });
    par_prefix(fp_start.data() + 1, N, nthr);
    const int64_t n_fp = fp_start[N];
    phase("  footprint offsets");
    int elem_bits = 1;
    while (((uint64_t)1 << elem_bits) < (uint64_t)3 * ctx->X * ctx->Y) elem_bits++;
    auto t1 = std::chrono::steady_clock::now();

    phase("priority order + keys");
    // ---- GPU conflict-free batching (K1/K2)
    std::vector<int32_t> batch_of_rank;
    int32_t nb = 0;
    DagDev dag;
    const bool snapshot = !ctx->snap_batch.empty();
    if (snapshot) {
        // paper-style batches (NEXT #1, R31): the caller's ids, no conflict DAG
        if ((int64_t)ctx->snap_batch.size() != N) return set_err(LA_EINVAL, "snapshot batches: wrong net count");
        batch_of_rank.resize(N);
        for (int64_t r = 0; r < N; r++) {
            const int32_t b = ctx->snap_batch[by_rank[r]];
            if (b < 0) return set_err(LA_EINVAL, "snapshot batches: negative batch id");
            batch_of_rank[r] = b;
            nb = std::max(nb, b + 1);
        }
    } else {
        up_thr.join();   // the footprints must have landed
        CK(up_err);
        hvec<int32_t> rank_of(N);
        par_for(N, nthr, [&](int64_t r) { rank_of[by_rank[r]] = (int32_t)r; });
        uint64_t *d_keys = nullptr;
        int64_t *d_fps = nullptr;
        int32_t *d_rank = nullptr;
        cudaError_t e = dmalloc(&d_keys, sizeof(uint64_t) * (size_t)std::max<int64_t>(n_fp, 1));
        if (e == cudaSuccess) e = dmalloc(&d_fps, sizeof(int64_t) * (size_t)(N + 1));
        if (e == cudaSuccess) e = dmalloc(&d_rank, sizeof(int32_t) * (size_t)std::max<int64_t>(N, 1));
        if (e == cudaSuccess) e = pinned_copy(d_fps, fp_start.data(), sizeof(int64_t) * (size_t)(N + 1), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = pinned_copy(d_rank, rank_of.data(), sizeof(int32_t) * (size_t)N, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = launch_fp_keys(d_fp_raw, d_fps, d_rank, N, d_keys, ctx->stream);
        ctx->stats.h2d_bytes += 8 * (N + 1) + 4 * N;
        ctx->stats.launches += 1;
        if (e == cudaSuccess)
            e = gpu_conflict_batches(nullptr, d_keys, n_fp, elem_bits, N, batch_of_rank, nb, ctx->stream,
                                     &ctx->stats.launches, &dag);
        cudaStreamSynchronize(ctx->stream);
        dfree(d_keys);
        dfree(d_fps);
        dfree(d_rank);
        if (e != cudaSuccess) { dag.release(); return cuda_fail(ctx, e, "conflict-free batching"); }
    }
    auto t2 = std::chrono::steady_clock::now();
    ctx->batch_of_net.assign(N, 0);
    par_for(N, nthr, [&](int64_t r) { ctx->batch_of_net[by_rank[r]] = batch_of_rank[r]; });

    phase("GPU batching");
    // ---- batch-major net order: by batch, then node count descending, then rank
    hvec<int64_t> pos_net(N);          // final position -> input net
    {
        std::vector<int64_t> cnt(nb + 1, 0);
        for (int64_t i = 0; i < N; i++) cnt[ctx->batch_of_net[i] + 1]++;
        for (int32_t b = 0; b < nb; b++) cnt[b + 1] += cnt[b];
        ctx->batch_net0.assign(cnt.begin(), cnt.end());
        std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
        for (int64_t r = 0; r < N; r++) pos_net[cur[batch_of_rank[r]]++] = by_rank[r];
        {
            int lat = 0, thr = 0, n_sm = 0;
            CK(assign_g_resident_ctas(ctx->L, ctx->LD, &lat, &thr));
            CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, ctx->device));
            int64_t per_warp = 8;
            if (const char *e = getenv("GAPLA_NMAX_NETS_PER_WARP")) per_warp = std::max(1, atoi(e));
            const int64_t warps = (int64_t)std::max(1, thr * n_sm) * ASSIGN_WARPS;
            nmax_of_batch.resize(std::max(nb, 1));
            for (int32_t b = 0; b < nb; b++)
                nmax_of_batch[b] = (int32_t)((cnt[b + 1] - cnt[b]) > per_warp * warps * ctx->world ? group_nmax_thr
                                                                                                   : group_nmax_lat);
        }
        // big nets (CTA path) first, then by node count descending, then rank: the longest nets
        // start first.  Key per position: !big | (65535 - nodes) | offset in the batch (rank order).
        std::atomic<int32_t> nxt{0};
        auto sorter = [&]() {
            std::vector<uint64_t> kk;
            for (;;) {
                const int32_t b = nxt.fetch_add(1);
                if (b >= nb) break;
                const int64_t p0 = ctx->batch_net0[b], p1 = ctx->batch_net0[b + 1];
                kk.resize(p1 - p0);
                for (int64_t p = p0; p < p1; p++) {
                    const int64_t net = pos_net[p];
                    kk[p - p0] = ((uint64_t)(is_big(net, b) ? 0 : 1) << 63) | ((uint64_t)(65535 - nn_of[net]) << 40) |
                                 (uint64_t)(p - p0);
                }
                std::sort(kk.begin(), kk.end());
                std::vector<int64_t> tmp(pos_net.begin() + p0, pos_net.begin() + p1);
                for (int64_t q = 0; q < p1 - p0; q++) pos_net[p0 + q] = tmp[kk[q] & ((1ull << 40) - 1)];
            }
        };
        std::vector<std::thread> th;
        for (unsigned i = 1; i < nthr; i++) th.emplace_back(sorter);
        sorter();
        for (auto &t : th) t.join();
    }
    phase("batch-major order");
    // role lists: big nets (CTA path) and small nets (group path), both in
    // forest = topological order; per batch the big nets are its leading positions
    int64_t max_big_nodes = 0, max_big_sinks = 0;
    std::vector<int32_t> big_pos, small_pos;
    big_pos.reserve(N / 16 + 1);
    small_pos.reserve(N);
    ctx->batch_big0.assign(1, 0);
    ctx->batch_small0.assign(1, 0);
    hvec<uint8_t> big_at(N);
    par_for(N, nthr, [&](int64_t p) {
        const int64_t net = pos_net[p];
        big_at[p] = is_big(net, ctx->batch_of_net[net]) ? 1 : 0;
    });
    {   // per batch (host threads over batches): counts, then the lists filled at their offsets
        std::vector<int64_t> nbig(nb, 0);
        std::vector<int64_t> mxn(nthr, 0), mxs(nthr, 0);
        auto over_batches = [&](auto body) {
            std::atomic<int32_t> nx{0};
            auto w = [&](unsigned t) { for (int32_t b; (b = nx.fetch_add(1)) < nb;) body(t, b); };
            std::vector<std::thread> th;
            for (unsigned i = 1; i < nthr && nb > 1; i++) th.emplace_back(w, i);
            w(0);
            for (auto &x : th) x.join();
        };
        over_batches([&](unsigned t, int32_t b) {
            int64_t c = 0;
            for (int64_t p = ctx->batch_net0[b]; p < ctx->batch_net0[b + 1]; p++)
                if (big_at[p]) {
                    const int64_t net = pos_net[p];
                    c++;
                    mxn[t] = std::max(mxn[t], nnodes_of(net));
                    mxs[t] = std::max(mxs[t], nsinks_of(net));
                }
            nbig[b] = c;
        });
        for (int32_t b = 0; b < nb; b++) {
            ctx->batch_big0.push_back(ctx->batch_big0.back() + nbig[b]);
            ctx->batch_small0.push_back(ctx->batch_small0.back() + (ctx->batch_net0[b + 1] - ctx->batch_net0[b]) - nbig[b]);
        }
        big_pos.resize(ctx->batch_big0.back());
        small_pos.resize(ctx->batch_small0.back());
        over_batches([&](unsigned, int32_t b) {
            int64_t ib = ctx->batch_big0[b], is = ctx->batch_small0[b];
            for (int64_t p = ctx->batch_net0[b]; p < ctx->batch_net0[b + 1]; p++) {
                if (big_at[p]) big_pos[ib++] = (int32_t)p;
                else small_pos[is++] = (int32_t)p;
            }
        });
        // the dataflow kernel's (k_assign) big nets: input order
        par_chunks(N, nthr, [&](unsigned t, int64_t lo, int64_t hi) {
            for (int64_t net = lo; net < hi; net++)
                if (is_big_flow(net)) {
                    mxn[t] = std::max(mxn[t], nnodes_of(net));
                    mxs[t] = std::max(mxs[t], nsinks_of(net));
                }
        });
        for (unsigned t = 0; t < nthr; t++) {
            max_big_nodes = std::max(max_big_nodes, mxn[t]);
            max_big_sinks = std::max(max_big_sinks, mxs[t]);
        }
    }
    phase("role lists");
    // dataflow DAG in forest order (snapshot batches: none -- every net has 0 predecessors)
    if (snapshot) {
        std::vector<int64_t> zoff(N + 1, 0);
        TRY(dev_upload(ctx, &ctx->d_succ_off, zoff.data(), N + 1));
        TRY(dev_alloc(ctx, &ctx->d_succ, 1));
        TRY(dev_alloc(ctx, &ctx->d_indeg, std::max<int64_t>(N, 1)));
        CK(cudaMemsetAsync(ctx->d_indeg, 0, sizeof(int32_t) * std::max<int64_t>(N, 1), ctx->stream));
        for (int i = 0; i < 3; i++) ctx->dev_allocs.pop_back();   // owned by the ctx fields, freed in ~la_ctx
        ctx->fuse_commit = false;                                  // commits after the whole batch (snapshot)
        ctx->schedule = LA_SCHED_BATCH;
    } else {
        hvec<int64_t> rank_of_net(N), rank_of_pos(N);
        par_for(N, nthr, [&](int64_t r) { rank_of_net[by_rank[r]] = r; });
        par_for(N, nthr, [&](int64_t p) { rank_of_pos[p] = rank_of_net[pos_net[p]]; });
        cudaError_t e = gpu_dag_to_positions(dag, rank_of_pos.data(), &ctx->d_succ_off, &ctx->d_succ, &ctx->d_indeg,
                                             ctx->stream, &ctx->stats.launches);
        if (e != cudaSuccess) { dag.release(); return cuda_fail(ctx, e, "dependency DAG"); }
        ctx->stats.h2d_bytes += 8 * N;
    }
    phase("DAG to positions");
    // offsets in final order
    hvec<int64_t> node0(N + 1), sink0g(N + 1);
    node0[0] = 0;
    sink0g[0] = 0;
    int64_t max_nodes = 0;
    {
        std::vector<int64_t> mx(nthr, 0);
        par_chunks(N, nthr, [&](unsigned t, int64_t lo, int64_t hi) {
            int64_t m = 0;
            for (int64_t p = lo; p < hi; p++) {
                node0[p + 1] = nn_of[pos_net[p]];
                sink0g[p + 1] = ns_of[pos_net[p]];
                m = std::max<int64_t>(m, node0[p + 1]);
            }
            mx[t] = m;
        });
        for (int64_t m : mx) max_nodes = std::max(max_nodes, m);
        par_prefix(node0.data() + 1, N, nthr);
        par_prefix(sink0g.data() + 1, N, nthr);
    }
    const int64_t NN = node0[N], NS = sink0g[N];
    ctx->n_nodes = NN;
    ctx->n_sinks = NS;
    phase("offsets");
    if (NN >= ((int64_t)1 << 31) || NS >= ((int64_t)1 << 31)) return set_err(LA_EINVAL, "forest too large");
    // ---- upload the trees as built (chunk by chunk, input order); k_permute_forest lays them out
    // batch-major on the GPU (rebasing child ids and sink offsets) -- no host staging pass
    if (cnode[nchunks] != NN || csink[nchunks] != NS) return set_err(LA_EINVAL, "internal: forest size mismatch");
    hvec<int64_t> src_node0(N), src_sink0(N);
    hvec<uint8_t> pdrv(N);
    hvec<int64_t> net_id(N);
    par_for(N, nthr, [&](int64_t p) {
        const int64_t net = pos_net[p];
        const int32_t c = chunk_of[net];
        const Chunk &ch = chunks[c];
        const int64_t i = net - ch.beg;
        src_node0[p] = cnode[c] + ch.node_off[i];
        src_sink0[p] = csink[c] + ch.sink_off[i];
        net_id[p] = net;
        pdrv[p] = n->pin_layer[n->pin_ptr[net]];
    });
    int64_t wl = 0, wsw = 0;
    int maxh = 0;
    for (auto &ch : chunks) { wl += ch.acc.wl; wsw += ch.acc.wsw; maxh = std::max(maxh, ch.max_height); }
    phase("forest source offsets");

    // the as-built arrays were uploaded by the background thread started after the build
    if (up_thr.joinable()) up_thr.join();
    CK(up_err);
    ctx->stats.h2d_bytes += up_bytes;
    int64_t *d_srcn = nullptr, *d_srcs = nullptr, *d_dsts = nullptr;
    CK(dmalloc(&d_srcn, sizeof(int64_t) * std::max<int64_t>(N, 1))); raw.push_back(d_srcn);
    CK(dmalloc(&d_srcs, sizeof(int64_t) * std::max<int64_t>(N, 1))); raw.push_back(d_srcs);
    CK(dmalloc(&d_dsts, sizeof(int64_t) * (N + 1))); raw.push_back(d_dsts);
    CK(copy_many({{d_srcn, src_node0.data(), sizeof(int64_t) * (size_t)N},
                  {d_srcs, src_sink0.data(), sizeof(int64_t) * (size_t)N},
                  {d_dsts, sink0g.data(), sizeof(int64_t) * (size_t)(N + 1)}}, ctx->device, cudaMemcpyHostToDevice));
    ctx->stats.h2d_bytes += 8 * (3 * N + 1);
    src.src_node0 = d_srcn; src.src_sink0 = d_srcs; src.dst_sink0 = d_dsts;
    // the as-built host arrays (GBs) are released on a background thread, joined by ~la_ctx
    ctx->free_thr = std::thread([c = std::move(chunks)]() mutable { c.clear(); c.shrink_to_fit(); });
    phase("forest upload (as built)");

    DevForest &F = ctx->F;
    F.n_nets = N; F.n_nodes = NN; F.n_sinks = NS;
    uint32_t *d_xy; int32_t *d_kid, *d_len, *d_sink0; uint8_t *d_edir, *d_nkid, *d_nl, *d_nh, *d_pl, *d_pdrv;
    uint16_t *d_nsink, *d_height; double *d_wd, *d_ur, *d_pc, *d_pw; int64_t *d_po, *d_node0, *d_netid;
    TRY(dev_alloc(ctx, &d_xy, NN)); TRY(dev_alloc(ctx, &d_kid, NN * 4));
    TRY(dev_alloc(ctx, &d_len, NN)); TRY(dev_alloc(ctx, &d_sink0, NN));
    TRY(dev_alloc(ctx, &d_edir, NN)); TRY(dev_alloc(ctx, &d_nkid, NN));
    TRY(dev_alloc(ctx, &d_nl, NN)); TRY(dev_alloc(ctx, &d_nh, NN));
    TRY(dev_alloc(ctx, &d_nsink, NN)); TRY(dev_alloc(ctx, &d_wd, NN));
    TRY(dev_alloc(ctx, &d_height, NN));
    TRY(dev_alloc(ctx, &d_ur, NN)); TRY(dev_alloc(ctx, &d_pl, NS));
    TRY(dev_alloc(ctx, &d_pc, NS)); TRY(dev_alloc(ctx, &d_pw, NS));
    TRY(dev_alloc(ctx, &d_po, NS)); TRY(dev_alloc(ctx, &d_node0, N + 1));
    TRY(dev_alloc(ctx, &d_netid, N)); TRY(dev_alloc(ctx, &d_pdrv, N));
    CK(copy_many({{d_node0, node0.data(), sizeof(int64_t) * (size_t)(N + 1)},
                  {d_netid, net_id.data(), sizeof(int64_t) * (size_t)N}, {d_pdrv, pdrv.data(), (size_t)N}},
                 ctx->device, cudaMemcpyHostToDevice));
    ctx->stats.h2d_bytes += 8 * (2 * N + 1) + N;
    F.xy = d_xy; F.kid = d_kid; F.len = d_len; F.edir = d_edir; F.nkid = d_nkid; F.nl = d_nl; F.nh = d_nh;
    F.sink0 = d_sink0; F.nsink = d_nsink; F.wd = d_wd; F.ur = d_ur; F.p_layer = d_pl; F.p_cap = d_pc; F.p_w = d_pw;
    F.p_orig = d_po; F.net_node0 = d_node0; F.net_id = d_netid; F.net_pdrv = d_pdrv; F.height = d_height;
    CK(launch_permute_forest(F, src, ctx->stream));
    ctx->stats.launches += N > 0 ? 1 : 0;
    CK(cudaStreamSynchronize(ctx->stream));
    for (void *q : raw) dfree(q);
    DevScratch &S = ctx->S;
    TRY(dev_alloc(ctx, &S.froot, N));
    // la_get_solution's buffers (allocated here, with the rest of the context's device memory):
    // counts / offsets, costs, the CUB scan scratch, and the rows -- N trees have NN - N edges
    // (wires) and at most NN via stacks
    TRY(dev_alloc(ctx, &ctx->d_sol_w, 4 * (N + 1)));   // wcnt, vcnt, wptr, vptr
    TRY(dev_alloc(ctx, &ctx->d_sol_cost, std::max<int64_t>(N, 1)));
    TRY(dev_alloc(ctx, &ctx->d_sol_vc, 1));
    CK(sol_count(F, S, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &ctx->sol_temp_bytes,
                 ctx->stream));
    TRY(dev_alloc(ctx, &ctx->d_sol_temp, std::max<size_t>(ctx->sol_temp_bytes, 16)));
    TRY(dev_alloc(ctx, &ctx->d_sol_rows, std::max<int64_t>(5 * (NN - N) + 4 * NN, 1)));
    TRY(dev_alloc(ctx, &S.lay, NN)); TRY(dev_alloc(ctx, &S.sb, NN)); TRY(dev_alloc(ctx, &S.st, NN));
    TRY(dev_alloc(ctx, &S.Cd, NN)); TRY(dev_alloc(ctx, &S.rcv, NN)); TRY(dev_alloc(ctx, &S.Tin, NN));
    TRY(dev_alloc(ctx, &S.sink_delay, std::max<int64_t>(ctx->n_pins, 1)));
    TRY(dev_alloc(ctx, &S.net_cap, N)); TRY(dev_alloc(ctx, &S.net_rc, N));
    if (ctx->world > 1 || ctx->nccl) TRY(dev_alloc(ctx, &S.dec, NN));
    phase("scratch alloc");
    // persistent k_assign grid, tickets, dataflow counters, big-net slots
    {
        int per_sm = 0, per_sm_thr = 0, n_sm = 0;
        CK(assign_resident_ctas(ctx->L, ctx->LD, ctx->NS, ctx->NP, &per_sm, &per_sm_thr, &n_sm));
        if (per_sm < 1 || per_sm_thr < 1) return set_err(LA_ECUDA, "k_assign does not fit on an SM");
        ctx->grid = per_sm * n_sm;
        ctx->grid_thr = per_sm_thr * n_sm;
        if (const char *e = getenv("GAPLA_ASSIGN_VARIANT")) ctx->assign_variant = atoi(e) != 0 ? 1 : 0;
        if (const char *e = getenv("GAPLA_THR_NETS_PER_WARP")) ctx->thr_nets_per_warp = std::max(1, atoi(e));
        CK(dmalloc(&ctx->d_ticket, sizeof(unsigned long long) * 2 * (nb + 1)));
        CK(cudaMemsetAsync(ctx->d_ticket, 0, sizeof(unsigned long long) * 2 * (nb + 1), ctx->stream));
        ctx->h_big_pos = big_pos;
        ctx->h_small_pos = small_pos;
        ctx->h_net_node0.swap(node0);      // node0 / sink0g are read through the ctx from here on
        ctx->h_net_sink0.swap(sink0g);
        const hvec<int64_t> &nd0 = ctx->h_net_node0, &sk0 = ctx->h_net_sink0;
        phase("  (ticket alloc)");
        const std::vector<int4> ib = pack_nets(ctx, big_pos), is = pack_nets(ctx, small_pos);
        phase("  (pack_nets)");
        TRY(dev_upload(ctx, &ctx->d_big_pos, ib.data(), ib.size()));
        TRY(dev_upload(ctx, &ctx->d_small_pos, is.data(), is.size()));
        // k_assign_g jobs (DESIGN §5 "group path"): this rank's share of each batch's small
        // nets, in list order (nodes descending), up to four consecutive nets whose group
        // states fit one warp arena together
        {
            int lat = 0, thr = 0;
            CK(assign_g_resident_ctas(ctx->L, ctx->LD, &lat, &thr));
            if (lat < 1 || thr < 1) return set_err(LA_ECUDA, "k_assign_g does not fit on an SM");
            ctx->grid_g = lat * n_sm;
            ctx->grid_g_thr = thr * n_sm;
            ctx->h_jobs.clear();
            ctx->batch_job0.assign(1, 0);
            const int WA = ctx->warp_arena;
            // batches are packed independently (host threads over batches), then concatenated in order
            std::vector<std::vector<int4>> bj(ctx->group_path ? nb : 0);
            std::atomic<int32_t> nxb{0};
            auto packer = [&]() {
                for (int32_t b; (b = nxb.fetch_add(1)) < (int32_t)bj.size();) {
                    std::vector<int4> &out = bj[b];
                    const int64_t m0 = ctx->batch_small0[b], m1 = ctx->batch_small0[b + 1];
                    int64_t s0 = 0, s1 = 0;
                    la_shard_range(m1 - m0, ctx->world, ctx->rank, &s0, &s1);
                    int4 cur{0, 0, 0, 0};
                    int used = 0;
                    for (int64_t idx = m0 + s0; idx < m0 + s1; idx++) {
                        const int32_t p = small_pos[idx];
                        const int bytes = (int)assign_group_net_bytes((int)(nd0[p + 1] - nd0[p]), (int)(sk0[p + 1] - sk0[p]),
                                                                      ctx->L, ctx->LD);
                        if (cur.y == 4 || (cur.y > 0 && used + bytes > WA)) {
                            out.push_back(cur);
                            cur = int4{0, 0, 0, 0};
                            used = 0;
                        }
                        if (cur.y == 0) cur.x = (int32_t)idx;
                        else if (cur.y == 1) cur.z = used;
                        else if (cur.y == 2) cur.z |= used << 16;
                        else cur.w = used;
                        cur.y++;
                        used += bytes;
                    }
                    if (cur.y) out.push_back(cur);
                }
            };
            {
                std::vector<std::thread> th;
                for (unsigned i = 1; i < nthr && bj.size() > 1; i++) th.emplace_back(packer);
                packer();
                for (auto &t : th) t.join();
            }
            for (auto &v : bj) {
                ctx->h_jobs.insert(ctx->h_jobs.end(), v.begin(), v.end());
                ctx->batch_job0.push_back((int64_t)ctx->h_jobs.size());
            }
            if (ctx->group_path) TRY(dev_upload(ctx, &ctx->d_jobs, ctx->h_jobs.data(), ctx->h_jobs.size()));
        }
        // world > 1: this rank's nets of every batch (its big and small shards), for la_eval_timing
        if (ctx->world > 1) {
            std::vector<int32_t> own;
            for (int32_t b = 0; b < nb; b++) {
                int64_t s0 = 0, s1 = 0;
                const int64_t g0 = ctx->batch_big0[b], g1 = ctx->batch_big0[b + 1];
                la_shard_range(g1 - g0, ctx->world, ctx->rank, &s0, &s1);
                for (int64_t i = g0 + s0; i < g0 + s1; i++) own.push_back(big_pos[i]);
                const int64_t m0 = ctx->batch_small0[b], m1 = ctx->batch_small0[b + 1];
                la_shard_range(m1 - m0, ctx->world, ctx->rank, &s0, &s1);
                for (int64_t i = m0 + s0; i < m0 + s1; i++) own.push_back(small_pos[i]);
            }
            ctx->n_own = (int64_t)own.size();
            TRY(dev_upload(ctx, &ctx->d_own_pos, own.data(), std::max<size_t>(own.size(), 1)));
        }
        // big-net CTAs: one per SM by default (GAPLA_BIG_CTAS overrides), none without big nets
        ctx->n_big_ctas = big_pos.empty() ? 0 : n_sm;
        if (const char *e = getenv("GAPLA_BIG_CTAS")) ctx->n_big_ctas = std::max(0, atoi(e));
        if (!big_pos.empty()) ctx->n_big_ctas = std::max(1, std::min(ctx->n_big_ctas, ctx->grid - 1));
        if (const char *e = getenv("GAPLA_HYBRID")) ctx->hybrid = atoi(e) != 0;
        if (const char *e = getenv("GAPLA_BIG_SPLIT")) ctx->big_split = atoi(e);
        CK(dmalloc(&ctx->d_wait, sizeof(int32_t) * std::max<int64_t>(N, 1)));
        if (N) CK(cudaMemcpyAsync(ctx->d_wait, ctx->d_indeg, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        // a big net keeps its DP state in its half-CTA's shared memory, or in a global slot taken
        // from a pool: one slot per half-CTA up to a byte budget (GAPLA_GSLOT_MB, default 1024)
        const size_t need = std::max(assign_net_bytes((int)max_big_nodes, (int)max_big_sinks, ctx->L, ctx->LD),
                                     assign_team_net_bytes((int)max_big_nodes, (int)max_big_sinks, ctx->L, ctx->LD));
        ctx->gslot_bytes = 0;
        if (max_big_nodes > 0 && (need > assign_cta_net_bytes(ctx->L, ctx->LD, ctx->NS, ctx->NP) ||
                                  need > (size_t)2 * ctx->warp_arena)) {
            ctx->gslot_bytes = (int64_t)((need + 255) & ~(size_t)255);
            int64_t budget = (int64_t)1024 << 20;
            if (const char *e = getenv("GAPLA_GSLOT_MB")) budget = std::max<int64_t>(1, atoll(e)) << 20;
            const int64_t halves = 2 * (int64_t)std::max(std::max(ctx->grid, ctx->grid_thr),
                                                         std::max(ctx->grid_g, ctx->grid_g_thr));
            ctx->n_gslots = (int32_t)std::max<int64_t>(1, std::min<int64_t>(halves, budget / ctx->gslot_bytes));
            CK(dmalloc(&ctx->d_gscratch, (size_t)ctx->gslot_bytes * ctx->n_gslots));
            CK(dmalloc(&ctx->d_glock, sizeof(int32_t) * ctx->n_gslots));
            CK(cudaMemsetAsync(ctx->d_glock, 0, sizeof(int32_t) * ctx->n_gslots, ctx->stream));
        }
    }
    CK(cudaMemsetAsync(S.froot, 0, sizeof(double) * std::max<int64_t>(N, 1), ctx->stream));
    phase("  (slots)");
    CK(cudaStreamSynchronize(ctx->stream));
    phase("  (sync)");
    ctx->h_net_id.swap(net_id);
    phase("grid/tickets/slots");
    auto t3 = std::chrono::steady_clock::now();

    la_stats &stt = ctx->stats;
    stt.n_nets = N; stt.n_pins = ctx->n_pins; stt.n_nodes = NN; stt.n_sinks = NS;
    stt.wirelength = wl; stt.footprint = n_fp; stt.n_batches = nb; stt.max_height = maxh;
    stt.max_net_nodes = max_nodes;
    stt.wire_state_words = wsw;
    stt.via_state_words = NN * (ctx->L - 1);
    stt.h2d_bytes += n_fp * 8;      // batching keys
    stt.d2h_bytes += N * 4;         // batch ids
    stt.max_batch_nets = 0;
    for (int32_t b = 0; b < nb; b++)
        stt.max_batch_nets = std::max(stt.max_batch_nets, ctx->batch_net0[b + 1] - ctx->batch_net0[b]);
    stt.batch_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
    stt.load_ms = std::chrono::duration<double, std::milli>((t1 - t0) + (t3 - t2)).count();
    ctx->loaded = true;
    ctx->next_batch = 0;
    ctx->pending_commit = false;
    if (n_batches) *n_batches = nb;
    return LA_OK;
}

static la_status check_ready(la_ctx *ctx) {
    if (!ctx) return set_err(LA_EINVAL, "null context");
    if (ctx->poisoned) return set_err(LA_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    if (!ctx->loaded) return set_err(LA_ESTATE, "nets not loaded");
    return LA_OK;
}

// This rank's share of batch k: contiguous ranges of the batch's big and small
// nets (role-list indices; their forest positions are contiguous as well).
struct RankShare { int64_t big_beg, big_end, small_beg, small_end; };
static RankShare rank_share(const la_ctx *ctx, int32_t batch) {
    RankShare r;
    int64_t s0, s1;
    const int64_t g0 = ctx->batch_big0[batch], g1 = ctx->batch_big0[batch + 1];
    la_shard_range(g1 - g0, ctx->world, ctx->rank, &s0, &s1);
    r.big_beg = g0 + s0;
    r.big_end = g0 + s1;
    const int64_t m0 = ctx->batch_small0[batch], m1 = ctx->batch_small0[batch + 1];
    la_shard_range(m1 - m0, ctx->world, ctx->rank, &s0, &s1);
    r.small_beg = m0 + s0;
    r.small_end = m0 + s1;
    return r;
}

// Grid of one launch: the big-role CTAs it needs, then the small-role CTAs.  *thr selects the
// kernel variant: a launch of many nets per resident warp runs the 7-CTA/SM build, one bound by
// its slowest net (and every dataflow launch) the 6-CTA/SM build.
static int launch_grid(const la_ctx *ctx, AssignLaunch &al, bool *thr) {
    const int64_t nbig = al.big_end - al.big_beg, nsmall = al.small_end - al.small_beg;
    const bool busy = nbig + nsmall > (int64_t)4 * ctx->grid * ASSIGN_WARPS;
    // big nets by half-CTAs when the launch is throughput-bound, by whole CTAs (lower latency
    // per big net) when it is bound by its slowest net
    al.big_split = ctx->big_split >= 0 ? ctx->big_split : (busy ? 1 : 0);
    const bool wide = nbig + nsmall > (int64_t)ctx->thr_nets_per_warp * ctx->grid * ASSIGN_WARPS;   // DESIGN §5 v11
    *thr = !al.wait && (ctx->assign_variant >= 0 ? ctx->assign_variant == 1 : wide);
    const int gmax = *thr ? ctx->grid_thr : ctx->grid;
    const int npc = assign_nets_per_cta();
    if (!al.wait && ctx->hybrid) {   // batch mode: every CTA takes the batch's big nets first
        al.hybrid = 1;
        al.n_big_ctas = 0;
        return (int)std::min<int64_t>(gmax, std::max<int64_t>(nbig, (nsmall + npc - 1) / npc));
    }
    al.hybrid = 0;
    const int32_t nbc = al.wait ? ctx->n_big_ctas_flow : ctx->n_big_ctas;
    al.n_big_ctas = (int32_t)std::min<int64_t>(nbc, nbig);
    const int64_t small_ctas = std::min<int64_t>(gmax - nbc, (nsmall + npc - 1) / npc);
    return al.n_big_ctas + (int)small_ctas;
}

// Grid of one k_assign_g launch: enough CTAs for the big nets and the jobs (four warps per CTA),
// at most the resident grid of the variant; the 7-CTA/SM variant for launches of many jobs per
// resident warp (GAPLA_THR_JOBS_PER_WARP, default 4), the 6-CTA/SM one for tail-bound launches.
static int launch_grid_g(const la_ctx *ctx, AssignLaunch &al, bool *thr) {
    const int64_t nbig = al.big_end - al.big_beg, njobs = al.job_end - al.job_beg;
    const bool busy = nbig + njobs > (int64_t)4 * ctx->grid_g * ASSIGN_WARPS;
    al.big_split = ctx->big_split >= 0 ? ctx->big_split : (busy ? 1 : 0);
    int64_t per_warp = 4;
    if (const char *e = getenv("GAPLA_THR_JOBS_PER_WARP")) per_warp = std::max(1, atoi(e));
    const bool wide = nbig + njobs > per_warp * ctx->grid_g * ASSIGN_WARPS;
    *thr = ctx->assign_variant >= 0 ? ctx->assign_variant == 1 : wide;
    const int gmax = *thr ? ctx->grid_g_thr : ctx->grid_g;
    al.hybrid = 1;
    al.n_big_ctas = 0;
    return (int)std::min<int64_t>(gmax, std::max<int64_t>(nbig, (njobs + ASSIGN_WARPS - 1) / ASSIGN_WARPS));
}

static AssignLaunch assign_launch(const la_ctx *ctx) {
    AssignLaunch al{};
    al.big_pos = ctx->d_big_pos;
    al.small_pos = ctx->d_small_pos;
    al.gscratch = ctx->d_gscratch;
    al.gslot_bytes = ctx->gslot_bytes;
    al.glock = ctx->d_glock;
    al.n_gslots = ctx->n_gslots;
    al.jobs = ctx->d_jobs;
    al.warp_arena = ctx->warp_arena;
    al.NS = ctx->NS;
    al.NP = ctx->NP;
    al.LD = ctx->LD;
    al.commit = ctx->fuse_commit ? 1 : 0;   // this rank's nets commit inside k_assign (any world)
    al.trace = ctx->tracing ? ctx->d_trace : nullptr;
    return al;
}

la_status la_assign_batch(la_ctx *ctx, int32_t batch) {
    TRY(check_ready(ctx));
    const int32_t nb = (int32_t)ctx->batch_net0.size() - 1;
    if (batch < 0 || batch >= nb) return set_err(LA_ERANGE, "batch index out of range");
    if (ctx->pending_commit || batch != ctx->next_batch)
        return set_err(LA_ESTATE, "batches must be assigned in order, each committed before the next");
    const int64_t b0 = ctx->batch_net0[batch], b1 = ctx->batch_net0[batch + 1];
    if (ctx->world > 1 || ctx->nccl)   // other ranks' net costs arrive through the reconcile sum
        CK(cudaMemsetAsync(ctx->S.froot + b0, 0, sizeof(double) * (b1 - b0), ctx->stream));
    ctx->sol_valid = false;
    AssignLaunch al = assign_launch(ctx);
    const RankShare r = rank_share(ctx, batch);
    al.big_beg = r.big_beg; al.big_end = r.big_end; al.small_beg = r.small_beg; al.small_end = r.small_end;
    al.ticket = ctx->d_ticket + 2 * (1 + batch);
    bool thr = false;
    int grid = 0;
    int pi = prof_begin(ctx, K_ASSIGN);
    if (ctx->group_path) {
        al.job_beg = ctx->batch_job0[batch];
        al.job_end = ctx->batch_job0[batch + 1];
        grid = launch_grid_g(ctx, al, &thr);
        CK(launch_assign_g(ctx->G, ctx->F, ctx->S, al, grid, thr, ctx->stream));
    } else {
        grid = launch_grid(ctx, al, &thr);
        CK(launch_assign(ctx->G, ctx->F, ctx->S, al, grid, thr, ctx->stream));
    }
    prof_end(ctx, pi);
    if (grid > 0) ctx->stats.launches += 1;
    ctx->pending_commit = true;
    return LA_OK;
}

// This rank's packed decisions for batch k in S.dec (its shard's nodes; every other slot 0).
static la_status pack_shard(la_ctx *ctx, int32_t batch) {
    const int64_t b0 = ctx->batch_net0[batch], b1 = ctx->batch_net0[batch + 1];
    const int64_t n0 = ctx->h_net_node0[b0], n1 = ctx->h_net_node0[b1];
    const RankShare r = rank_share(ctx, batch);
    CK(cudaMemsetAsync(ctx->S.dec + n0, 0, sizeof(uint32_t) * (n1 - n0), ctx->stream));
    // the shard's big nets and small nets are two contiguous position ranges
    const int64_t ranges[2][2] = {{r.big_beg, r.big_end}, {r.small_beg, r.small_end}};
    for (int k = 0; k < 2; k++) {
        if (ranges[k][1] <= ranges[k][0]) continue;
        const int64_t p0 = k == 0 ? ctx->h_big_pos[ranges[k][0]] : ctx->h_small_pos[ranges[k][0]];
        const int64_t p1 = (k == 0 ? ctx->h_big_pos[ranges[k][1] - 1] : ctx->h_small_pos[ranges[k][1] - 1]) + 1;
        CK(launch_pack_decisions(ctx->S, ctx->h_net_node0[p0], ctx->h_net_node0[p1], ctx->stream));
        ctx->stats.launches += 1;
    }
    return LA_OK;
}

la_status la_batch_extent(la_ctx *ctx, int32_t batch, int64_t *nodes, int64_t *nets) {
    TRY(check_ready(ctx));
    const int32_t nb = (int32_t)ctx->batch_net0.size() - 1;
    if (batch < 0 || batch >= nb) return set_err(LA_ERANGE, "batch index out of range");
    const int64_t b0 = ctx->batch_net0[batch], b1 = ctx->batch_net0[batch + 1];
    if (nodes) *nodes = ctx->h_net_node0[b1] - ctx->h_net_node0[b0];
    if (nets) *nets = b1 - b0;
    return LA_OK;
}

la_status la_get_decisions(la_ctx *ctx, int32_t batch, uint32_t *dec, double *net_cost) {
    TRY(check_ready(ctx));
    if (!ctx->host_xport) return set_err(LA_ESTATE, "not a host-transport context (world > 1, nccl_id NULL)");
    if (!ctx->pending_commit || batch != ctx->next_batch) return set_err(LA_ESTATE, "batch not just assigned");
    if (!dec || !net_cost) return set_err(LA_EINVAL, "null argument");
    const int64_t b0 = ctx->batch_net0[batch], b1 = ctx->batch_net0[batch + 1];
    const int64_t n0 = ctx->h_net_node0[b0], n1 = ctx->h_net_node0[b1];
    TRY(pack_shard(ctx, batch));
    CK(cudaMemcpyAsync(dec, ctx->S.dec + n0, sizeof(uint32_t) * (n1 - n0), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(net_cost, ctx->S.froot + b0, sizeof(double) * (b1 - b0), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stats.d2h_bytes += 4 * (n1 - n0) + 8 * (b1 - b0);
    return LA_OK;
}

la_status la_put_decisions(la_ctx *ctx, int32_t batch, const uint32_t *dec, const double *net_cost) {
    TRY(check_ready(ctx));
    if (!ctx->host_xport) return set_err(LA_ESTATE, "not a host-transport context (world > 1, nccl_id NULL)");
    if (!ctx->pending_commit || batch != ctx->next_batch) return set_err(LA_ESTATE, "batch not just assigned");
    if (!dec || !net_cost) return set_err(LA_EINVAL, "null argument");
    const int64_t b0 = ctx->batch_net0[batch], b1 = ctx->batch_net0[batch + 1];
    const int64_t n0 = ctx->h_net_node0[b0], n1 = ctx->h_net_node0[b1];
    CK(cudaMemcpyAsync(ctx->S.dec + n0, dec, sizeof(uint32_t) * (n1 - n0), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->S.froot + b0, net_cost, sizeof(double) * (b1 - b0), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stats.h2d_bytes += 4 * (n1 - n0) + 8 * (b1 - b0);
    ctx->put_batch = batch;
    return LA_OK;
}

la_status la_commit_demand(la_ctx *ctx, int32_t batch) {
    TRY(check_ready(ctx));
    if (!ctx->pending_commit || batch != ctx->next_batch)
        return set_err(LA_ESTATE, "commit must follow the assignment of the same batch");
    ctx->sol_valid = false;
    const int64_t b0 = ctx->batch_net0[batch], b1 = ctx->batch_net0[batch + 1];
    const int64_t n0 = ctx->h_net_node0[b0], n1 = ctx->h_net_node0[b1];
    if (ctx->host_xport) {
        // the caller summed every rank's packed decisions and net costs (la_put_decisions)
        if (ctx->put_batch != batch) return set_err(LA_ESTATE, "host transport: la_put_decisions must precede the commit");
        CK(launch_unpack_decisions(ctx->S, n0, n1, ctx->stream));
        ctx->stats.launches += 1;
    } else if (ctx->nccl) {
        // reconcile: every rank contributes its shard's packed decisions (others 0) -> sum
        int pr = prof_begin(ctx, K_RECONCILE);
        TRY(pack_shard(ctx, batch));
        NK(ncclAllReduce(ctx->S.dec + n0, ctx->S.dec + n0, (size_t)(n1 - n0), ncclUint32, ncclSum, ctx->comm,
                         ctx->stream));
        NK(ncclAllReduce(ctx->S.froot + b0, ctx->S.froot + b0, (size_t)(b1 - b0), ncclFloat64, ncclSum, ctx->comm,
                         ctx->stream));
        CK(launch_unpack_decisions(ctx->S, n0, n1, ctx->stream));
        prof_end(ctx, pr);
        ctx->stats.launches += 2;
    }
    // demand: this rank's nets were committed inside k_assign (fuse_commit); replay the others'
    // decisions (integer adds: every replica ends identical).  Snapshot batches commit everything here.
    std::vector<std::pair<int64_t, int64_t>> todo;
    if (!ctx->fuse_commit) {
        todo.push_back({n0, n1});
    } else if (ctx->world > 1) {
        const RankShare r = rank_share(ctx, batch);
        auto first_node = [&](bool big, int64_t i, int64_t end) {   // node of list entry i, or of the list's end
            const std::vector<int32_t> &lst = big ? ctx->h_big_pos : ctx->h_small_pos;
            return i < end ? ctx->h_net_node0[lst[i]] : -1;
        };
        // the batch's positions: its big shards (rank 0..), then its small shards; own = two ranges
        const int64_t ob0 = r.big_end > r.big_beg ? first_node(true, r.big_beg, r.big_end) : -1;
        const int64_t ob1 = r.big_end > r.big_beg ? ctx->h_net_node0[ctx->h_big_pos[r.big_end - 1] + 1] : -1;
        const int64_t os0 = r.small_end > r.small_beg ? first_node(false, r.small_beg, r.small_end) : -1;
        const int64_t os1 = r.small_end > r.small_beg ? ctx->h_net_node0[ctx->h_small_pos[r.small_end - 1] + 1] : -1;
        int64_t cur = n0;
        for (auto own : {std::make_pair(ob0, ob1), std::make_pair(os0, os1)}) {
            if (own.first < 0) continue;
            if (own.first > cur) todo.push_back({cur, own.first});
            cur = own.second;
        }
        if (n1 > cur) todo.push_back({cur, n1});
    }
    if (!todo.empty()) {
        int pc = prof_begin(ctx, K_COMMIT);
        for (auto &t : todo) {
            CK(launch_commit(ctx->G, ctx->F, ctx->S, t.first, t.second, ctx->stream));
            ctx->stats.launches += 1;
        }
        prof_end(ctx, pc);
    }
    ctx->pending_commit = false;
    ctx->next_batch = batch + 1;
    return LA_OK;
}

// Packed k_assign records of the nets at forest positions `pos` (+ one dummy: never empty).
static std::vector<int4> pack_nets(const la_ctx *ctx, const std::vector<int32_t> &pos) {
    std::vector<int4> v(pos.size() + 1, int4{0, 0, 0, 0});
    const unsigned nthr = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    par_for((int64_t)pos.size(), nthr, [&](int64_t i) {
        const int64_t p = pos[i];
        const int64_t n0 = ctx->h_net_node0[p], nn = ctx->h_net_node0[p + 1] - n0;
        const int64_t q0 = ctx->h_net_sink0[p], ns = ctx->h_net_sink0[p + 1] - q0;
        v[i] = int4{(int)p, (int)n0, (int)(nn | (ns << 16)), (int)q0};
    });
    return v;
}

// Dataflow priority lists, built on the first dataflow run: nets are taken
// in descending weighted bottom level (longest chain of dependent work still ahead of the
// net; weight ~ its latency), ties by position.  Bottom levels strictly decrease along DAG
// edges, so the order is topological; critical chains start first.
static la_status build_flow_lists(la_ctx *ctx) {
    if (ctx->d_flow_big_pos) return LA_OK;
    const int64_t N = ctx->n_nets;
    std::vector<int64_t> off(N + 1, 0);
    if (N) CK(cudaMemcpyAsync(off.data(), ctx->d_succ_off, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost,
                              ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<int32_t> succ((size_t)std::max<int64_t>(off[N], 1));
    if (off[N])
        CK(cudaMemcpyAsync(succ.data(), ctx->d_succ, sizeof(int32_t) * off[N], cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    // the dataflow kernel's own roles: big = more than NS nodes or NP sinks (its warp slot)
    std::vector<uint8_t> big(N, 0);
    std::vector<int32_t> fb, fs;
    for (int64_t p = 0; p < N; p++) {
        big[p] = (ctx->h_net_node0[p + 1] - ctx->h_net_node0[p] > ctx->NS ||
                  ctx->h_net_sink0[p + 1] - ctx->h_net_sink0[p] > ctx->NP) ? 1 : 0;
        (big[p] ? fb : fs).push_back((int32_t)p);
    }
    ctx->n_flow_big = (int64_t)fb.size();
    ctx->n_flow_small = (int64_t)fs.size();
    {   // big-net CTAs of the dataflow launch: one per SM by default (GAPLA_BIG_CTAS overrides)
        int n_sm = 0;
        CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, ctx->device));
        ctx->n_big_ctas_flow = fb.empty() ? 0 : n_sm;
        if (const char *e = getenv("GAPLA_BIG_CTAS")) ctx->n_big_ctas_flow = std::max(0, atoi(e));
        if (!fb.empty()) ctx->n_big_ctas_flow = std::max(1, std::min(ctx->n_big_ctas_flow, ctx->grid - 1));
    }
    std::vector<int64_t> bl(N);
    for (int64_t p = N - 1; p >= 0; p--) {
        const int64_t nn = ctx->h_net_node0[p + 1] - ctx->h_net_node0[p];
        int64_t m = 0;
        for (int64_t e = off[p]; e < off[p + 1]; e++) m = std::max(m, bl[succ[e]]);   // succ positions > p
        bl[p] = m + 8 + (big[p] ? nn / 4 : nn);
    }
    auto by_prio = [&](int32_t a, int32_t c) { return bl[a] != bl[c] ? bl[a] > bl[c] : a < c; };
    const unsigned nthr = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    par_sort(fb, by_prio, nthr);
    par_sort(fs, by_prio, nthr);
    const std::vector<int4> ib = pack_nets(ctx, fb), is = pack_nets(ctx, fs);
    TRY(dev_upload(ctx, &ctx->d_flow_big_pos, ib.data(), ib.size()));
    TRY(dev_upload(ctx, &ctx->d_flow_small_pos, is.data(), is.size()));
    CK(cudaStreamSynchronize(ctx->stream));
    return LA_OK;
}

la_status la_assign_all(la_ctx *ctx) {
    TRY(check_ready(ctx));
    const int32_t nb = (int32_t)ctx->batch_net0.size() - 1;
    // automatic schedule: one dataflow launch when the whole design fits in one wave
    // of resident warps (latency-bound), batch by batch otherwise (throughput-bound)
    const int32_t sched = ctx->schedule >= 0 ? ctx->schedule
                        : (ctx->n_nets <= (int64_t)ctx->grid * ASSIGN_WARPS ? LA_SCHED_DATAFLOW : LA_SCHED_BATCH);
    if (ctx->world == 1 && !ctx->nccl && ctx->fuse_commit && sched == LA_SCHED_DATAFLOW && !ctx->pending_commit &&
        ctx->next_batch == 0 && !ctx->flow_dirty) {
        // one persistent launch over every net, in bottom-level priority order
        TRY(build_flow_lists(ctx));
        ctx->sol_valid = false;
        AssignLaunch al = assign_launch(ctx);
        al.big_pos = ctx->d_flow_big_pos;
        al.small_pos = ctx->d_flow_small_pos;
        al.big_beg = 0;
        al.big_end = ctx->n_flow_big;
        al.small_beg = 0;
        al.small_end = ctx->n_flow_small;
        al.ticket = ctx->d_ticket;
        al.wait = ctx->d_wait;
        al.succ_off = ctx->d_succ_off;
        al.succ = ctx->d_succ;
        bool thr = false;
        const int grid = launch_grid(ctx, al, &thr);
        int pi = prof_begin(ctx, K_ASSIGN);
        CK(launch_assign(ctx->G, ctx->F, ctx->S, al, grid, thr, ctx->stream));
        prof_end(ctx, pi);
        if (grid > 0) ctx->stats.launches += 1;
        ctx->flow_dirty = true;
        ctx->next_batch = nb;
        return LA_OK;
    }
    for (int32_t b = ctx->next_batch; b < nb; b++) {
        if (!ctx->pending_commit) TRY(la_assign_batch(ctx, b));
        TRY(la_commit_demand(ctx, b));
    }
    return LA_OK;
}

la_status la_paper_batches(la_ctx *ctx, const la_net_desc *n, const int32_t *criticality, double alpha, int32_t th,
                           int64_t max_batch, int32_t *batch_of, int32_t *n_batches) {
    if (!ctx) return set_err(LA_EINVAL, "null context");
    if (ctx->poisoned) return set_err(LA_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    if (!n || !criticality || !batch_of || !n_batches) return set_err(LA_EINVAL, "null argument");
    if (!(alpha > 0.0) || max_batch < 1 || th < 0) return set_err(LA_EINVAL, "alpha must be > 0, th >= 0, max_batch >= 1");
    const int64_t N = n->n_nets;
    if (N < 0 || N >= ((int64_t)1 << 31)) return set_err(LA_EINVAL, "net count out of range");
    if (N > 0 && (!n->pin_ptr || !n->pin_slack || !n->seg_ptr || !n->seg_xy)) return set_err(LA_EINVAL, "bad net descriptor");
    for (int64_t j = 0; j < N; j++)
        if (criticality[j] < 0) return set_err(LA_EINVAL, "negative criticality");
    *n_batches = 0;
    if (N == 0) return LA_OK;
    const int64_t NP = n->pin_ptr[N], NSG = n->seg_ptr[N];
    CK(cudaSetDevice(ctx->device));
    // inputs to the device (freed on return: this call keeps no state in the context)
    int64_t *d_pp = nullptr, *d_sp = nullptr;
    double *d_sl = nullptr;
    int32_t *d_xy = nullptr, *d_cr = nullptr, *d_out = nullptr;
    auto release = [&] { for (void *p : {(void *)d_pp, (void *)d_sp, (void *)d_sl, (void *)d_xy, (void *)d_cr, (void *)d_out}) dfree(p); };
    cudaError_t e = cudaSuccess;
    do {
        if ((e = dmalloc(&d_pp, 8 * (N + 1))) || (e = dmalloc(&d_sp, 8 * (N + 1))) || (e = dmalloc(&d_sl, 8 * NP)) ||
            (e = dmalloc(&d_xy, 16 * NSG)) || (e = dmalloc(&d_cr, 4 * N)) || (e = dmalloc(&d_out, 4 * N)))
            break;
        const int pe = prof_begin(ctx, K_ORDER);
        if ((e = copy_many({{d_pp, n->pin_ptr, 8 * (size_t)(N + 1)}, {d_sp, n->seg_ptr, 8 * (size_t)(N + 1)},
                            {d_sl, n->pin_slack, 8 * (size_t)NP}, {d_xy, n->seg_xy, 16 * (size_t)NSG},
                            {d_cr, criticality, 4 * (size_t)N}}, ctx->device, cudaMemcpyHostToDevice)))
            break;
        ctx->stats.h2d_bytes += 16 * (N + 1) + 8 * NP + 16 * NSG + 4 * N;
        const int pk = prof_begin(ctx, K_ORDER_KERNELS);
        OrderIn in{N, d_pp, d_sp, d_sl, d_xy, d_cr, n->wns, alpha, th, max_batch};
        int32_t nb = 0;
        if ((e = gpu_paper_batches(in, d_out, &nb, ctx->stream, &ctx->stats.launches))) break;
        prof_end(ctx, pk);
        if ((e = cudaMemcpyAsync(batch_of, d_out, 4 * N, cudaMemcpyDeviceToHost, ctx->stream))) break;
        prof_end(ctx, pe);
        if ((e = cudaStreamSynchronize(ctx->stream))) break;
        ctx->stats.d2h_bytes += 4 * N;
        *n_batches = nb;
    } while (0);
    release();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "la_paper_batches");
    return LA_OK;
}

// Chunks of the tree passes (la_tree.cu): consecutive forest positions packed into runs of at
// most CHUNK_NODES nodes / CHUNK_SINKS sinks / 32 nets; a net beyond that is a chunk of its own.
// pos: the positions to cover, ascending (nullptr: all); a chunk never spans a gap.
static la_status build_chunks(la_ctx *ctx, const std::vector<int32_t> *pos, int4 **d_out, int64_t *n_out) {
    if (*d_out) return LA_OK;
    const int64_t M = pos ? (int64_t)pos->size() : ctx->n_nets;
    auto P = [&](int64_t i) -> int64_t { return pos ? (int64_t)(*pos)[i] : i; };
    std::vector<int4> ch;
    ch.reserve((size_t)(M / 6 + 16));
    int64_t i = 0;
    while (i < M) {
        const int64_t p0 = P(i);
        const int64_t n0 = ctx->h_net_node0[p0], q0 = ctx->h_net_sink0[p0];
        int64_t nodes = 0, sinks = 0, k = 0;
        while (i + k < M && k < 32 && P(i + k) == p0 + k) {
            const int64_t p = p0 + k;
            const int64_t a = ctx->h_net_node0[p + 1] - ctx->h_net_node0[p];
            const int64_t b = ctx->h_net_sink0[p + 1] - ctx->h_net_sink0[p];
            if (nodes + a > CHUNK_NODES || sinks + b > CHUNK_SINKS) break;
            nodes += a;
            sinks += b;
            k++;
        }
        if (k == 0) {   // one bigger net
            k = 1;
            ch.push_back(make_int4((int)p0, (int)n0, (int)q0, (int)(1u << 31)));
        } else {
            ch.push_back(make_int4((int)p0, (int)n0, (int)q0, (int)(k | (sinks << 6) | (nodes << 13))));
        }
        i += k;
    }
    *n_out = (int64_t)ch.size();
    TRY(dev_upload(ctx, d_out, ch.data(), std::max<size_t>(ch.size(), 1)));
    return LA_OK;
}

la_status la_pre_timing(la_ctx *ctx, double r_h, double r_v, double c_h, double c_v, double *sink_delay,
                        double *net_cap) {
    TRY(check_ready(ctx));
    if (!(std::isnan(r_h) || r_h >= 0) || !(std::isnan(r_v) || r_v >= 0) || !(std::isnan(c_h) || c_h >= 0) ||
        !(std::isnan(c_v) || c_v >= 0))
        return set_err(LA_EINVAL, "negative unit R / C");
    CK(cudaSetDevice(ctx->device));
    TRY(build_chunks(ctx, nullptr, &ctx->d_chunks, &ctx->n_chunks));
    // per-direction averages over the routable layers (R44): plain mean, ascending l
    PreRC P{};
    const double give_r[2] = {r_h, r_v}, give_c[2] = {c_h, c_v};
    for (int t = 0; t < 2; t++) {
        double sr = 0.0, sc = 0.0;
        int cnt = 0;
        for (int l = 0; l < ctx->L; l++)
            if (ctx->routable[l] && ctx->dir[l] == t) { sr = sr + ctx->r[l]; sc = sc + ctx->c[l]; cnt++; }
        P.rd[t] = std::isnan(give_r[t]) ? (cnt ? sr / (double)cnt : 0.0) : give_r[t];
        P.cd[t] = std::isnan(give_c[t]) ? (cnt ? sc / (double)cnt : 0.0) : give_c[t];
    }
    if (ctx->n_pins) CK(cudaMemsetAsync(ctx->S.sink_delay, 0, sizeof(double) * ctx->n_pins, ctx->stream));
    const int pe = prof_begin(ctx, K_PRETIME);
    CK(launch_pre_timing(ctx->F, ctx->d_chunks, ctx->n_chunks, P, ctx->S.Cd, ctx->S.Tin, ctx->S.sink_delay,
                         ctx->S.net_cap, ctx->stream));
    prof_end(ctx, pe);
    ctx->stats.launches += 1;
    if (sink_delay && ctx->n_pins)
        CK(cudaMemcpyAsync(sink_delay, ctx->S.sink_delay, sizeof(double) * ctx->n_pins, cudaMemcpyDeviceToHost, ctx->stream));
    if (net_cap && ctx->n_nets)
        CK(cudaMemcpyAsync(net_cap, ctx->S.net_cap, sizeof(double) * ctx->n_nets, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stats.d2h_bytes += (sink_delay ? 8 * ctx->n_pins : 0) + (net_cap ? 8 * ctx->n_nets : 0);
    return LA_OK;
}

la_status la_set_schedule(la_ctx *ctx, int32_t schedule) {
    if (!ctx) return set_err(LA_EINVAL, "null context");
    if (schedule != LA_SCHED_DATAFLOW && schedule != LA_SCHED_BATCH) return set_err(LA_EINVAL, "unknown schedule");
    if (!ctx->snap_batch.empty() && schedule == LA_SCHED_DATAFLOW)
        return set_err(LA_EINVAL, "snapshot batches run batch by batch (no dataflow schedule)");
    ctx->schedule = schedule;
    return LA_OK;
}

la_status la_set_snapshot_batches(la_ctx *ctx, const int32_t *batch_of, int64_t n_nets) {
    if (!ctx) return set_err(LA_EINVAL, "null context");
    if (ctx->loaded) return set_err(LA_ESTATE, "snapshot batches must be set before la_load_nets");
    if (!batch_of) {
        ctx->snap_batch.clear();
        return LA_OK;
    }
    if (n_nets < 0) return set_err(LA_EINVAL, "negative net count");
    ctx->snap_batch.assign(batch_of, batch_of + n_nets);
    return LA_OK;
}

static la_status require_done(la_ctx *ctx) {
    TRY(check_ready(ctx));
    const int32_t nb = (int32_t)ctx->batch_net0.size() - 1;
    if (ctx->next_batch != nb || ctx->pending_commit) return set_err(LA_ESTATE, "not every batch is committed");
    return LA_OK;
}

la_status la_eval_timing(la_ctx *ctx, double *sink_delay, double *net_cap, double *net_rc) {
    TRY(require_done(ctx));
    const bool shard = ctx->world > 1;
    if (ctx->n_pins) CK(cudaMemsetAsync(ctx->S.sink_delay, 0, sizeof(double) * ctx->n_pins, ctx->stream));
    if (shard && ctx->n_nets) {   // other ranks' nets stay 0 here: the outputs are summed over ranks
        CK(cudaMemsetAsync(ctx->S.net_cap, 0, sizeof(double) * ctx->n_nets, ctx->stream));
        CK(cudaMemsetAsync(ctx->S.net_rc, 0, sizeof(double) * ctx->n_nets, ctx->stream));
    }
    static const bool v1 = getenv("GAPLA_ELMORE_V1") && atoi(getenv("GAPLA_ELMORE_V1")) != 0;   // A/B: round-1 kernel
    int pe = prof_begin(ctx, K_ELMORE);
    const int64_t ne = shard ? ctx->n_own : ctx->n_nets;
    const int32_t *lst = shard ? ctx->d_own_pos : nullptr;
    if (v1) CK(launch_elmore_v1(ctx->G, ctx->F, ctx->S, 0, ne, lst, ctx->stream));
    else CK(launch_elmore(ctx->F, ctx->S, ctx->d_tab, ctx->L, 0, ne, lst, ctx->stream));
    prof_end(ctx, pe);
    ctx->stats.launches += 1;
    if (ctx->nccl) {
        // allgather of disjoint outputs as one sum (every value has exactly one nonzero contributor)
        int pr = prof_begin(ctx, K_RECONCILE);
        if (ctx->n_pins)
            NK(ncclAllReduce(ctx->S.sink_delay, ctx->S.sink_delay, (size_t)ctx->n_pins, ncclFloat64, ncclSum, ctx->comm,
                             ctx->stream));
        if (ctx->n_nets) {
            NK(ncclAllReduce(ctx->S.net_cap, ctx->S.net_cap, (size_t)ctx->n_nets, ncclFloat64, ncclSum, ctx->comm,
                             ctx->stream));
            NK(ncclAllReduce(ctx->S.net_rc, ctx->S.net_rc, (size_t)ctx->n_nets, ncclFloat64, ncclSum, ctx->comm,
                             ctx->stream));
        }
        prof_end(ctx, pr);
    }
    CK(cudaStreamSynchronize(ctx->stream));
    {   // outputs to the caller's (pageable) buffers through the pinned pipeline
        std::vector<Xfer> xs;
        if (sink_delay && ctx->n_pins) xs.push_back({sink_delay, ctx->S.sink_delay, sizeof(double) * (size_t)ctx->n_pins});
        if (net_cap && ctx->n_nets) xs.push_back({net_cap, ctx->S.net_cap, sizeof(double) * (size_t)ctx->n_nets});
        if (net_rc && ctx->n_nets) xs.push_back({net_rc, ctx->S.net_rc, sizeof(double) * (size_t)ctx->n_nets});
        CK(copy_many(xs, ctx->device, cudaMemcpyDeviceToHost));
    }
    ctx->stats.d2h_bytes += (sink_delay ? 8 * ctx->n_pins : 0) + (net_cap ? 8 * ctx->n_nets : 0) +
                            (net_rc ? 8 * ctx->n_nets : 0);
    return LA_OK;
}

la_status la_get_solution(la_ctx *ctx, int64_t *n_wires, int64_t *n_vias, int64_t *wire_ptr, int32_t *wires,
                          int64_t *via_ptr, int32_t *vias, double *net_cost) {
    TRY(require_done(ctx));
    const int64_t N = ctx->n_nets, NN = ctx->n_nodes;
    const unsigned nthr = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const bool verbose = getenv("GAPLA_VERBOSE") != nullptr;   // phase times to stderr
    auto tph = std::chrono::steady_clock::now();
    auto phase = [&](const char *what) {
        if (!verbose) return;
        auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[gapla solution] %-24s %9.1f ms\n", what, std::chrono::duration<double, std::milli>(t - tph).count());
        tph = t;
    };
    // counts, offsets, costs and the rows on the GPU (la_solution.cu); the caller's buffers are
    // filled through the pinned pipeline
    if (!ctx->d_sol_w) return set_err(LA_ESTATE, "internal: solution buffers missing");   // allocated at load
    int64_t *wcnt = ctx->d_sol_w, *vcnt = wcnt + (N + 1), *wptr = vcnt + (N + 1), *vptr = wptr + (N + 1);
    if (!ctx->sol_valid) {
        CK(sol_count(ctx->F, ctx->S, wcnt, vcnt, wptr, vptr, ctx->d_sol_cost, ctx->d_sol_vc, ctx->d_sol_temp,
                     &ctx->sol_temp_bytes, ctx->stream));
        ctx->stats.launches += 3;
        int64_t tot[2] = {0, 0};
        unsigned long long vc = 0;
        CK(cudaMemcpyAsync(&tot[0], wptr + N, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&tot[1], vptr + N, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&vc, ctx->d_sol_vc, sizeof(vc), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->stats.d2h_bytes += 24;
        ctx->sol_nw_total = tot[0];
        ctx->sol_nv_total = tot[1];
        ctx->stats.via_cuts = (int64_t)vc;
        ctx->sol_valid = true;
        phase("counts (GPU)");
    }
    const int64_t NWt = ctx->sol_nw_total, NVt = ctx->sol_nv_total;
    if (n_wires) *n_wires = NWt;
    if (n_vias) *n_vias = NVt;
    std::vector<Xfer> xs;
    int32_t *d_rows = ctx->d_sol_rows;   // allocated at load: 5 (nodes - nets) + 4 nodes int32 >= the rows
    if (wires || vias) {
        cudaError_t e = sol_fill(ctx->F, ctx->S, wptr, vptr, d_rows, d_rows + 5 * NWt, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "la_get_solution: fill");
        ctx->stats.launches += 1;
        if (wires && NWt) xs.push_back({wires, d_rows, sizeof(int32_t) * 5 * (size_t)NWt});
        if (vias && NVt) xs.push_back({vias, d_rows + 5 * NWt, sizeof(int32_t) * 4 * (size_t)NVt});
        phase("rows (GPU)");
    }
    if (wire_ptr) xs.push_back({wire_ptr, wptr, sizeof(int64_t) * (size_t)(N + 1)});
    if (via_ptr) xs.push_back({via_ptr, vptr, sizeof(int64_t) * (size_t)(N + 1)});
    if (net_cost && N) xs.push_back({net_cost, ctx->d_sol_cost, sizeof(double) * (size_t)N});
    cudaError_t e = copy_many(xs, ctx->device, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "la_get_solution: copies");
    for (const Xfer &x : xs) ctx->stats.d2h_bytes += (int64_t)x.bytes;
    phase("to host");
    return LA_OK;
}

la_status la_get_demand(la_ctx *ctx, int32_t *wire_dem, int32_t *via_dem) {
    if (!ctx) return set_err(LA_EINVAL, "null context");
    if (ctx->poisoned) return set_err(LA_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    int32_t *dw = nullptr, *dv = nullptr;
    CK(dmalloc(&dw, sizeof(int32_t) * std::max<int64_t>(ctx->n_wire_api, 1)));
    cudaError_t e = dmalloc(&dv, sizeof(int32_t) * std::max<int64_t>(ctx->n_via_api, 1));
    if (e == cudaSuccess) e = launch_unpack_demand(ctx->G, ctx->d_wcap, ctx->d_vcap, dw, dv, ctx->d_wire_off, ctx->stream);
    if (e == cudaSuccess && wire_dem)
        e = cudaMemcpyAsync(wire_dem, dw, sizeof(int32_t) * ctx->n_wire_api, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && via_dem)
        e = cudaMemcpyAsync(via_dem, dv, sizeof(int32_t) * ctx->n_via_api, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e == cudaSuccess)
        ctx->stats.d2h_bytes += (wire_dem ? 4 * ctx->n_wire_api : 0) + (via_dem ? 4 * ctx->n_via_api : 0);
    dfree(dw);
    if (dv) dfree(dv);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "la_get_demand");
    return LA_OK;
}

la_status la_get_batches(la_ctx *ctx, int32_t *batch_of) {
    TRY(check_ready(ctx));
    if (batch_of) std::memcpy(batch_of, ctx->batch_of_net.data(), sizeof(int32_t) * ctx->n_nets);
    return LA_OK;
}

la_status la_reset(la_ctx *ctx) {
    TRY(check_ready(ctx));
    ctx->sol_valid = false;
    size_t bH = sizeof(int32_t) * (size_t)(ctx->X - 1) * ctx->Y * ctx->LH;
    size_t bV = sizeof(int32_t) * (size_t)ctx->X * (ctx->Y - 1) * ctx->LV;
    size_t bVia = sizeof(int32_t) * (size_t)ctx->n_via_api;
    CK(cudaMemcpyAsync(ctx->d_wH, ctx->d_wH0, bH, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_wV, ctx->d_wV0, bV, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_via, ctx->d_via0, bVia, cudaMemcpyDeviceToDevice, ctx->stream));
    const int32_t nb = (int32_t)ctx->batch_net0.size() - 1;
    CK(cudaMemsetAsync(ctx->d_ticket, 0, sizeof(unsigned long long) * 2 * (nb + 1), ctx->stream));
    if (ctx->n_nets)
        CK(cudaMemcpyAsync(ctx->d_wait, ctx->d_indeg, sizeof(int32_t) * ctx->n_nets, cudaMemcpyDeviceToDevice,
                           ctx->stream));
    ctx->flow_dirty = false;
    ctx->next_batch = 0;
    ctx->pending_commit = false;
    return LA_OK;
}

la_status la_get_stats(la_ctx *ctx, la_stats *out) {
    if (!ctx || !out) return set_err(LA_EINVAL, "null argument");
    *out = ctx->stats;
    return LA_OK;
}

la_status la_set_profiling(la_ctx *ctx, int32_t enable) {
    if (!ctx) return set_err(LA_EINVAL, "null context");
    ctx->prof = enable != 0;
    return LA_OK;
}

la_status la_get_profile(la_ctx *ctx, la_profile *out, int32_t reset) {
    if (!ctx || !out) return set_err(LA_EINVAL, "null argument");
    if (ctx->poisoned) return set_err(LA_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto &sp : ctx->spans) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, sp.a, sp.b));
        switch (sp.kind) {
            case K_ASSIGN: ctx->acc.assign_ms += ms; ctx->acc.assign_launches++; break;
            case K_COMMIT: ctx->acc.commit_ms += ms; ctx->acc.commit_launches++; break;
            case K_ELMORE: ctx->acc.elmore_ms += ms; ctx->acc.elmore_launches++; break;
            case K_EVAL: ctx->acc.eval_ms += ms; ctx->acc.eval_launches++; break;
            case K_PRETIME: ctx->acc.pretime_ms += ms; ctx->acc.pretime_launches++; break;
            case K_ORDER: ctx->acc.order_ms += ms; ctx->acc.order_calls++; break;
            case K_ORDER_KERNELS: ctx->acc.order_kernel_ms += ms; break;
            default: ctx->acc.reconcile_ms += ms; ctx->acc.reconcile_calls++; break;
        }
        ctx->ev_pool.push_back(sp.a);
        ctx->ev_pool.push_back(sp.b);
    }
    ctx->spans.clear();
    *out = ctx->acc;
    if (reset) ctx->acc = la_profile{};
    return LA_OK;
}

la_status la_eval_overflow(la_ctx *ctx, la_eval *out) {
    TRY(require_done(ctx));
    if (!out) return set_err(LA_EINVAL, "null argument");
    const int L = ctx->L, dlo = ctx->G.delta_lo, dhi = ctx->G.delta_hi, nbins = dhi - dlo + 1;
    const size_t nh = (size_t)MAXL * 2 * nbins;
    const size_t nwords = 2 * nh + 2 * MAXL + 1 + MAXL + 1;   // hist w, hist v, legacy w, legacy v, oob, wl, vcuts
    if (!ctx->d_eval) {
        CK(dmalloc(&ctx->d_eval, sizeof(unsigned long long) * nwords));
        int8_t lay[3][MAXL] = {};
        for (int l = 0; l < L; l++) lay[ctx->dir[l]][ctx->G.lidx[l]] = (int8_t)l;
        for (int k = 0; k < L - 1; k++) lay[2][k] = (int8_t)k;            // via cut k: ofw of its lower layer (R36)
        CK(dmalloc(&ctx->d_eval_lay, sizeof(lay)));
        CK(cudaMemcpyAsync(ctx->d_eval_lay, lay, sizeof(lay), cudaMemcpyHostToDevice, ctx->stream));
    }
    unsigned long long *b = ctx->d_eval;
    const int64_t nH = (int64_t)(ctx->X - 1) * ctx->Y * ctx->LH, nV = (int64_t)ctx->X * (ctx->Y - 1) * ctx->LV;
    // Per-layer wirelength and the via-cut count follow from the plane histograms: every committed
    // unit wire edge (via cut) adds 1 to one word, so on each layer Σ(d - c) grows by exactly its
    // wirelength.  Σ(d - c) of the initial state comes from one histogram pass over the pristine
    // planes, once per context; a value clamped to [δ_lo, δ_hi] (R20) in either pass makes the sums
    // inexact, and then the node pass (k_eval_nodes) counts them instead.
    auto plane_sums = [&](const unsigned long long *hh, int nlay, std::vector<long long> &sum) {
        sum.assign(MAXL, 0);
        for (int l = 0; l < nlay; l++)
            for (int f = 0; f < 2; f++)
                for (int i = 0; i < nbins; i++) sum[l] += (long long)hh[((size_t)l * 2 + f) * nbins + i] * (dlo + i);
    };
    if (!ctx->eval0_done) {
        CK(cudaMemsetAsync(b, 0, sizeof(unsigned long long) * nwords, ctx->stream));
        EvalDev E0{b, b + 2 * nh, b + 2 * nh + 2 * MAXL, b + 2 * nh + 2 * MAXL + 1, b + 2 * nh + 3 * MAXL + 1};
        EvalDev V0 = E0;
        V0.hist = b + nh;
        V0.legacy = b + 2 * nh + MAXL;
        CK(launch_eval_plane(ctx->d_wH0, nH, ctx->LH, ctx->d_eval_lay, E0, dlo, dhi, ctx->stream));
        CK(launch_eval_plane(ctx->d_wV0, nV, ctx->LV, ctx->d_eval_lay + MAXL, E0, dlo, dhi, ctx->stream));
        CK(launch_eval_plane(ctx->d_via0, ctx->n_via_api, L - 1, ctx->d_eval_lay + 2 * MAXL, V0, dlo, dhi, ctx->stream));
        std::vector<unsigned long long> h0(nwords);
        CK(cudaMemcpyAsync(h0.data(), b, sizeof(unsigned long long) * nwords, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        plane_sums(h0.data(), L, ctx->eval0_wire);
        plane_sums(h0.data() + nh, L - 1, ctx->eval0_via);
        ctx->eval0_oob = (int64_t)h0[2 * nh + 2 * MAXL];
        ctx->eval0_done = true;
    }
    CK(cudaMemsetAsync(b, 0, sizeof(unsigned long long) * nwords, ctx->stream));
    EvalDev Ew{b, b + 2 * nh, b + 2 * nh + 2 * MAXL, b + 2 * nh + 2 * MAXL + 1, b + 2 * nh + 3 * MAXL + 1};
    EvalDev Ev = Ew;
    Ev.hist = b + nh;
    Ev.legacy = b + 2 * nh + MAXL;
    int pe = prof_begin(ctx, K_EVAL);
    CK(launch_eval_plane(ctx->d_wH, nH, ctx->LH, ctx->d_eval_lay, Ew, dlo, dhi, ctx->stream));
    CK(launch_eval_plane(ctx->d_wV, nV, ctx->LV, ctx->d_eval_lay + MAXL, Ew, dlo, dhi, ctx->stream));
    CK(launch_eval_plane(ctx->d_via, ctx->n_via_api, L - 1, ctx->d_eval_lay + 2 * MAXL, Ev, dlo, dhi, ctx->stream));
    prof_end(ctx, pe);
    ctx->stats.launches += 3;
    std::vector<unsigned long long> h(nwords);
    CK(cudaMemcpyAsync(h.data(), b, sizeof(unsigned long long) * nwords, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stats.d2h_bytes += (int64_t)(8 * nwords);
    const bool from_planes = h[2 * nh + 2 * MAXL] == 0 && ctx->eval0_oob == 0;
    if (from_planes) {
        std::vector<long long> sw, sv;
        plane_sums(h.data(), L, sw);
        plane_sums(h.data() + nh, L - 1, sv);
        long long vc = 0;
        for (int l = 0; l < MAXL; l++) {
            h[2 * nh + 2 * MAXL + 1 + l] = (unsigned long long)(sw[l] - ctx->eval0_wire[l]);
            vc += sv[l] - ctx->eval0_via[l];
        }
        h[2 * nh + 3 * MAXL + 1] = (unsigned long long)vc;
    } else {   // a clamped value: count wirelength and via cuts from the nodes
        unsigned long long *nb = b + 2 * nh + 2 * MAXL + 1;
        CK(cudaMemsetAsync(nb, 0, sizeof(unsigned long long) * (MAXL + 1), ctx->stream));
        int pn = prof_begin(ctx, K_EVAL);
        CK(launch_eval_nodes(ctx->F, ctx->S, Ew, ctx->stream));
        prof_end(ctx, pn);
        ctx->stats.launches += 1;
        CK(cudaMemcpyAsync(h.data() + 2 * nh + 2 * MAXL + 1, nb, sizeof(unsigned long long) * (MAXL + 1),
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    // Eq. (3): per layer, bins in a fixed order (c > 0 then c == 0, d - c ascending), then layers ascending
    auto tof = [&](const unsigned long long *hist, int nlay) {
        double t = 0.0;
        for (int l = 0; l < nlay; l++) {
            double acc = 0.0;
            for (int f = 0; f < 2; f++) {
                const double sl = f ? ctx->s_zero : ctx->s_pos;
                for (int i = 0; i < nbins; i++) {
                    const unsigned long long c = hist[((size_t)l * 2 + f) * nbins + i];
                    if (c) acc = acc + (double)c * std::exp(sl * (double)(dlo + i));
                }
            }
            t = t + ctx->ofw[l] * acc;
        }
        return t;
    };
    la_eval r{};
    r.tof_wire = tof(h.data(), L);
    r.tof_via = tof(h.data() + nh, L - 1);
    for (int l = 0; l < MAXL; l++) {
        r.legacy_wire += (int64_t)h[2 * nh + l];
        r.legacy_via += (int64_t)h[2 * nh + MAXL + l];
        r.wirelength[l] = (int64_t)h[2 * nh + 2 * MAXL + 1 + l];
    }
    r.out_of_domain = (int64_t)h[2 * nh + 2 * MAXL];
    r.via_cuts = (int64_t)h[2 * nh + 3 * MAXL + 1];
    r.wire_cap = 0.0;
    for (int l = 0; l < L; l++) r.wire_cap = r.wire_cap + ctx->c[l] * (double)r.wirelength[l];
    *out = r;
    return LA_OK;
}

la_status la_set_tracing(la_ctx *ctx, int32_t enable) {
    TRY(check_ready(ctx));
    if (enable && !ctx->d_trace) {
        CK(dmalloc(&ctx->d_trace, sizeof(int64_t) * 5 * std::max<int64_t>(ctx->n_nets, 1)));
        CK(cudaMemsetAsync(ctx->d_trace, 0, sizeof(int64_t) * 5 * std::max<int64_t>(ctx->n_nets, 1), ctx->stream));
    }
    ctx->tracing = enable != 0;
    return LA_OK;
}

la_status la_get_trace(la_ctx *ctx, int64_t *out) {
    TRY(check_ready(ctx));
    if (!out) return set_err(LA_EINVAL, "null argument");
    if (!ctx->d_trace) return set_err(LA_ESTATE, "tracing was never enabled");
    std::vector<int64_t> t((size_t)5 * ctx->n_nets);
    CK(cudaMemcpyAsync(t.data(), ctx->d_trace, sizeof(int64_t) * t.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int64_t p = 0; p < ctx->n_nets; p++)
        for (int k = 0; k < 5; k++) out[ctx->h_net_id[p] * 5 + k] = t[p * 5 + k];
    return LA_OK;
}

la_status la_nccl_unique_id(void *out128) {
    if (!out128) return set_err(LA_EINVAL, "null argument");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return set_err(LA_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
    return LA_OK;
}

la_status la_fp64_peak(int32_t device, double *ops_per_s) {
    if (!ops_per_s) return set_err(LA_EINVAL, "null argument");
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = gapla::fp64_peak(ops_per_s);
    if (e != cudaSuccess) return set_err(LA_ECUDA, std::string("la_fp64_peak: ") + cudaGetErrorString(e));
    return LA_OK;
}

la_status la_sync(la_ctx *ctx) {
    if (!ctx) return set_err(LA_EINVAL, "null context");
    if (ctx->poisoned) return set_err(LA_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    CK(cudaStreamSynchronize(ctx->stream));
    return LA_OK;
}

void la_destroy(la_ctx *ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    delete ctx;
}

}  // extern "C"
