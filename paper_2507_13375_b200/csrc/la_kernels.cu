// Hand-written sm_100a kernels of the GAP-LA layer-assignment hot path.
//
//   k_pack_state / k_unpack_demand   a0: API-layout capacity/demand <-> packed planes
//   k_commit     (K8)                demand commit with int32 atomics (Alg. 2 input D, l.343);
//                                    used when the commit is not fused into k_assign (world > 1)
//   (k_assign, K4 + K5, lives in la_assign.cu)
//   k_elmore     (K6 + K7)           Elmore / downstream cap on the 3D RC trees (l.146, l.443-444)
//
// Bit-exactness contract: this translation unit is compiled with
// --fmad=false; every fp64 value is produced by the same expression tree, in the
// same operand order, as DESIGN §3 (O5, O6, O9) prescribes; no transcendental
// function runs on the device (Eq. (3) comes from host tables); cross-lane
// reductions are min/argmin only, with a total-order key.
#include <cuda_runtime.h>

#include <algorithm>

#include "la_device.cuh"
#include "la_internal.h"

namespace gapla {

namespace {

// ------------------------------------------------------------------ a0 ------
__global__ void k_pack_wire(DevGrid G, const int32_t *__restrict__ cap, const int32_t *__restrict__ dem,
                            const int64_t *__restrict__ wire_off, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int l = 0;
    while (i >= wire_off[l + 1]) l++;
    int64_t e = i - wire_off[l];
    int dtype = G.dir[l];
    int W = dtype == 0 ? G.X - 1 : G.X;
    int x = (int)(e % W), y = (int)(e / W);
    int32_t c = cap[i], d = dem ? dem[i] : 0;
    int32_t w = (int32_t)((uint32_t)(d - c) << 1) | (c == 0 ? 1 : 0);
    (dtype == 0 ? G.wH : G.wV)[wire_word(G, dtype, l, x, y)] = w;
}

__global__ void k_pack_via(DevGrid G, const int32_t *__restrict__ cap, const int32_t *__restrict__ dem, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // API index [(k*Y + y)*X + x]
    if (i >= n) return;
    int64_t XY = (int64_t)G.X * G.Y;
    int k = (int)(i / XY);
    int64_t g = i - k * XY;
    int32_t c = cap[i], d = dem ? dem[i] : 0;
    G.via[g * (G.L - 1) + k] = (int32_t)((uint32_t)(d - c) << 1) | (c == 0 ? 1 : 0);
}

__global__ void k_unpack_wire(DevGrid G, const int32_t *__restrict__ cap, int32_t *__restrict__ dem,
                              const int64_t *__restrict__ wire_off, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int l = 0;
    while (i >= wire_off[l + 1]) l++;
    int64_t e = i - wire_off[l];
    int dtype = G.dir[l];
    int W = dtype == 0 ? G.X - 1 : G.X;
    int x = (int)(e % W), y = (int)(e / W);
    int32_t w = (dtype == 0 ? G.wH : G.wV)[wire_word(G, dtype, l, x, y)];
    dem[i] = (w >> 1) + cap[i];
}

__global__ void k_unpack_via(DevGrid G, const int32_t *__restrict__ cap, int32_t *__restrict__ dem, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t XY = (int64_t)G.X * G.Y;
    int k = (int)(i / XY);
    int64_t g = i - k * XY;
    dem[i] = (G.via[g * (G.L - 1) + k] >> 1) + cap[i];
}

// ------------------------------------------------------------------ K8 ------
// +1 demand (packed +2) per unit edge of the node's parent run on its layer and
// per via cut of its stack.  Batches are conflict-free, so the
// atomics are uncontended; integer adds commute, so any order is exact.
__global__ void k_commit(DevGrid G, DevForest F, DevScratch S, int64_t node_beg, int64_t node_end) {
    int64_t n = node_beg + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= node_end) return;
    const uint32_t xy = F.xy[n];
    const int x = xy & 0xffff, y = xy >> 16;
    const uint8_t ed = F.edir[n];
    if (ed != NO_DIR) {
        const int l = S.lay[n], len = F.len[n];
        const int a = run_lo(ed, x, y, len);
        if (ed <= 1) {
            int32_t *wp = G.wH + ((int64_t)y * (G.X - 1) + a) * G.LH + G.lidx[l];
            for (int i = 0; i < len; ++i) red_add(wp + (int64_t)i * G.LH, 2);
        } else {
            int32_t *wp = G.wV + ((int64_t)x * (G.Y - 1) + a) * G.LV + G.lidx[l];
            for (int i = 0; i < len; ++i) red_add(wp + (int64_t)i * G.LV, 2);
        }
    }
    const int b = S.sb[n], t = S.st[n];
    int32_t *vp = G.via + ((int64_t)y * G.X + x) * (G.L - 1);
    for (int k = b; k < t; ++k) red_add(vp + k, 2);
}

__global__ void k_pack_dec(DevScratch S, int64_t node_beg, int64_t node_end) {
    int64_t n = node_beg + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= node_end) return;
    S.dec[n] = (uint32_t)S.lay[n] | ((uint32_t)S.sb[n] << 8) | ((uint32_t)S.st[n] << 16) | (1u << 24);
}

__global__ void k_unpack_dec(DevScratch S, int64_t node_beg, int64_t node_end) {
    int64_t n = node_beg + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= node_end) return;
    const uint32_t d = S.dec[n];
    S.lay[n] = (uint8_t)(d & 0xff);
    S.sb[n] = (uint8_t)((d >> 8) & 0xff);
    S.st[n] = (uint8_t)((d >> 16) & 0xff);
}

// ------------------------------------------------------------------ K6 + K7 --
// Canonical fast Elmore form (DESIGN §3 O9), one thread per net: the round-1 kernel, kept for
// A/B runs (GAPLA_ELMORE_V1=1); la_eval_timing runs the chunked k_elmore of la_tree.cu.
constexpr int ELMORE_THREADS = 128;

__global__ void __launch_bounds__(ELMORE_THREADS) k_elmore_v1(DevGrid G, DevForest F, DevScratch S, int64_t net_beg,
                                                          int64_t net_end, const int32_t *list) {
    __shared__ TechTab T;
    __shared__ double Tks[MAXL][ELMORE_THREADS];   // T(n, k) of the current node, one column per thread
    stage_tab(T, G.tab);
    __syncthreads();
    const int64_t idx = net_beg + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= net_end) return;
    const int64_t net = list ? (int64_t)list[idx] : idx;      // this rank's nets (multi-GPU) or all
    const int64_t n0 = F.net_node0[net], n1 = F.net_node0[net + 1];
    // bottom-up: Cdown(n) = C0 + ((Cw1 + Cd1) + ...); rc(n) = F0u + ((c1 + c2) + ...)
    for (int64_t n = n0; n < n1; ++n) {
        const int ln = S.lay[n];
        double C0 = 0.0, F0u = 0.0;
        const int q0 = F.sink0[n], qn = F.nsink[n];
        for (int q = q0; q < q0 + qn; ++q) {
            const double cq = F.p_cap[q];
            C0 = C0 + cq;
            F0u = F0u + cq * T.VR[F.p_layer[q] * MAXL + ln];
        }
        double K = 0.0, R = 0.0;
        const int nk = F.nkid[n];
        for (int i = 0; i < nk; ++i) {
            const int64_t s = F.kid[n * 4 + i];
            const int ls = S.lay[s], len = F.len[s];
            const double Cw = T.c[ls] * (double)len, Rw = T.r[ls] * (double)len;
            const double Cd = S.Cd[s];
            K = K + (Cw + Cd);
            R = R + ((S.rcv[s] + Rw * (0.5 * Cw + Cd)) + (Cw + Cd) * T.VR[ln * MAXL + ls]);
        }
        S.Cd[n] = C0 + K;
        S.rcv[n] = F0u + R;
    }
    const int64_t nid = F.net_id[net];
    S.net_cap[nid] = S.Cd[n1 - 1];
    S.net_rc[nid] = S.rcv[n1 - 1];
    // top-down: via stacks (C>= / C<= over the branches attached at each layer) and pi wires
    double *Tk = &Tks[0][threadIdx.x];               // Tk[k * ELMORE_THREADS]: no local-memory array
#define TK(k) Tk[(k) * ELMORE_THREADS]
    for (int64_t n = n1 - 1; n >= n0; --n) {
        const int ln = S.lay[n], b = S.sb[n], t = S.st[n];
        TK(ln) = (n == n1 - 1) ? 0.0 : S.Tin[n];
        const int q0 = F.sink0[n], qn = F.nsink[n], nk = F.nkid[n];
        // the node's branches, read once: sons (layer, Cw + Cdown, Rw, Cw, Cdown) and up to 4
        // sinks (layer, C_q) in registers; the C>= / C<= sums below keep the canonical order
        int lsk[MAXKIDS];
        double cbk[MAXKIDS], rwk[MAXKIDS], cwk[MAXKIDS], cdk[MAXKIDS];
        int64_t sk[MAXKIDS];
#pragma unroll
        for (int i = 0; i < MAXKIDS; ++i) {
            lsk[i] = 0; cbk[i] = rwk[i] = cwk[i] = cdk[i] = 0.0; sk[i] = 0;
            if (i < nk) {
                const int64_t s = F.kid[n * 4 + i];
                const int ls = S.lay[s], len = F.len[s];
                sk[i] = s;
                lsk[i] = ls;
                cwk[i] = T.c[ls] * (double)len;
                rwk[i] = T.r[ls] * (double)len;
                cdk[i] = S.Cd[s];
                cbk[i] = cwk[i] + cdk[i];
            }
        }
        const bool few = qn <= 4;
        int pl[4];
        double pc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pl[u] = 0; pc[u] = 0.0;
            if (few && u < qn) { pl[u] = F.p_layer[q0 + u]; pc[u] = F.p_cap[q0 + u]; }
        }
        // C>=(n, j) (up = true) or C<=(n, j): sinks in input order, then sons in child order
        auto branch_sum = [&](int j, bool up) {
            double acc = 0.0;
            if (few) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < qn && (up ? pl[u] >= j : pl[u] <= j)) acc = acc + pc[u];
            } else {
                for (int q = q0; q < q0 + qn; ++q) {
                    const int pq = F.p_layer[q];
                    if (up ? pq >= j : pq <= j) acc = acc + F.p_cap[q];
                }
            }
#pragma unroll
            for (int i = 0; i < MAXKIDS; ++i)
                if (i < nk && (up ? lsk[i] >= j : lsk[i] <= j)) acc = acc + cbk[i];
            return acc;
        };
        for (int k = ln; k < t; ++k) TK(k + 1) = TK(k) + T.vr[k] * branch_sum(k + 1, true);
        for (int k = ln; k > b; --k) TK(k - 1) = TK(k) + T.vr[k - 1] * branch_sum(k - 1, false);
        if (few) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (u < qn) S.sink_delay[F.p_orig[q0 + u]] = TK(pl[u]);
        } else {
            for (int q = q0; q < q0 + qn; ++q) S.sink_delay[F.p_orig[q]] = TK(F.p_layer[q]);
        }
#pragma unroll
        for (int i = 0; i < MAXKIDS; ++i)
            if (i < nk) S.Tin[sk[i]] = TK(lsk[i]) + rwk[i] * (0.5 * cwk[i] + cdk[i]);
    }
#undef TK
}

// ------------------------------------------------------------ forest layout --
// la_load_nets uploads the trees as the host threads built them (input-order chunks, net-local
// child ids and sink offsets) and this kernel lays them out batch-major: a warp per net, lanes
// over its nodes and sinks.  src holds the built arrays, F the destination (its pointers are
// const for the kernels that read it; they were allocated here, so the casts are sound).
__global__ void k_permute_forest(DevForest F, ForestSrc src, int64_t n_nets) {
    const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= n_nets) return;
    const int64_t d0 = F.net_node0[p], nn = F.net_node0[p + 1] - d0;
    const int64_t e0 = src.dst_sink0[p], ns = src.dst_sink0[p + 1] - e0;
    const int64_t s0 = src.src_node0[p], q0 = src.src_sink0[p];
    for (int64_t j = lane; j < nn; j += 32) {
        const int64_t d = d0 + j, s = s0 + j;
        const_cast<uint32_t *>(F.xy)[d] = src.xy[s];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t c = src.kid[s * 4 + k];
            const_cast<int32_t *>(F.kid)[d * 4 + k] = c < 0 ? -1 : (int32_t)(d0 + c);
        }
        const_cast<int32_t *>(F.len)[d] = src.len[s];
        const_cast<uint8_t *>(F.edir)[d] = src.edir[s];
        const_cast<uint8_t *>(F.nkid)[d] = src.nkid[s];
        const_cast<uint8_t *>(F.nl)[d] = src.nl[s];
        const_cast<uint8_t *>(F.nh)[d] = src.nh[s];
        const_cast<int32_t *>(F.sink0)[d] = (int32_t)(e0 + src.sink0[s]);
        const_cast<uint16_t *>(F.nsink)[d] = src.nsink[s];
        const_cast<double *>(F.wd)[d] = src.wd[s];
        const_cast<double *>(F.ur)[d] = src.ur[s];
        const_cast<uint16_t *>(F.height)[d] = src.height[s];
    }
    for (int64_t j = lane; j < ns; j += 32) {
        const int64_t d = e0 + j, q = q0 + j;
        const_cast<uint8_t *>(F.p_layer)[d] = src.p_layer[q];
        const_cast<double *>(F.p_cap)[d] = src.p_cap[q];
        const_cast<double *>(F.p_w)[d] = src.p_w[q];
        const_cast<int64_t *>(F.p_orig)[d] = src.p_orig[q];
    }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

cudaError_t launch_pack_state(const DevGrid &G, const int32_t *wcap, const int32_t *wdem, const int32_t *vcap,
                              const int32_t *vdem, const int64_t *wire_off, cudaStream_t s) {
    int64_t nw = (int64_t)(G.X - 1) * G.Y * G.LH + (int64_t)G.X * (G.Y - 1) * G.LV;
    int64_t nv = (int64_t)(G.L - 1) * G.X * G.Y;
    if (nw) k_pack_wire<<<nblk(nw, 256), 256, 0, s>>>(G, wcap, wdem, wire_off, nw);
    if (nv) k_pack_via<<<nblk(nv, 256), 256, 0, s>>>(G, vcap, vdem, nv);
    return cudaGetLastError();
}

cudaError_t launch_unpack_demand(const DevGrid &G, const int32_t *wcap, const int32_t *vcap, int32_t *wdem,
                                 int32_t *vdem, const int64_t *wire_off, cudaStream_t s) {
    int64_t nw = (int64_t)(G.X - 1) * G.Y * G.LH + (int64_t)G.X * (G.Y - 1) * G.LV;
    int64_t nv = (int64_t)(G.L - 1) * G.X * G.Y;
    if (nw && wdem) k_unpack_wire<<<nblk(nw, 256), 256, 0, s>>>(G, wcap, wdem, wire_off, nw);
    if (nv && vdem) k_unpack_via<<<nblk(nv, 256), 256, 0, s>>>(G, vcap, vdem, nv);
    return cudaGetLastError();
}

cudaError_t launch_commit(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t node_beg,
                          int64_t node_end, cudaStream_t s) {
    int64_t n = node_end - node_beg;
    if (n <= 0) return cudaSuccess;
    k_commit<<<nblk(n, 256), 256, 0, s>>>(G, F, S, node_beg, node_end);
    return cudaGetLastError();
}

cudaError_t launch_pack_decisions(const DevScratch &S, int64_t node_beg, int64_t node_end, cudaStream_t s) {
    int64_t n = node_end - node_beg;
    if (n <= 0) return cudaSuccess;
    k_pack_dec<<<nblk(n, 256), 256, 0, s>>>(S, node_beg, node_end);
    return cudaGetLastError();
}

cudaError_t launch_unpack_decisions(const DevScratch &S, int64_t node_beg, int64_t node_end, cudaStream_t s) {
    int64_t n = node_end - node_beg;
    if (n <= 0) return cudaSuccess;
    k_unpack_dec<<<nblk(n, 256), 256, 0, s>>>(S, node_beg, node_end);
    return cudaGetLastError();
}

cudaError_t launch_permute_forest(const DevForest &F, const ForestSrc &src, cudaStream_t s) {
    if (F.n_nets <= 0) return cudaSuccess;
    k_permute_forest<<<nblk(F.n_nets * 32, 256), 256, 0, s>>>(F, src, F.n_nets);
    return cudaGetLastError();
}

// FP64 pipe peak (la_fp64_peak): 8 independent DADD chains per thread; a lane DADD = 1 op.
__global__ void __launch_bounds__(256) k_fp64_peak(double *out, int iters, double step) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
        a0 = a0 + step; a1 = a1 + step; a2 = a2 + step; a3 = a3 + step;
        a4 = a4 + step; a5 = a5 + step; a6 = a6 + step; a7 = a7 + step;
    }
    const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == -1.0) out[0] = r;                       // keeps the chains live
}

cudaError_t fp64_peak(double *ops_per_s) {
    int dev = 0, n_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    double *d = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&d, 8);
    cudaEvent_t a = nullptr, b = nullptr;
    if (e == cudaSuccess) e = cudaEventCreate(&a);
    if (e == cudaSuccess) e = cudaEventCreate(&b);
    const int iters = 1 << 14, grid = n_sm * 8, threads = 256;
    float ms = 0.f;
    for (int rep = 0; rep < 3 && e == cudaSuccess; ++rep) {   // the last of three timed runs
        cudaEventRecord(a);
        k_fp64_peak<<<grid, threads>>>(d, iters, 1e-300);
        cudaEventRecord(b);
        e = cudaEventSynchronize(b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
    }
    if (e == cudaSuccess) *ops_per_s = (double)grid * threads * 8.0 * iters / (ms * 1e-3);
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    if (d) cudaFree(d);
    return e;
}

cudaError_t launch_elmore_v1(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t net_beg,
                             int64_t net_end, const int32_t *list, cudaStream_t s) {
    int64_t n = net_end - net_beg;
    if (n <= 0) return cudaSuccess;
    k_elmore_v1<<<nblk(n, ELMORE_THREADS), ELMORE_THREADS, 0, s>>>(G, F, S, net_beg, net_end, list);
    return cudaGetLastError();
}

}  // namespace gapla

// ------------------------------------------------------------------ evaluator
// k_eval_plane (PAPER Eq. (2)/(3) l.174-182): one pass over a packed
// demand plane (the element of slot s of group i is words[i * slots + s]).  Every word gives
// d - c (w >> 1) and the zero-capacity flag (w & 1); counts per (layer, flag, d - c) go to a
// shared-memory window of d - c (EV_COPIES copies, one per lane & 3, plain shared atomics), the
// rest straight to the global bins; max(0, d - c) is summed exactly per layer.  HBM-bound: 4 B per element,
// read once with 16-byte loads; grid = a multiple of the SM count.
namespace gapla {
namespace {
constexpr int EV_LO = -48, EV_W = 64;              // shared window of d - c
constexpr int EV_COPIES = 4;                        // histogram copies (lane & 3): lanes of one warp that
                                                    // hold the same layer slot mostly hit different copies
constexpr int EV_THREADS = 512;

__device__ __forceinline__ void eval_word(int32_t w, int slot, uint32_t (*sh)[2][EV_W], unsigned long long *shleg,
                                          const int8_t *layer_of, EvalDev &E, int dlo, int dhi, int nbins) {
    const int d = w >> 1, f = w & 1;
    if (d > 0) atomicAdd(&shleg[slot], (unsigned long long)d);
    if (d >= EV_LO && d < EV_LO + EV_W) {
        atomicAdd(&sh[slot][f][d - EV_LO], 1u);
    } else {
        const int dc = min(max(d, dlo), dhi);
        if (dc != d) atomicAdd(E.oob, 1ull);
        atomicAdd(&E.hist[((int)layer_of[slot] * 2 + f) * nbins + (dc - dlo)], 1ull);
    }
}

__global__ void __launch_bounds__(EV_THREADS) k_eval_plane(const int32_t *__restrict__ words, int64_t n, int slots,
                                                           const int8_t *__restrict__ layer_of, EvalDev E, int dlo,
                                                           int dhi) {
    __shared__ uint32_t shc[EV_COPIES][MAXL][2][EV_W];
    __shared__ unsigned long long shleg[MAXL];
    for (int i = threadIdx.x; i < EV_COPIES * MAXL * 2 * EV_W; i += blockDim.x) (&shc[0][0][0][0])[i] = 0;
    if (threadIdx.x < MAXL) shleg[threadIdx.x] = 0;
    __syncthreads();
    uint32_t (*sh)[2][EV_W] = shc[threadIdx.x & (EV_COPIES - 1)];
    const int nbins = dhi - dlo + 1;
    const int64_t n4 = n / 4;
    const int4 *w4 = reinterpret_cast<const int4 *>(words);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int slot = (int)((4 * i0) % slots);                  // slot of word 4i, advanced without 64-bit modulo
    const int step = (int)((4 * stride) % slots);
    for (int64_t i = i0; i < n4; i += stride) {
        const int4 v = __ldcs(w4 + i);
        int s1 = slot + 1, s2 = slot + 2, s3 = slot + 3;
        s1 -= s1 >= slots ? slots : 0;
        s2 = s2 >= slots ? s2 - slots : s2;
        s2 -= s2 >= slots ? slots : 0;
        s3 = s3 % slots;
        eval_word(v.x, slot, sh, shleg, layer_of, E, dlo, dhi, nbins);
        eval_word(v.y, s1, sh, shleg, layer_of, E, dlo, dhi, nbins);
        eval_word(v.z, s2, sh, shleg, layer_of, E, dlo, dhi, nbins);
        eval_word(v.w, s3, sh, shleg, layer_of, E, dlo, dhi, nbins);
        slot += step;
        slot -= slot >= slots ? slots : 0;
    }
    for (int64_t e = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride)
        eval_word(words[e], (int)(e % slots), sh, shleg, layer_of, E, dlo, dhi, nbins);
    __syncthreads();
    for (int i = threadIdx.x; i < slots * 2 * EV_W; i += blockDim.x) {
        const int s = i / (2 * EV_W), f = (i / EV_W) & 1, b = i % EV_W;
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < EV_COPIES; ++k) c += shc[k][s][f][b];
        const int d = EV_LO + b;
        if (c) atomicAdd(&E.hist[((int)layer_of[s] * 2 + f) * nbins + (min(max(d, dlo), dhi) - dlo)], (unsigned long long)c);
        if (c && (d < dlo || d > dhi)) atomicAdd(E.oob, (unsigned long long)c);
    }
    if (threadIdx.x < slots && shleg[threadIdx.x]) atomicAdd(&E.legacy[layer_of[threadIdx.x]], shleg[threadIdx.x]);
}

// k_eval_nodes: unit wire edges per layer (len of every parent run on its layer) and via cuts;
// four nodes per thread and iteration (32-bit loads of the byte arrays, one 16-byte load of the
// lengths), per-thread counters in registers (layer index unrolled), one warp reduction per layer.
__global__ void __launch_bounds__(256) k_eval_nodes(DevForest F, DevScratch S, EvalDev E) {
    uint32_t wl[MAXL];
#pragma unroll
    for (int l = 0; l < MAXL; ++l) wl[l] = 0;
    unsigned long long myv = 0;
    auto node = [&](int l, int ed, int len, int b, int t) {
        const uint32_t w = ed != NO_DIR ? (uint32_t)len : 0u;
#pragma unroll
        for (int k = 0; k < MAXL; ++k) wl[k] += k == l ? w : 0u;
        myv += (unsigned)(t - b);
    };
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = F.n_nodes / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint32_t l4 = reinterpret_cast<const uint32_t *>(S.lay)[i];
        const uint32_t e4 = reinterpret_cast<const uint32_t *>(F.edir)[i];
        const uint32_t b4 = reinterpret_cast<const uint32_t *>(S.sb)[i];
        const uint32_t t4 = reinterpret_cast<const uint32_t *>(S.st)[i];
        const int4 len = reinterpret_cast<const int4 *>(F.len)[i];
        node(l4 & 0xff, e4 & 0xff, len.x, b4 & 0xff, t4 & 0xff);
        node((l4 >> 8) & 0xff, (e4 >> 8) & 0xff, len.y, (b4 >> 8) & 0xff, (t4 >> 8) & 0xff);
        node((l4 >> 16) & 0xff, (e4 >> 16) & 0xff, len.z, (b4 >> 16) & 0xff, (t4 >> 16) & 0xff);
        node(l4 >> 24, e4 >> 24, len.w, b4 >> 24, t4 >> 24);
    }
    for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F.n_nodes; i += stride)
        node(S.lay[i], F.edir[i], F.len[i], S.sb[i], S.st[i]);
#pragma unroll
    for (int k = 0; k < MAXL; ++k) {
        unsigned long long v = wl[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&E.wl[k], v);
    }
    for (int o = 16; o > 0; o >>= 1) myv += __shfl_xor_sync(FULL_MASK, myv, o);
    if ((threadIdx.x & 31) == 0 && myv) atomicAdd(E.vcuts, myv);
}
}  // namespace

static int sm_count() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

cudaError_t launch_eval_plane(const int32_t *words, int64_t n, int slots, const int8_t *layer_of_slot, EvalDev E,
                              int delta_lo, int delta_hi, cudaStream_t s) {
    if (n <= 0 || slots <= 0) return cudaSuccess;
    const int64_t want = (n / 4 + EV_THREADS - 1) / EV_THREADS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * 4));
    k_eval_plane<<<grid, EV_THREADS, 0, s>>>(words, n, slots, layer_of_slot, E, delta_lo, delta_hi);
    return cudaGetLastError();
}

cudaError_t launch_eval_nodes(const DevForest &F, const DevScratch &S, EvalDev E, cudaStream_t s) {
    if (F.n_nodes <= 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((F.n_nodes + 255) / 256, (int64_t)sm_count() * 8));
    k_eval_nodes<<<grid, 256, 0, s>>>(F, S, E);
    return cudaGetLastError();
}
}  // namespace gapla
