// la_get_solution on the GPU (SURVEY §8(b) outputs; include/la.h la_get_solution): per input net
// the wire count (tree edges = nodes - 1), the via-stack count (nodes with t > b) and f[root],
// offsets by an exclusive scan, then every net's wires (x1, y1, x2, y2, layer) and via stacks
// (x, y, b, t) in ascending lexicographic order.  Pure data movement over the decisions the DP
// wrote (lay, sb, st per node): no arithmetic of the method.
//
//   k_sol_count  thread per forest position: counts into input-net order, f[root], via cuts
//   k_sol_fill   warp per forest position: each lane keys one node's wire / via stack; its rank
//                among the net's keys (warp-shuffle comparisons, 32 x 32 per pair of node chunks)
//                is its row in the net's output range
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "la_internal.h"

namespace gapla {
namespace {

constexpr int SOL_T = 256;

__global__ void __launch_bounds__(SOL_T) k_sol_count(DevForest F, DevScratch S, int64_t *wcnt, int64_t *vcnt,
                                                      double *cost, unsigned long long *vcuts) {
    const int64_t p = blockIdx.x * (int64_t)SOL_T + threadIdx.x;
    unsigned long long vc = 0;
    if (p < F.n_nets) {
        const int64_t a = F.net_node0[p], b = F.net_node0[p + 1];
        const int64_t net = F.net_id[p];
        int64_t v = 0;
        for (int64_t k = a; k < b; ++k) {
            const int sb = S.sb[k], st = S.st[k];
            v += st > sb;
            vc += (unsigned long long)(st - sb);
        }
        wcnt[net] = b - a - 1;
        vcnt[net] = v;
        cost[net] = S.froot[p];
    }
    vc = __reduce_add_sync(0xffffffffu, (unsigned)vc);
    if ((threadIdx.x & 31) == 0 && vc) atomicAdd(vcuts, vc);
}

struct SolKeys {
    unsigned long long w, v;   // wire key x1 y1 x2 y2 (16 bits each); via key x y b t
    int wl;                    // wire layer (the key's last field)
    bool hw, hv;               // node has a wire (non-root) / a via stack (t > b)
};

__device__ __forceinline__ SolKeys sol_keys(const DevForest &F, const DevScratch &S, int64_t k, bool valid) {
    SolKeys r{0ull, 0ull, 0, false, false};
    if (!valid) return r;
    const uint32_t xy = F.xy[k];
    const int x = xy & 0xffff, y = xy >> 16;
    const int ed = F.edir[k];
    if (ed != NO_DIR) {
        const int ln = F.len[k];
        int qx = x, qy = y;   // parent GCell
        if (ed == 0) qx = x - ln;
        else if (ed == 1) qx = x + ln;
        else if (ed == 2) qy = y - ln;
        else qy = y + ln;
        r.w = ((unsigned long long)min(x, qx) << 48) | ((unsigned long long)min(y, qy) << 32) |
              ((unsigned long long)max(x, qx) << 16) | (unsigned long long)max(y, qy);
        r.wl = S.lay[k];
        r.hw = true;
    }
    const int sb = S.sb[k], st = S.st[k];
    if (st > sb) {
        r.v = ((unsigned long long)x << 48) | ((unsigned long long)y << 32) | ((unsigned long long)sb << 16) |
              (unsigned long long)st;
        r.hv = true;
    }
    return r;
}

__global__ void __launch_bounds__(SOL_T) k_sol_fill(DevForest F, DevScratch S, const int64_t *__restrict__ wptr,
                                                     const int64_t *__restrict__ vptr, int32_t *wires, int32_t *vias) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (SOL_T / 32);
    for (int64_t p = blockIdx.x * (int64_t)(SOL_T / 32) + (threadIdx.x >> 5); p < F.n_nets; p += nw) {
        const int64_t a = F.net_node0[p];
        const int m = (int)(F.net_node0[p + 1] - a);
        const int64_t net = F.net_id[p];
        const int64_t w0 = wptr[net], v0 = vptr[net];
        for (int c0 = 0; c0 < m; c0 += 32) {
            const int i = c0 + lane;
            const SolKeys me = sol_keys(F, S, a + i, i < m);
            int rw = 0, rv = 0;
            for (int d0 = 0; d0 < m; d0 += 32) {
                const int j = d0 + lane;
                const SolKeys o = sol_keys(F, S, a + j, j < m);
                const int cnt = min(32, m - d0);
                for (int s = 0; s < cnt; ++s) {
                    const unsigned long long ow = __shfl_sync(0xffffffffu, o.w, s);
                    const int owl = __shfl_sync(0xffffffffu, o.wl, s);
                    const bool ohw = __shfl_sync(0xffffffffu, o.hw, s);
                    const unsigned long long ov = __shfl_sync(0xffffffffu, o.v, s);
                    const bool ohv = __shfl_sync(0xffffffffu, o.hv, s);
                    const int jj = d0 + s;
                    // total order (key, node index): a permutation of the net's rows even on equal keys
                    rw += ohw && (ow < me.w || (ow == me.w && (owl < me.wl || (owl == me.wl && jj < i))));
                    rv += ohv && (ov < me.v || (ov == me.v && jj < i));
                }
            }
            if (i < m && me.hw) {
                int32_t *o = wires + 5 * (w0 + rw);
                o[0] = (int32_t)(me.w >> 48);
                o[1] = (int32_t)((me.w >> 32) & 0xffff);
                o[2] = (int32_t)((me.w >> 16) & 0xffff);
                o[3] = (int32_t)(me.w & 0xffff);
                o[4] = me.wl;
            }
            if (i < m && me.hv) {
                int32_t *o = vias + 4 * (v0 + rv);
                o[0] = (int32_t)(me.v >> 48);
                o[1] = (int32_t)((me.v >> 32) & 0xffff);
                o[2] = (int32_t)((me.v >> 16) & 0xffff);
                o[3] = (int32_t)(me.v & 0xffff);
            }
        }
    }
}

}  // namespace

// Counts, offsets (wptr / vptr [N+1], exclusive sums of the counts), net cost and via cuts.
// wcnt / vcnt: [N+1] scratch; temp: CUB scratch (temp_bytes in/out: query with temp == nullptr).
cudaError_t sol_count(const DevForest &F, const DevScratch &S, int64_t *wcnt, int64_t *vcnt, int64_t *wptr,
                      int64_t *vptr, double *cost, unsigned long long *vcuts, void *temp, size_t *temp_bytes,
                      cudaStream_t s) {
    const int64_t N = F.n_nets;
    if (!temp) {
        size_t b1 = 0;
        cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, b1, wcnt, wptr, N + 1, s);
        *temp_bytes = b1;
        return e;
    }
    cudaError_t e = cudaMemsetAsync(wcnt + N, 0, sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(vcnt + N, 0, sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(vcuts, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    if (N > 0) {
        k_sol_count<<<(unsigned)((N + SOL_T - 1) / SOL_T), SOL_T, 0, s>>>(F, S, wcnt, vcnt, cost, vcuts);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    e = cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, wcnt, wptr, N + 1, s);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, vcnt, vptr, N + 1, s);
    return e;
}

cudaError_t sol_fill(const DevForest &F, const DevScratch &S, const int64_t *wptr, const int64_t *vptr, int32_t *wires,
                     int32_t *vias, cudaStream_t s) {
    if (F.n_nets <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    const int64_t want = (F.n_nets + SOL_T / 32 - 1) / (SOL_T / 32);
    const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)sms * 8);
    k_sol_fill<<<grid, SOL_T, 0, s>>>(F, S, wptr, vptr, wires, vias);
    return cudaGetLastError();
}

}  // namespace gapla
