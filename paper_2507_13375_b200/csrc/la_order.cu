// The step before the hot path, on the GPU (the pre-assignment pi-model
// timing that goes with it is k_pre_timing in la_tree.cu):
//
//   k_order_keys ..   Alg. 1 lines 3-10 (PAPER §III-A l.213-262; readings R31, R33, R42, R43):
//   k_batch_ids       Divide, PartitionAndSort(N_c), PartitionAndSort(N_s), Sort(N_n),
//                     GetBatches, Concat; two stable CUB radix passes (a library sort
//                     primitive) order the nets, hand-written kernels form the keys and batches.
//
// Compiled with --fmad=false: every fp64 expression is evaluated as written (the band bounds
// C / 2^k and (1 - 0.01 k k) WNS must be the oracle's doubles bit for bit).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "la_device.cuh"
#include "la_internal.h"

namespace gapla {
namespace {

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// ---------------------------------------------------------- Alg. 1 l.3-10 --
// Per net: net slack (minimum over its sinks, l.217), 2D wirelength (sum of its segments'
// lengths), the class (Divide, l.3: 0 = N_c, 1 = N_s, 2 = N_n), the band and the two sort keys:
//   key1: N_c / N_s: net slack as an order-preserving 64-bit integer; N_n: wirelength;
//   key2: class << 48 | band << 32 | (N_c: INT32_MAX - criticality, so criticality descends).
// Two stable radix passes (key1, then key2) over the identity permutation order the nets by
// (class, band, -criticality, slack or wirelength, index) — the oracle's sort keys.
__device__ __forceinline__ uint64_t ordered_bits(double v) {
    if (v == 0.0) v = 0.0;                 // -0 and +0 compare equal: one key
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_crit_max(const int32_t *__restrict__ crit, int64_t n, int32_t th, int32_t *__restrict__ cmax) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int32_t c = (j < n && crit[j] > th) ? crit[j] : 0;
    c = __reduce_max_sync(FULL_MASK, c);
    if ((threadIdx.x & 31) == 0 && c > 0) atomicMax(cmax, c);
}

__global__ void k_order_keys(OrderIn in, const int32_t *__restrict__ cmax, uint64_t *__restrict__ key1,
                             uint64_t *__restrict__ key2, int32_t *__restrict__ idx) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= in.n_nets) return;
    double m = dinf();
    for (int64_t p = in.pin_ptr[j] + 1; p < in.pin_ptr[j + 1]; ++p) {   // sinks: pin 0 is the driver
        const double s = in.pin_slack[p];
        m = (s < m) ? s : m;
    }
    const int32_t c = in.crit[j];
    uint64_t k1, k2;
    if (c > in.th) {                                   // N_c: [C, C], [C/2, C), [C/4, C/2), ...
        const int32_t C = *cmax;
        uint64_t b = 0;
        if (c < C) {   // th >= 0 (la_paper_batches), so c >= 1 and b <= 31: C / 2^b is exact
            b = 1;
            while ((double)c < (double)C / (double)(1ull << b)) ++b;
        }
        k1 = ordered_bits(m);
        k2 = (0ull << 48) | (b << 32) | (uint64_t)(uint32_t)(0x7fffffff - c);
    } else if (in.wns < 0.0 && m < in.alpha * in.wns) {   // N_s: slack == WNS, (f_{k-1} WNS, f_k WNS]
        uint64_t b = 0;
        if (!(m <= in.wns)) {
            b = 1;
            while (b < 10 && !(m <= (1.0 - 0.01 * (double)b * (double)b) * in.wns)) ++b;
        }
        k1 = ordered_bits(m);
        k2 = (1ull << 48) | (b << 32);
    } else {                                           // N_n: congestion-driven, 2D wirelength (R43)
        int64_t wl = 0;
        for (int64_t s = in.seg_ptr[j]; s < in.seg_ptr[j + 1]; ++s) {
            const int4 q = reinterpret_cast<const int4 *>(in.seg_xy)[s];
            wl += abs(q.z - q.x) + abs(q.w - q.y);
        }
        k1 = (uint64_t)wl;
        k2 = 2ull << 48;
    }
    key1[j] = k1;
    key2[j] = k2;
    idx[j] = (int32_t)j;
}

__global__ void k_gather_key(const uint64_t *__restrict__ key, const int32_t *__restrict__ idx, int64_t n,
                             uint64_t *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = key[idx[i]];
}

// GetBatches + Concat: a subset starts where (class, band) changes; a batch starts at a subset
// start and every max_batch nets after it.  subset_start = running max of the subsets' starts.
__global__ void k_subset_heads(const uint64_t *__restrict__ k2s, int64_t n, int64_t *__restrict__ head_at) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    head_at[i] = (i == 0 || (k2s[i] >> 32) != (k2s[i - 1] >> 32)) ? i : 0;
}

__global__ void k_batch_flags(const int64_t *__restrict__ sub0, int64_t n, int64_t max_batch,
                              int32_t *__restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = ((i - sub0[i]) % max_batch) == 0 ? 1 : 0;
}

__global__ void k_batch_scatter(const int32_t *__restrict__ incl, const int32_t *__restrict__ idx, int64_t n,
                                int32_t *__restrict__ batch_of) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) batch_of[idx[i]] = incl[i] - 1;
}

struct MaxI64 {
    __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

#define OCK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

}  // namespace

cudaError_t gpu_paper_batches(const OrderIn &in, int32_t *batch_of, int32_t *n_batches, cudaStream_t s,
                              int64_t *launches) {
    const int64_t n = in.n_nets;
    *n_batches = 0;
    if (n == 0) return cudaSuccess;
    char *buf = nullptr;
    // key1 | key2 | key_a | key_b (4 x 8n) | idx_a | idx_b | flags | incl (4 x 4n) | sub0 heads (2 x 8n) | cmax
    const size_t b8 = 8 * (size_t)n, b4 = 4 * (size_t)n;
    size_t tmp_sort = 0, tmp_max = 0, tmp_sum = 0;
    OCK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                        (int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 64, s));
    OCK(cub::DeviceScan::InclusiveScan(nullptr, tmp_max, (int64_t *)nullptr, (int64_t *)nullptr, MaxI64(), (int)n,
                                       s));
    OCK(cub::DeviceScan::InclusiveSum(nullptr, tmp_sum, (int32_t *)nullptr, (int32_t *)nullptr, (int)n, s));
    const size_t tmp = std::max(tmp_sort, std::max(tmp_max, tmp_sum));
    const size_t total = 6 * b8 + 4 * b4 + 256 + tmp;
    OCK(dmalloc(&buf, total));
    uint64_t *key1 = (uint64_t *)buf, *key2 = key1 + n, *ka = key2 + n, *kb = ka + n;
    int64_t *heads = (int64_t *)(kb + n), *sub0 = heads + n;
    int32_t *idx_a = (int32_t *)(sub0 + n), *idx_b = idx_a + n, *flag = idx_b + n, *incl = flag + n;
    int32_t *cmax = (int32_t *)(incl + n);
    void *tmpp = (char *)cmax + 256;
    cudaError_t e = cudaSuccess;
    do {
        const int T = 256;
        if ((e = cudaMemsetAsync(cmax, 0, 4, s))) break;
        k_crit_max<<<nblk(n, T), T, 0, s>>>(in.crit, n, in.th, cmax);
        k_order_keys<<<nblk(n, T), T, 0, s>>>(in, cmax, key1, key2, idx_a);
        size_t tb = tmp;
        // pass 1: key1 (stable over the identity order = ties by net index)
        if ((e = cub::DeviceRadixSort::SortPairs(tmpp, tb, key1, ka, idx_a, idx_b, (int)n, 0, 64, s))) break;
        k_gather_key<<<nblk(n, T), T, 0, s>>>(key2, idx_b, n, key1);
        // pass 2: key2 (class, band, criticality descending), stable over pass 1's order
        tb = tmp;
        if ((e = cub::DeviceRadixSort::SortPairs(tmpp, tb, key1, kb, idx_b, idx_a, (int)n, 0, 50, s))) break;
        k_subset_heads<<<nblk(n, T), T, 0, s>>>(kb, n, heads);
        tb = tmp;
        if ((e = cub::DeviceScan::InclusiveScan(tmpp, tb, heads, sub0, MaxI64(), (int)n, s))) break;
        k_batch_flags<<<nblk(n, T), T, 0, s>>>(sub0, n, in.max_batch, flag);
        tb = tmp;
        if ((e = cub::DeviceScan::InclusiveSum(tmpp, tb, flag, incl, (int)n, s))) break;
        k_batch_scatter<<<nblk(n, T), T, 0, s>>>(incl, idx_a, n, batch_of);
        if ((e = cudaGetLastError())) break;
        if ((e = cudaMemcpyAsync(n_batches, incl + n - 1, 4, cudaMemcpyDeviceToHost, s))) break;
        e = cudaStreamSynchronize(s);
        if (launches) *launches += 11;
    } while (0);
    dfree(buf);
    return e;
}

}  // namespace gapla
