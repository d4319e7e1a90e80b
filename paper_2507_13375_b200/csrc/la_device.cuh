// Device helpers shared by the hot-path kernels (la_assign.cu, la_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "la_internal.h"

namespace gapla {

constexpr unsigned FULL_MASK = 0xffffffffu;

// Demand commit: a fire-and-forget integer reduction (RED, no returned value to wait for).
__device__ __forceinline__ void red_add(int32_t *p, int32_t v) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Eq. (3) marginal cost of one more unit on an element (reading R18):
// packed word w = ((d - c) << 1) | (c == 0); host-built table over the clamped d - c (R20).
__device__ __forceinline__ double marginal(const DevGrid &G, int32_t w) {
    int delta = w >> 1;
    delta = min(max(delta, G.delta_lo), G.delta_hi);
    const double *M = (w & 1) ? G.Mzero : G.Mpos;
    return __ldg(M + (delta - G.delta_lo));
}

// Packed word index of the unit edge with lower endpoint (x, y) on layer l.
__device__ __forceinline__ int64_t wire_word(const DevGrid &G, int dtype, int l, int x, int y) {
    return dtype == 0 ? ((int64_t)y * (G.X - 1) + x) * G.LH + G.lidx[l]
                      : ((int64_t)x * (G.Y - 1) + y) * G.LV + G.lidx[l];
}

// Lowest coordinate of the unit edges of a node's parent run (runs are summed in
// ascending coordinate, reading R23).
__device__ __forceinline__ int run_lo(int edir, int x, int y, int len) {
    switch (edir) {
        case 0: return x - len;   // parent lies west
        case 1: return x;
        case 2: return y - len;
        default: return y;
    }
}

__device__ __forceinline__ void stage_tab(TechTab &T, const TechTab *src) {
    const double *s = reinterpret_cast<const double *>(src);
    double *d = reinterpret_cast<double *>(&T);
    for (int i = threadIdx.x; i < (int)(sizeof(TechTab) / sizeof(double)); i += blockDim.x) d[i] = s[i];
}

}  // namespace gapla
