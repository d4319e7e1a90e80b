// Chunked tree passes over the batch-major forest (DESIGN §5 "Chunked tree passes"):
//
//   k_elmore      (K6 + K7)  Elmore delay / downstream cap on the 3D RC trees of the assigned
//                            nets (PAPER §II-C l.146, §III-D l.443-444; DESIGN §3 O9): a thread
//                            per net (see below; not chunked)
//   k_pre_timing             pre-assignment timing on the 2D LA trees with the pi model and the
//                            per-direction average unit R / C (PAPER §III-B l.283-286; Alg. 1
//                            inputs r_avg, c_avg l.240-241; reading R44)
//
// A warp runs one CHUNK at a time: consecutive forest positions whose nets hold at most
// CHUNK_NODES nodes and CHUNK_SINKS sinks together (lane = node), or one bigger net alone.  Small
// chunks load every node and sink field once, lane by lane (coalesced: a chunk's nodes and sinks
// are contiguous), keep the per-node values (Cdown, rc, T(in)) in shared memory and run the
// recursions in height steps (a node's sons have smaller heights: they finish one step earlier);
// a bigger net is walked in windows of 32 nodes with its per-node values in global scratch.
// The chunk record carries the
// chunk's first node and sink, so a warp's loads do not wait on another lookup, and the next
// chunk's record is fetched while the current one runs.
//
// k_elmore keeps the oracle's expression trees operand for operand: its outputs are
// bitwise equal to the oracle's; the via-stack sums of one node run in registers as a running
// sum up from and down from the entry layer, each sink / son picking up the value at its layer.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "la_device.cuh"
#include "la_internal.h"

namespace gapla {
namespace {

constexpr int TW = 8;   // warps per CTA

struct Chunk {
    int64_t pb, n0, q0;
    int np, nq, nn;
    bool big;
};

__device__ __forceinline__ Chunk decode(const DevForest &F, int4 c) {
    Chunk k;
    k.pb = c.x;
    k.n0 = c.y;
    k.q0 = c.z;
    k.big = (c.w >> 31) & 1;
    if (!k.big) {
        k.np = c.w & 63;
        k.nq = (c.w >> 6) & 127;
        k.nn = (c.w >> 13) & 63;
    } else {              // one bigger net
        k.np = 1;
        k.nq = 0;
        k.nn = (int)(F.net_node0[k.pb + 1] - k.n0);
    }
    return k;
}

// ---------------------------------------------------------------- k_elmore --
// A thread per net (lanes = consecutive forest positions: their nodes are adjacent, so a warp's
// loads share sectors), nodes walked in forest order for the bottom-up pass and backward for the
// top-down one.  The per-node values (Cdown, rc, then T(in) in rc's place: rc of a node is dead
// once its parent has read it) live in shared memory, [node][thread], for nets of at most
// ELM_LOCAL nodes, in global scratch beyond.  Measured alternatives (profiles/r02_elm_*): a warp
// per chunk of nets with lane = node in height steps ran 4x slower (2.5 active lanes per
// instruction in the via-stack loops).  Round 2, session 4 (config 5, one box, 10 steps): the
// via stacks sum each branch set once per change point (via_stack): 4.61 -> 4.18 ms, 1.34G warp
// instructions; a CTA per block of consecutive nets with every field staged into shared memory
// by coalesced loads (row-major 7.5-10 ms: bank conflicts; transposed [node-in-net][net] columns
// 7.6-8.9 ms for 64/128-thread CTAs and 192-1024-node capacities): DRAM 7.9 -> 4.8 GB, but 2.5x
// the instructions, 10-13 active lanes and barrier stalls between the phases; the next node's
// fields loaded before the current node's arithmetic: 4.35 ms (107 registers; config 4 2.94 ->
// 2.64 ms); register caps of 80 / 64 (6 / 8 CTAs per SM): 4.97 / 8.57 ms (spills); CTAs of 64 / 32
// threads (ELM_T_DEF; more resident warps at 93 registers): 4.18 / 4.41 ms vs 4.17 at 128, and 64
// threads at 80 registers 4.41 ms.
#ifndef ELM_LOCAL
#define ELM_LOCAL 6
#endif
#ifndef ELM_T_DEF
#define ELM_T_DEF 128
#endif
constexpr int ELM_T = ELM_T_DEF;   // threads per k_elmore CTA
#ifndef ELM_MINB
#define ELM_MINB 1      // k_elmore CTAs per SM the register budget must allow
#endif

struct Vals {          // node values: element of node n at p[(n - base) * stride]
    double *Cd, *Rc, *Tin;
    int64_t base, stride;
    __device__ __forceinline__ int64_t at(int64_t n) const { return (n - base) * stride; }
};

// Bottom-up (K6): Cdown(n) = C0 + ((Cw1 + Cd1) + ...); rc(n) = F0u + ((c1 + c2) + ...)
__device__ __forceinline__ void elm_up(const Vals &V, const TechTab &T, const DevForest &F, const uint8_t *lay,
                                       int64_t n, int ln, int64_t qa, int ns, int nk, const int kid[4]) {
    double C0 = 0.0, F0u = 0.0;
    for (int64_t q = qa; q < qa + ns; ++q) {
        const double cq = F.p_cap[q];
        C0 = C0 + cq;
        F0u = F0u + cq * T.VR[F.p_layer[q] * MAXL + ln];
    }
    double K = 0.0, R = 0.0;
#pragma unroll
    for (int i = 0; i < MAXKIDS; ++i) {
        if (i < nk) {
            const int64_t s = kid[i];
            const int ls = lay[s];
            const double len = (double)F.len[s];
            const double Cw = T.c[ls] * len, Rw = T.r[ls] * len;
            const double Cd = V.Cd[V.at(s)];
            K = K + (Cw + Cd);
            R = R + ((V.Rc[V.at(s)] + Rw * (0.5 * Cw + Cd)) + (Cw + Cd) * T.VR[ln * MAXL + ls]);
        }
    }
    V.Cd[V.at(n)] = C0 + K;
    V.Rc[V.at(n)] = F0u + R;
}

// The via stack of one node (K7): T(k+1) = T(k) + vr[k] C>=(k+1) going up from the entry layer
// to t, T(k-1) = T(k) + vr[k-1] C<=(k-1) going down to b.  C>=(j) sums the branches (sinks in
// input order, then sons in child order) with layer >= j in that canonical order; the set only
// changes where j passes a branch's layer, so one sum serves every level up to the smallest
// branch layer >= j (down: the largest <= j) — the same terms in the same order, hence the same
// double, bit for bit, with one sum per distinct branch layer instead of one per level.
// each(f) calls f(layer, C) for every branch in canonical order; TK(k) is T at layer k.
template <class Each, class TKf>
__device__ __forceinline__ void via_stack(const TechTab &T, int ln, int b, int t, Each each, TKf TK) {
    for (int j = ln + 1; j <= t;) {
        double acc = 0.0;
        int lim = t;
        each([&](int l, double c) {
            if (l >= j) {
                acc = acc + c;
                lim = min(lim, l);
            }
        });
        for (; j <= lim; ++j) TK(j) = TK(j - 1) + T.vr[j - 1] * acc;
    }
    for (int j = ln - 1; j >= b;) {
        double acc = 0.0;
        int lim = b;
        each([&](int l, double c) {
            if (l <= j) {
                acc = acc + c;
                lim = max(lim, l);
            }
        });
        for (; j >= lim; --j) TK(j) = TK(j + 1) + T.vr[j] * acc;
    }
}

// Top-down (K7): T through the via stack [b, t] of node n (entry layer ln), then the pi wires of
// its sons.  T(k+1) = T(k) + vr[k] C>=(k+1) going up, T(k-1) = T(k) + vr[k-1] C<=(k-1) going
// down (branches: sinks in input order, then sons in child order), into the thread's shared-
// memory column Tk[k * ELM_T]; each sink takes T at its pin layer, each son T(ls) + Rw (Cw / 2 +
// Cdown).  (A running sum in registers that hands each branch its value on the way costs more
// instructions: measured 5.9 vs 5.1 ms.)
__device__ __forceinline__ void elm_down(const Vals &V, const TechTab &T, const DevForest &F, const uint8_t *lay,
                                         double *sink_delay, double *Tk, int64_t n, int ln, int b, int t, bool root,
                                         int64_t qa, int ns, int nk, const int kid[4]) {
#define TK(k) Tk[(k) * ELM_T]
    TK(ln) = root ? 0.0 : V.Tin[V.at(n)];
    int lsk[MAXKIDS];
    double cbk[MAXKIDS], tail[MAXKIDS];   // Cw + Cdown; Rw (Cw / 2 + Cdown)
#pragma unroll
    for (int i = 0; i < MAXKIDS; ++i) {
        lsk[i] = 0;
        cbk[i] = tail[i] = 0.0;
        if (i < nk) {
            const int64_t s = kid[i];
            const int ls = lay[s];
            const double len = (double)F.len[s];
            const double cw = T.c[ls] * len, rw = T.r[ls] * len, cd = V.Cd[V.at(s)];
            lsk[i] = ls;
            cbk[i] = cw + cd;
            tail[i] = rw * (0.5 * cw + cd);
        }
    }
    const bool few = ns <= 4;
    int pl[4];
    double pc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        pl[u] = 0;
        pc[u] = 0.0;
        if (few && u < ns) {
            pl[u] = F.p_layer[qa + u];
            pc[u] = F.p_cap[qa + u];
        }
    }
    auto each = [&](auto f) {
        if (few) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (u < ns) f(pl[u], pc[u]);
        } else {
            for (int64_t q = qa; q < qa + ns; ++q) f((int)F.p_layer[q], F.p_cap[q]);
        }
#pragma unroll
        for (int i = 0; i < MAXKIDS; ++i)
            if (i < nk) f(lsk[i], cbk[i]);
    };
    via_stack(T, ln, b, t, each, [&](int k) -> double & { return TK(k); });
    if (few) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (u < ns) sink_delay[F.p_orig[qa + u]] = TK(pl[u]);
    } else {
        for (int64_t q = qa; q < qa + ns; ++q) sink_delay[F.p_orig[q]] = TK(F.p_layer[q]);
    }
#pragma unroll
    for (int i = 0; i < MAXKIDS; ++i)
        if (i < nk) V.Tin[V.at(kid[i])] = TK(lsk[i]) + tail[i];
#undef TK
}

__global__ void __launch_bounds__(ELM_T, ELM_MINB) k_elmore(DevForest F, DevScratch S, const TechTab *__restrict__ tab,
                                                 int64_t net_beg, int64_t net_end, const int32_t *__restrict__ list) {
    __shared__ TechTab T;
    __shared__ double sv[2][ELM_LOCAL][ELM_T];   // Cdown; rc, then T(in)
    extern __shared__ double Tks[];               // [L][ELM_T]: T(n, k) of the current node, a column per thread
    stage_tab(T, tab);
    __syncthreads();
    const int64_t idx = net_beg + blockIdx.x * (int64_t)ELM_T + threadIdx.x;
    if (idx >= net_end) return;
    const int64_t p = list ? (int64_t)list[idx] : idx;   // this rank's nets (multi-GPU) or all
    const int64_t n0 = F.net_node0[p], n1 = F.net_node0[p + 1];
    const bool local = n1 - n0 <= ELM_LOCAL;
    const Vals V = local ? Vals{&sv[0][0][threadIdx.x], &sv[1][0][threadIdx.x], &sv[1][0][threadIdx.x], n0, ELM_T}
                         : Vals{S.Cd, S.rcv, S.Tin, 0, 1};
    const uint8_t *lay = S.lay;
    for (int64_t n = n0; n < n1; ++n) {
        const int4 k4 = reinterpret_cast<const int4 *>(F.kid)[n];
        const int kid[4] = {k4.x, k4.y, k4.z, k4.w};
        elm_up(V, T, F, lay, n, lay[n], F.sink0[n], F.nsink[n], F.nkid[n], kid);
    }
    const int64_t nid = F.net_id[p];
    S.net_cap[nid] = V.Cd[V.at(n1 - 1)];
    S.net_rc[nid] = V.Rc[V.at(n1 - 1)];
    for (int64_t n = n1 - 1; n >= n0; --n) {
        const int4 k4 = reinterpret_cast<const int4 *>(F.kid)[n];
        const int kid[4] = {k4.x, k4.y, k4.z, k4.w};
        elm_down(V, T, F, lay, S.sink_delay, &Tks[threadIdx.x], n, lay[n], S.sb[n], S.st[n], n == n1 - 1,
                 F.sink0[n], F.nsink[n], F.nkid[n], kid);
    }
}

// ------------------------------------------------------------ k_pre_timing --
// Cdn(n) = sum of its sink caps + sum over sons s of (C_s + Cdn(s)); D(root) = 0,
// D(s) = D(n) + R_s (C_s / 2 + Cdn(s)); edge into n: R = r_t len, C = c_t len (t: E / W = H).
__device__ __forceinline__ int dtype_of(int edir) { return edir <= 1 ? 0 : 1; }

struct PreSmem {
    double Cd[32], D[32], R[32], C[32];
    double q[CHUNK_SINKS];
};

__device__ __forceinline__ void pre_small(const DevForest &F, const PreRC &P, const Chunk &c, PreSmem &m,
                                          double *sink_delay, double *net_cap) {
    const int lane = threadIdx.x & 31;
    const bool act = lane < c.nn;
    const int64_t n = c.n0 + lane;
    int4 k4 = make_int4(-1, -1, -1, -1);
    int nk = 0, h = 0, s0 = 0, ns = 0, e = 0, ed = 255, len = 0;
    int64_t nid = 0;
    if (act) {
        k4 = reinterpret_cast<const int4 *>(F.kid)[n];
        nk = F.nkid[n];
        h = F.height[n];
        s0 = (int)(F.sink0[n] - c.q0);
        ns = F.nsink[n];
        ed = F.edir[n];
        len = F.len[n];
    }
    for (int k = lane; k < c.nq; k += 32) m.q[k] = F.p_cap[c.q0 + k];
    if (lane < c.np) {
        e = (int)(F.net_node0[c.pb + lane + 1] - c.n0) - 1;
        nid = F.net_id[c.pb + lane];
    }
    double R = 0.0, C = 0.0;
    if (act && ed != NO_DIR) {
        const bool v = dtype_of(ed);   // (selects, not an indexed parameter: no local-memory copy)
        R = (v ? P.rd[1] : P.rd[0]) * (double)len;
        C = (v ? P.cd[1] : P.cd[0]) * (double)len;
    }
    m.R[lane] = R;
    m.C[lane] = C;
    const unsigned roots = __reduce_or_sync(FULL_MASK, lane < c.np ? 1u << e : 0u);
    const bool root = (roots >> lane) & 1u;
    const int hmax = __reduce_max_sync(FULL_MASK, act ? h : 0);
    const int kl[4] = {k4.x - (int)c.n0, k4.y - (int)c.n0, k4.z - (int)c.n0, k4.w - (int)c.n0};
    __syncwarp();
    for (int hh = 0; hh <= hmax; ++hh) {
        if (act && h == hh) {
            double c0 = 0.0;
            for (int k = 0; k < ns; ++k) c0 = c0 + m.q[s0 + k];
            double K = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (i < nk) K = K + (m.C[kl[i]] + m.Cd[kl[i]]);
            m.Cd[lane] = c0 + K;
        }
        __syncwarp();
    }
    if (root) m.D[lane] = 0.0;
    __syncwarp();
    for (int hh = hmax; hh >= 0; --hh) {
        if (act && h == hh) {
            const double D = m.D[lane];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (i < nk) m.D[kl[i]] = D + m.R[kl[i]] * (0.5 * m.C[kl[i]] + m.Cd[kl[i]]);
            for (int k = 0; k < ns; ++k) m.q[s0 + k] = D;   // the sink caps are no longer needed
        }
        __syncwarp();
    }
    for (int k = lane; k < c.nq; k += 32) sink_delay[F.p_orig[c.q0 + k]] = m.q[k];
    if (lane < c.np) net_cap[nid] = m.Cd[e];
    __syncwarp();
}

// One bigger net per warp, walked in windows of 32 nodes (lane = node), height steps inside a
// window, per-node values in global scratch: bottom-up with the windows forward, top-down
// backward (measured 3.2 ms at config 5 against 4.1 ms for a lane per net in groups of 32).
__device__ __forceinline__ void pre_big(const DevForest &F, const PreRC &P, const Chunk &c, double *Cd, double *Dg,
                                        double *sink_delay, double *net_cap) {
    const int lane = threadIdx.x & 31;
    const int nn = c.nn;
    auto Rof = [&](int64_t s) { return (dtype_of(F.edir[s]) ? P.rd[1] : P.rd[0]) * (double)F.len[s]; };
    auto Cof = [&](int64_t s) { return (dtype_of(F.edir[s]) ? P.cd[1] : P.cd[0]) * (double)F.len[s]; };
    for (int wb = 0; wb < nn; wb += 32) {
        const bool act = wb + lane < nn;
        const int64_t n = c.n0 + wb + lane;
        const int h = act ? F.height[n] : 0;
        const int hlo = __reduce_min_sync(FULL_MASK, act ? h : 0x7fffffff);
        const int hhi = __reduce_max_sync(FULL_MASK, act ? h : 0);
        for (int hh = hlo; hh <= hhi; ++hh) {
            if (act && h == hh) {
                double c0 = 0.0;
                const int64_t q = F.sink0[n];
                for (int k = 0; k < F.nsink[n]; ++k) c0 = c0 + F.p_cap[q + k];
                double K = 0.0;
                for (int i = 0; i < F.nkid[n]; ++i) {
                    const int64_t s = F.kid[n * 4 + i];
                    K = K + (Cof(s) + Cd[s]);
                }
                Cd[n] = c0 + K;
            }
            __syncwarp();
        }
    }
    const int64_t rt = c.n0 + nn - 1;
    if (lane == 0) {
        Dg[rt] = 0.0;
        net_cap[F.net_id[c.pb]] = Cd[rt];
    }
    __syncwarp();
    for (int wb = ((nn - 1) / 32) * 32; wb >= 0; wb -= 32) {
        const bool act = wb + lane < nn;
        const int64_t n = c.n0 + wb + lane;
        const int h = act ? F.height[n] : 0;
        const int hlo = __reduce_min_sync(FULL_MASK, act ? h : 0x7fffffff);
        const int hhi = __reduce_max_sync(FULL_MASK, act ? h : 0);
        for (int hh = hhi; hh >= hlo; --hh) {
            if (act && h == hh) {
                const double D = Dg[n];
                for (int i = 0; i < F.nkid[n]; ++i) {
                    const int64_t s = F.kid[n * 4 + i];
                    Dg[s] = D + Rof(s) * (0.5 * Cof(s) + Cd[s]);
                }
                const int64_t q = F.sink0[n];
                for (int k = 0; k < F.nsink[n]; ++k) sink_delay[F.p_orig[q + k]] = D;
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(TW * 32, 4) k_pre_timing(DevForest F, const int4 *__restrict__ chunks,
                                                          int64_t n_chunks, PreRC P, double *Cd, double *Dg,
                                                          double *sink_delay, double *net_cap) {
    __shared__ PreSmem sm[TW];
    const int w = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * TW;
    int64_t ci = (int64_t)blockIdx.x * TW + w;
    int4 nxt = ci < n_chunks ? chunks[ci] : make_int4(0, 0, 0, 0);
    for (; ci < n_chunks; ci += nw) {
        const int4 cur = nxt;
        if (ci + nw < n_chunks) nxt = chunks[ci + nw];   // the next record, fetched while this chunk runs
        const Chunk c = decode(F, cur);
        if (!c.big) pre_small(F, P, c, sm[w], sink_delay, net_cap);
        else pre_big(F, P, c, Cd, Dg, sink_delay, net_cap);
    }
}

// Thread-per-net variant of k_pre_timing (A/B: GAPLA_PRE_V1=1): lane = net, nodes walked in
// forest order with per-node values in global scratch (the round-1 k_elmore layout).
__global__ void __launch_bounds__(128) k_pre_timing_v1(DevForest F, int64_t n_nets, PreRC P, double *Cd, double *Dg,
                                                      double *sink_delay, double *net_cap) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n_nets) return;
    auto Rof = [&](int64_t s) { return (dtype_of(F.edir[s]) ? P.rd[1] : P.rd[0]) * (double)F.len[s]; };
    auto Cof = [&](int64_t s) { return (dtype_of(F.edir[s]) ? P.cd[1] : P.cd[0]) * (double)F.len[s]; };
    const int64_t n0 = F.net_node0[p], n1 = F.net_node0[p + 1];
    for (int64_t n = n0; n < n1; ++n) {
        double c0 = 0.0;
        const int64_t q = F.sink0[n];
        const int ns = F.nsink[n], nk = F.nkid[n];
        for (int k = 0; k < ns; ++k) c0 = c0 + F.p_cap[q + k];
        const int4 k4 = reinterpret_cast<const int4 *>(F.kid)[n];
        const int kid[4] = {k4.x, k4.y, k4.z, k4.w};
        double K = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (i < nk) K = K + (Cof(kid[i]) + Cd[kid[i]]);
        Cd[n] = c0 + K;
    }
    net_cap[F.net_id[p]] = Cd[n1 - 1];
    double D = 0.0;
    for (int64_t n = n1 - 1; n >= n0; --n) {
        if (n != n1 - 1) D = Dg[n];
        const int nk = F.nkid[n], ns = F.nsink[n];
        const int4 k4 = reinterpret_cast<const int4 *>(F.kid)[n];
        const int kid[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (i < nk) Dg[kid[i]] = D + Rof(kid[i]) * (0.5 * Cof(kid[i]) + Cd[kid[i]]);
        const int64_t q = F.sink0[n];
        for (int k = 0; k < ns; ++k) sink_delay[F.p_orig[q + k]] = D;
    }
}

template <class K>
cudaError_t tree_grid(K kernel, int64_t n_chunks, unsigned *grid) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, TW * 32, 0);
    const int64_t want = (n_chunks + TW - 1) / TW;
    *grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1)));
    return e;
}

}  // namespace

cudaError_t launch_elmore(const DevForest &F, const DevScratch &S, const TechTab *tab, int L, int64_t net_beg,
                          int64_t net_end, const int32_t *list, cudaStream_t s) {
    const int64_t n = net_end - net_beg;
    if (n <= 0) return cudaSuccess;
    const size_t sm = sizeof(double) * (size_t)L * ELM_T;
    k_elmore<<<(unsigned)((n + ELM_T - 1) / ELM_T), ELM_T, sm, s>>>(F, S, tab, net_beg, net_end, list);
    return cudaGetLastError();
}

cudaError_t launch_pre_timing(const DevForest &F, const int4 *chunks, int64_t n_chunks, const PreRC &P, double *Cd,
                              double *Dg, double *sink_delay, double *net_cap, cudaStream_t s) {
    if (n_chunks == 0) return cudaSuccess;
    static const bool v1 = getenv("GAPLA_PRE_V1") && atoi(getenv("GAPLA_PRE_V1")) != 0;
    if (v1) {
        k_pre_timing_v1<<<(unsigned)((F.n_nets + 127) / 128), 128, 0, s>>>(F, F.n_nets, P, Cd, Dg, sink_delay, net_cap);
        return cudaGetLastError();
    }
    unsigned grid = 1;
    cudaError_t e = tree_grid(k_pre_timing, n_chunks, &grid);
    if (e != cudaSuccess) return e;
    k_pre_timing<<<grid, TW * 32, 0, s>>>(F, chunks, n_chunks, P, Cd, Dg, sink_delay, net_cap);
    return cudaGetLastError();
}

}  // namespace gapla
