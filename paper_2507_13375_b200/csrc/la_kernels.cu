// Hand-written sm_100a kernels of the GAP-LA layer-assignment hot path.
//
//   k_pack_state / k_unpack_demand   a0: API-layout capacity/demand <-> packed planes
//   k_assign     (K4 + K5)           Alg. 3 getSubtreeCandidate + Alg. 4 traceBackSolution
//                                    (PAPER l.355-435), one warp per net of a batch
//   k_commit     (K8)                demand commit with int32 atomics (Alg. 2 input D, l.343)
//   k_elmore     (K6 + K7)           Elmore / downstream cap on the 3D RC trees (l.146, l.443-444)
//
// Bit-exactness contract: this translation unit is compiled with
// --fmad=false; every fp64 value is produced by the same expression tree, in the
// same operand order, as DESIGN §3 (O5, O6, O9) prescribes; no transcendental
// function runs on the device (Eq. (3) comes from host tables); cross-lane
// reductions are min/argmin only, with a total-order key.
#include <cuda_runtime.h>

#include "la_internal.h"

namespace gapla {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int AW = 4;            // warps per CTA of k_assign

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Eq. (3) marginal cost of one more unit on an element (reading R18):
// packed word w = ((d - c) << 1) | (c == 0); table over the clamped d - c (R20).
__device__ __forceinline__ double marginal(const DevGrid &G, int32_t w) {
    int delta = w >> 1;
    delta = min(max(delta, G.delta_lo), G.delta_hi);
    const double *M = (w & 1) ? G.Mzero : G.Mpos;
    return __ldg(M + (delta - G.delta_lo));
}

__device__ __forceinline__ int64_t wire_word(const DevGrid &G, int dtype, int l, int x, int y) {
    return dtype == 0 ? ((int64_t)y * (G.X - 1) + x) * G.LH + G.lidx[l]
                      : ((int64_t)x * (G.Y - 1) + y) * G.LV + G.lidx[l];
}

// Lowest coordinate of the unit edges of a node's parent run (ascending order, R23).
__device__ __forceinline__ int run_lo(uint8_t edir, int x, int y, int len) {
    switch (edir) {
        case 0: return x - len;   // parent is west: run from parent.x
        case 1: return x;
        case 2: return y - len;
        default: return y;
    }
}

__device__ void stage_tab(TechTab &T, const TechTab *src) {
    const double *s = reinterpret_cast<const double *>(src);
    double *d = reinterpret_cast<double *>(&T);
    for (int i = threadIdx.x; i < (int)(sizeof(TechTab) / sizeof(double)); i += blockDim.x) d[i] = s[i];
}

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

// ------------------------------------------------------------------ K4 + K5 --
struct WarpSm {
    double kap[MAXL];                                   // ViaCong per cut at this node
    double sA[MAXKIDS][MAXL], sB[MAXKIDS][MAXL], sC[MAXKIDS][MAXL];   // sons' O5 terms
    double pGp[MAXPAIRS], pG[MAXPAIRS], pK[MAXPAIRS];   // best span per (l, b) lane task
    uint32_t pjs[MAXPAIRS];
    uint8_t pl[MAXPAIRS], pb[MAXPAIRS], pt[MAXPAIRS];   // pt = 255: no feasible span
    int16_t goff[MAXL], gcnt[MAXL];
};

// One warp per net of the batch.  For every node (leaves first): lanes own
// (entry layer l, span bottom b) tasks and sweep the span top t upward,
// keeping each son's running argmin over [b, t] of cost' (Alg. 3 l.370-395);
// then one lane per layer picks the span by the key (G', t-b, b) (l.404),
// folds in the pin terms (l.4-7) and, for a non-root node, produces the
// parent-edge terms A, B, capb of DESIGN §3 O5 for every layer j of its edge.
// After the root, lane 0 walks the net top-down (Alg. 4).
__global__ void __launch_bounds__(AW * 32) k_assign(DevGrid G, DevForest F, DevScratch S, int64_t net_beg,
                                                    int64_t net_end) {
    __shared__ TechTab T;
    __shared__ WarpSm Wsm[AW];
    stage_tab(T, G.tab);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t net = net_beg + (int64_t)blockIdx.x * AW + warp;
    if (net >= net_end) return;
    WarpSm &w = Wsm[warp];
    const int L = G.L;
    const double INF = dinf();
    const int64_t n0 = F.net_node0[net], n1 = F.net_node0[net + 1];
    const int pdrv = F.net_pdrv[net];

    for (int64_t n = n0; n < n1; ++n) {
        const bool root = (n == n1 - 1);
        const uint32_t xy = F.xy[n];
        const int x = xy & 0xffff, y = xy >> 16;
        const int nk = F.nkid[n];
        const int nl = F.nl[n], nh = F.nh[n];
        const bool has_pins = nl != 255;
        const uint8_t ed = F.edir[n];
        const int dtype = ed <= 1 ? 0 : 1;
        const double urn = F.ur[n];

        // ViaCong per cut k at (x, y): W_VIA + (W_CONG * ofw[k]) * M (reading R11)
        if (lane < L - 1) {
            int32_t vw = G.via[((int64_t)y * G.X + x) * (L - 1) + lane];
            w.kap[lane] = G.W_VIA + (G.W_CONG * T.ofw[lane]) * marginal(G, vw);
        }
        for (int i = 0; i < nk; ++i) {
            const int64_t s = F.kid[n * 4 + i];
            if (lane < L) {
                w.sA[i][lane] = S.A[s * L + lane];
                w.sB[i][lane] = S.B[s * L + lane];
                w.sC[i][lane] = S.Cap[s * L + lane];
            }
        }
        // entry layers (R13, R15) and span bottoms b <= b0 (Alg. 3 l.10-12, R14)
        int cnt = 0;
        if (lane < L) {
            const bool ent = root ? (lane == pdrv) : (G.routable[lane] && G.dir[lane] == dtype);
            if (ent) cnt = (has_pins ? min(lane, nl) : lane) + 1;
        }
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += v;
        }
        const int P = __shfl_sync(FULL, inc, 31);
        if (lane < L) {
            w.goff[lane] = (int16_t)(inc - cnt);
            w.gcnt[lane] = (int16_t)cnt;
            for (int b = 0; b < cnt; ++b) {
                w.pl[inc - cnt + b] = (uint8_t)lane;
                w.pb[inc - cnt + b] = (uint8_t)b;
            }
        }
        __syncwarp();

        for (int p = lane; p < P; p += 32) {
            const int l = w.pl[p], b = w.pb[p];
            const int t0 = has_pins ? max(l, nh) : l;
            const double *VRl = &T.VR[l * MAXL];
            double V = 0.0;
            for (int k = b; k < t0; ++k) V = V + w.kap[k];
            int jb[MAXKIDS];
            double cpb[MAXKIDS], cbv[MAXKIDS], capv[MAXKIDS];
#pragma unroll
            for (int i = 0; i < MAXKIDS; ++i) { jb[i] = -1; cpb[i] = 0.0; cbv[i] = 0.0; capv[i] = 0.0; }
            // cost(l; s, j) = A + B*VR[l][j]; cost' = cost + B*ur_n; argmin of cost', ties -> lowest j
            auto cand = [&](int j) {
#pragma unroll
                for (int i = 0; i < MAXKIDS; ++i) {
                    if (i < nk) {
                        const double A = w.sA[i][j];
                        if (A < INF) {
                            const double Bv = w.sB[i][j];
                            const double cost = A + Bv * VRl[j];
                            const double cp = cost + Bv * urn;
                            if (isfinite(cp) && (jb[i] < 0 || cp < cpb[i])) {
                                jb[i] = j; cpb[i] = cp; cbv[i] = cost; capv[i] = w.sC[i][j];
                            }
                        }
                    }
                }
            };
            for (int j = b; j <= t0; ++j) cand(j);
            bool have = false;
            double bGp = 0.0, bG = 0.0, bK = 0.0;
            int bt = 255;
            uint32_t bjs = 0;
            for (int t = t0; t < L; ++t) {
                if (t > t0) {
                    V = V + w.kap[t - 1];
                    cand(t);
                }
                bool feas = true;
#pragma unroll
                for (int i = 0; i < MAXKIDS; ++i) if (i < nk && jb[i] < 0) feas = false;
                if (!feas) continue;
                double Gp = V, Gv = V, K = 0.0;
                uint32_t js = 0;
#pragma unroll
                for (int i = 0; i < MAXKIDS; ++i) {
                    if (i < nk) {
                        Gp = Gp + cpb[i];
                        Gv = Gv + cbv[i];
                        K = K + capv[i];
                        js |= (uint32_t)jb[i] << (8 * i);
                    }
                }
                if (!have || Gp < bGp) {   // same b: later t has larger t-b, loses ties
                    have = true; bGp = Gp; bG = Gv; bK = K; bt = t; bjs = js;
                }
            }
            w.pGp[p] = bGp; w.pG[p] = bG; w.pK[p] = bK; w.pjs[p] = bjs;
            w.pt[p] = have ? (uint8_t)bt : (uint8_t)255;
        }
        __syncwarp();

        if (lane < L) {
            const int l = lane;
            const int c = w.gcnt[l], g0 = w.goff[l];
            double A = INF, Bv = 0.0, Cp = 0.0;
            if (c > 0) {
                int best = -1;
                for (int q = g0; q < g0 + c; ++q) {
                    if (w.pt[q] == 255) continue;
                    if (best < 0) { best = q; continue; }
                    const double a = w.pGp[q], bb = w.pGp[best];
                    const int sq = w.pt[q] - w.pb[q], sbst = w.pt[best] - w.pb[best];
                    if (a < bb || (a == bb && (sq < sbst || (sq == sbst && w.pb[q] < w.pb[best])))) best = q;
                }
                if (best >= 0) {
                    // pin-via delay terms, Alg. 3 l.4-7 (sinks in input order; driver excluded)
                    double F0 = 0.0, C0 = 0.0;
                    const int q0 = F.sink0[n], qn = F.nsink[n];
                    for (int q = q0; q < q0 + qn; ++q) {
                        const double cq = F.p_cap[q];
                        F0 = F0 + F.p_w[q] * (cq * T.VR[F.p_layer[q] * MAXL + l]);
                        C0 = C0 + cq;
                    }
                    const double f = F0 + w.pG[best];
                    const double dlc = C0 + w.pK[best];
                    S.choice[n * L + l] = (uint16_t)(w.pb[best] | (w.pt[best] << 8));
                    S.entry[n * L + l] = w.pjs[best];
                    if (root) {
                        S.froot[net] = f;
                    } else if (f < INF) {
                        // O5 parent-edge terms of this node on layer l
                        const int len = F.len[n];
                        const int a = run_lo(ed, x, y, len);
                        double Sc = 0.0;
                        if (dtype == 0) {
                            const int32_t *wp = G.wH + ((int64_t)y * (G.X - 1) + a) * G.LH + G.lidx[l];
                            for (int i = 0; i < len; ++i) Sc = Sc + marginal(G, wp[(int64_t)i * G.LH]);
                        } else {
                            const int32_t *wp = G.wV + ((int64_t)x * (G.Y - 1) + a) * G.LV + G.lidx[l];
                            for (int i = 0; i < len; ++i) Sc = Sc + marginal(G, wp[(int64_t)i * G.LV]);
                        }
                        const double Rw = T.r[l] * (double)len;
                        const double Cw = T.c[l] * (double)len;
                        const double wd = F.wd[n];
                        A = ((f + wd * (Rw * (0.5 * Cw + dlc))) + G.W_CAP * Cw) + (G.W_CONG * T.ofw[l]) * Sc;
                        Bv = wd * (Cw + dlc);
                        Cp = Cw + dlc;
                    }
                } else if (root) {
                    S.froot[net] = INF;
                }
            }
            if (!root) {
                S.A[n * L + l] = A;
                S.B[n * L + l] = Bv;
                S.Cap[n * L + l] = Cp;
            }
        }
        __syncwarp();
    }

    // Alg. 4: root layer = driver pin layer (R13); top-down over the height order.
    if (lane == 0) {
        for (int64_t n = n1 - 1; n >= n0; --n) {
            int l;
            if (n == n1 - 1) { l = pdrv; S.lay[n] = (uint8_t)pdrv; }
            else l = S.lay[n];
            const uint16_t ch = S.choice[n * L + l];
            S.sb[n] = (uint8_t)(ch & 0xff);
            S.st[n] = (uint8_t)(ch >> 8);
            const uint32_t js = S.entry[n * L + l];
            const int nk = F.nkid[n];
            for (int i = 0; i < nk; ++i) S.lay[F.kid[n * 4 + i]] = (uint8_t)((js >> (8 * i)) & 0xff);
        }
    }
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
            for (int i = 0; i < len; ++i) atomicAdd(wp + (int64_t)i * G.LH, 2);
        } else {
            int32_t *wp = G.wV + ((int64_t)x * (G.Y - 1) + a) * G.LV + G.lidx[l];
            for (int i = 0; i < len; ++i) atomicAdd(wp + (int64_t)i * G.LV, 2);
        }
    }
    const int b = S.sb[n], t = S.st[n];
    int32_t *vp = G.via + ((int64_t)y * G.X + x) * (G.L - 1);
    for (int k = b; k < t; ++k) atomicAdd(vp + k, 2);
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
// Canonical fast Elmore form (DESIGN §3 O9), one thread per net.
__global__ void k_elmore(DevGrid G, DevForest F, DevScratch S, int64_t net_beg, int64_t net_end) {
    __shared__ TechTab T;
    stage_tab(T, G.tab);
    __syncthreads();
    const int64_t net = net_beg + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (net >= net_end) return;
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
    double Tk[MAXL];
    for (int64_t n = n1 - 1; n >= n0; --n) {
        const int ln = S.lay[n], b = S.sb[n], t = S.st[n];
        Tk[ln] = (n == n1 - 1) ? 0.0 : S.Tin[n];
        const int q0 = F.sink0[n], qn = F.nsink[n], nk = F.nkid[n];
        for (int k = ln; k < t; ++k) {
            const int j = k + 1;
            double acc = 0.0;
            for (int q = q0; q < q0 + qn; ++q) if (F.p_layer[q] >= j) acc = acc + F.p_cap[q];
            for (int i = 0; i < nk; ++i) {
                const int64_t s = F.kid[n * 4 + i];
                const int ls = S.lay[s];
                if (ls >= j) acc = acc + (T.c[ls] * (double)F.len[s] + S.Cd[s]);
            }
            Tk[k + 1] = Tk[k] + T.vr[k] * acc;
        }
        for (int k = ln; k > b; --k) {
            const int j = k - 1;
            double acc = 0.0;
            for (int q = q0; q < q0 + qn; ++q) if (F.p_layer[q] <= j) acc = acc + F.p_cap[q];
            for (int i = 0; i < nk; ++i) {
                const int64_t s = F.kid[n * 4 + i];
                const int ls = S.lay[s];
                if (ls <= j) acc = acc + (T.c[ls] * (double)F.len[s] + S.Cd[s]);
            }
            Tk[k - 1] = Tk[k] + T.vr[k - 1] * acc;
        }
        for (int q = q0; q < q0 + qn; ++q) S.sink_delay[F.p_orig[q]] = Tk[F.p_layer[q]];
        for (int i = 0; i < nk; ++i) {
            const int64_t s = F.kid[n * 4 + i];
            const int ls = S.lay[s], len = F.len[s];
            const double Cw = T.c[ls] * (double)len, Rw = T.r[ls] * (double)len;
            S.Tin[s] = Tk[ls] + Rw * (0.5 * Cw + S.Cd[s]);
        }
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

cudaError_t launch_assign(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t net_beg,
                          int64_t net_end, cudaStream_t s) {
    int64_t n = net_end - net_beg;
    if (n <= 0) return cudaSuccess;
    k_assign<<<nblk(n, AW), AW * 32, 0, s>>>(G, F, S, net_beg, net_end);
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

cudaError_t launch_elmore(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t net_beg,
                          int64_t net_end, cudaStream_t s) {
    int64_t n = net_end - net_beg;
    if (n <= 0) return cudaSuccess;
    k_elmore<<<nblk(n, 128), 128, 0, s>>>(G, F, S, net_beg, net_end);
    return cudaGetLastError();
}

}  // namespace gapla
