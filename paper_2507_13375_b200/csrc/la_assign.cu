// K4 + K5 (+ fused K8): Alg. 3 getSubtreeCandidate + Alg. 4 traceBackSolution
// for every net of one conflict-free batch, in ONE launch.
//
// Design ("k_assign"): the paper launches one thread per (node,
// layer) and one launch per tree level (Alg. 2, l.345-351).  On B200 that is
// launch- and latency-bound (~100 batches x tens of levels), so here:
//   * small nets (<= NS_MAX nodes, <= NP_MAX sinks, ~99% of nets): ONE WARP PER
//     NET.  The warp first gathers everything the DP reads from HBM -- node
//     records, sinks, the via-cut words of every node GCell (-> ViaCong kappa)
//     and the wire words of every parent run on every legal layer (-> the
//     congestion sum S) -- with all loads of the net in flight at once, into
//     shared memory.  The DP then runs entirely out of shared memory, node by
//     node in height order: lanes own (entry layer l, span bottom b) tasks and
//     sweep the span top t upward with each son's running argmin of cost'
//     (l.370-395); one lane per entry layer reduces by the key (G', t-b, b)
//     (l.404).  Backtrack is level-parallel over lanes (l.418-435).
//   * big nets: ONE CTA PER NET, the same node routine with DP state in a
//     global (L2-resident) scratch, nodes of one height level spread over the
//     CTA's warps, one __syncthreads per level.
//   * the demand commit of the batch (K8) is fused at the end when there is a
//     single rank: batches are conflict-free, so no net of the batch reads what
//     another commits.
// Bit-exactness: compiled with --fmad=false; expression trees and operand order
// exactly as DESIGN §3 O5/O6; min/argmin only across lanes, never sums.
#include <cuda_runtime.h>

#include "la_device.cuh"
#include "la_internal.h"

namespace gapla {
namespace {

// ---------------------------------------------------------------- layouts --
// Per-warp shared-memory layout of the small path (byte offsets).
struct WLay {
    int wd, ur, kap, A, B, C, pcap, pw, pGp, pG, pK;        // double
    int xy, len, entry, pjs;                                // uint32
    int choice, nsink, sink0;                               // uint16
    int edir, nkid, nl, nh, kid, height, lay, sb, st, player, pl, pb, pt;   // uint8
    int bytes;
};

__host__ __device__ inline WLay wlayout(int L, int LD, int MP) {
    WLay w;
    int o = 0;
    auto take = [&](int bytes) { int r = o; o += (bytes + 7) & ~7; return r; };
    const int NS = NS_MAX, NP = NP_MAX;
    w.wd = take(8 * NS); w.ur = take(8 * NS); w.kap = take(8 * NS * (L - 1));
    w.A = take(8 * NS * LD); w.B = take(8 * NS * LD); w.C = take(8 * NS * LD);
    w.pcap = take(8 * NP); w.pw = take(8 * NP);
    w.pGp = take(8 * MP); w.pG = take(8 * MP); w.pK = take(8 * MP);
    w.xy = take(4 * NS); w.len = take(4 * NS); w.entry = take(4 * NS * LD); w.pjs = take(4 * MP);
    w.choice = take(2 * NS * LD); w.nsink = take(2 * NS); w.sink0 = take(2 * NS);
    w.edir = take(NS); w.nkid = take(NS); w.nl = take(NS); w.nh = take(NS); w.kid = take(4 * NS);
    w.height = take(NS); w.lay = take(NS); w.sb = take(NS); w.st = take(NS); w.player = take(NP);
    w.pl = take(MP); w.pb = take(MP); w.pt = take(MP);
    w.bytes = o;
    return w;
}

constexpr int MAX_LEVELS = 512;

struct Shared {          // per-CTA static shared memory
    TechTab T;
    uint8_t dir[MAXL], routable[MAXL], lidx[MAXL];
    uint16_t lvl[MAX_LEVELS + 1];   // big path: level boundaries
    int nlvl;
};

// Per-warp task scratch of the pair phase (both paths).
struct PairScratch {
    double *Gp, *G, *K;
    uint32_t *js;
    uint8_t *l, *b, *t;
};

__device__ __forceinline__ PairScratch pair_scratch(char *base, const WLay &w) {
    return PairScratch{reinterpret_cast<double *>(base + w.pGp), reinterpret_cast<double *>(base + w.pG),
                       reinterpret_cast<double *>(base + w.pK), reinterpret_cast<uint32_t *>(base + w.pjs),
                       reinterpret_cast<uint8_t *>(base + w.pl), reinterpret_cast<uint8_t *>(base + w.pb),
                       reinterpret_cast<uint8_t *>(base + w.pt)};
}

// ------------------------------------------------------------- net views --
// Node-local view of one net: everything the node routine reads or writes,
// in shared memory (small path) or global memory (big path).
struct SmallView {
    const uint32_t *xy_; const int32_t *len_; const uint16_t *sink0_, *nsink_;
    const uint8_t *edir_, *nkid_, *nl_, *nh_, *kid_;
    const double *wd_, *ur_, *kap_;
    double *A_, *B_, *C_;
    uint16_t *choice_; uint32_t *entry_;
    const uint8_t *player_; const double *pcap_, *pw_;
    int Lm1, LD;
    __device__ int nkid(int i) const { return nkid_[i]; }
    __device__ int kid(int i, int k) const { return kid_[i * 4 + k]; }
    __device__ int nl(int i) const { return nl_[i]; }
    __device__ int nh(int i) const { return nh_[i]; }
    __device__ int edir(int i) const { return edir_[i]; }
    __device__ double ur(int i) const { return ur_[i]; }
    __device__ double wd(int i) const { return wd_[i]; }
    __device__ int len(int i) const { return len_[i]; }
    __device__ const double *kap(int i) const { return kap_ + i * Lm1; }
    __device__ int sbeg(int i) const { return sink0_[i]; }
    __device__ int scnt(int i) const { return nsink_[i]; }
    __device__ double pcap(int q) const { return pcap_[q]; }
    __device__ double pw(int q) const { return pw_[q]; }
    __device__ int player(int q) const { return player_[q]; }
};

struct BigView {
    const DevForest *F; int64_t n0;
    const double *kap_; double *A_, *B_, *C_;
    uint16_t *choice_; uint32_t *entry_;
    int Lm1, LD;
    __device__ int nkid(int i) const { return F->nkid[n0 + i]; }
    __device__ int kid(int i, int k) const { return (int)(F->kid[(n0 + i) * 4 + k] - n0); }
    __device__ int nl(int i) const { return F->nl[n0 + i]; }
    __device__ int nh(int i) const { return F->nh[n0 + i]; }
    __device__ int edir(int i) const { return F->edir[n0 + i]; }
    __device__ double ur(int i) const { return F->ur[n0 + i]; }
    __device__ double wd(int i) const { return F->wd[n0 + i]; }
    __device__ int len(int i) const { return F->len[n0 + i]; }
    __device__ const double *kap(int i) const { return kap_ + (int64_t)i * Lm1; }
    __device__ int sbeg(int i) const { return F->sink0[n0 + i]; }
    __device__ int scnt(int i) const { return F->nsink[n0 + i]; }
    __device__ double pcap(int q) const { return F->p_cap[q]; }
    __device__ double pw(int q) const { return F->p_w[q]; }
    __device__ int player(int q) const { return F->p_layer[q]; }
};

// ------------------------------------------------------------ node routine --
// Final step for entry layer l of node i once its best span is known: pin terms
// (Alg. 3 l.4-7), f and dlc (l.405), choice / entry (l.406-408), and for a
// non-root node the O5 parent-edge terms A, B, capb on layer l (its edge layer).
template <class VW>
__device__ __forceinline__ void finish_layer(const VW &v, const Shared &sh, const DevGrid &G, int i, bool root, int l,
                                             bool have, double Gv, double K, int b, int t, uint32_t js,
                                             double *froot) {
    const int slot = root ? 0 : sh.lidx[l];
    const int64_t at = (int64_t)i * v.LD + slot;
    if (!have) {
        if (root) *froot = dinf();
        else v.A_[at] = dinf();
        return;
    }
    double F0 = 0.0, C0 = 0.0;
    const int q0 = v.sbeg(i), qn = v.scnt(i);
    for (int q = q0; q < q0 + qn; ++q) {
        const double cq = v.pcap(q);
        F0 = F0 + v.pw(q) * (cq * sh.T.VR[v.player(q) * MAXL + l]);
        C0 = C0 + cq;
    }
    const double f = F0 + Gv;
    const double dlc = C0 + K;
    v.choice_[at] = (uint16_t)(b | (t << 8));
    v.entry_[at] = js;
    if (root) {
        *froot = f;
        return;
    }
    const int len = v.len(i);
    const double Sc = v.A_[at];                         // congestion sum gathered up front
    const double Rw = sh.T.r[l] * (double)len;
    const double Cw = sh.T.c[l] * (double)len;
    const double wd = v.wd(i);
    v.A_[at] = ((f + wd * (Rw * (0.5 * Cw + dlc))) + G.W_CAP * Cw) + (G.W_CONG * sh.T.ofw[l]) * Sc;
    v.B_[at] = wd * (Cw + dlc);
    v.C_[at] = Cw + dlc;
}

// Alg. 3 for node i, all entry layers, executed by one warp (lanes 0..31).
template <class VW>
__device__ void node_dp(const VW &v, const Shared &sh, const DevGrid &G, const PairScratch &ps, int i, bool root,
                        int pdrv, double *froot, int lane) {
    const int L = G.L;
    const int nk = v.nkid(i);
    const int nl = v.nl(i), nh = v.nh(i);
    const bool has_pins = nl != 255;
    const int dtype = v.edir(i) <= 1 ? 0 : 1;
    const double *kap = v.kap(i);
    // entry layers (R13 root: driver pin layer only; R15 otherwise: legal layers of
    // the parent edge) and the number of span bottoms b <= b0 (Alg. 3 l.10-12, R14)
    int cnt = 0;
    if (lane < L) {
        const bool ent = root ? (lane == pdrv) : (sh.routable[lane] && sh.dir[lane] == dtype);
        if (ent) cnt = (has_pins ? min(lane, nl) : lane) + 1;
    }
    if (nk == 0) {
        // Leaf: no son terms, G' = V(b, t) >= V(b0, t0) for every admissible span
        // (kappa >= 0 and rounded addition is monotone), and the key prefers the
        // smaller span on ties -> the choice is (b0, t0) with G = V(b0, t0).
        if (cnt > 0) {
            const int l = lane, b0 = cnt - 1, t0 = has_pins ? max(l, nh) : l;
            double V = 0.0;
            for (int k = b0; k < t0; ++k) V = V + kap[k];
            finish_layer(v, sh, G, i, root, l, true, V, 0.0, b0, t0, 0u, froot);
        }
        return;
    }
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(FULL_MASK, inc, o);
        if (lane >= o) inc += x;
    }
    const int P = __shfl_sync(FULL_MASK, inc, 31);
    for (int b = 0; b < cnt; ++b) {
        ps.l[inc - cnt + b] = (uint8_t)lane;
        ps.b[inc - cnt + b] = (uint8_t)b;
    }
    int kid[MAXKIDS], kdt[MAXKIDS];
#pragma unroll
    for (int k = 0; k < MAXKIDS; ++k) {
        kid[k] = k < nk ? v.kid(i, k) : 0;
        kdt[k] = k < nk ? (v.edir(kid[k]) <= 1 ? 0 : 1) : 0;
    }
    const double urn = v.ur(i);
    __syncwarp();

    for (int p = lane; p < P; p += 32) {
        const int l = ps.l[p], b = ps.b[p];
        const int t0 = has_pins ? max(l, nh) : l;
        const double *VRl = &sh.T.VR[l * MAXL];
        double V = 0.0;
        for (int k = b; k < t0; ++k) V = V + kap[k];
        int jb[MAXKIDS];
        double cpb[MAXKIDS], cbv[MAXKIDS], capv[MAXKIDS];
#pragma unroll
        for (int k = 0; k < MAXKIDS; ++k) { jb[k] = -1; cpb[k] = 0.0; cbv[k] = 0.0; capv[k] = 0.0; }
        // cost(l; s, j) = A + B*VR[l][j]; cost' = cost + B*ur_n; son argmin of cost', ties -> lowest j
        auto cand = [&](int j) {
            const bool rj = sh.routable[j];
            const int dj = sh.dir[j], sj = sh.lidx[j];
#pragma unroll
            for (int k = 0; k < MAXKIDS; ++k) {
                if (k < nk && rj && dj == kdt[k]) {
                    const int64_t at = (int64_t)kid[k] * v.LD + sj;
                    const double A = v.A_[at];
                    if (A < dinf()) {
                        const double Bv = v.B_[at];
                        const double cost = A + Bv * VRl[j];
                        const double cp = cost + Bv * urn;
                        if (isfinite(cp) && (jb[k] < 0 || cp < cpb[k])) {
                            jb[k] = j; cpb[k] = cp; cbv[k] = cost; capv[k] = v.C_[at];
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
                V = V + kap[t - 1];
                cand(t);
            }
            bool feas = true;
#pragma unroll
            for (int k = 0; k < MAXKIDS; ++k) if (k < nk && jb[k] < 0) feas = false;
            if (!feas) continue;
            double Gp = V, Gv = V, K = 0.0;
            uint32_t js = 0;
#pragma unroll
            for (int k = 0; k < MAXKIDS; ++k) {
                if (k < nk) {
                    Gp = Gp + cpb[k];
                    Gv = Gv + cbv[k];
                    K = K + capv[k];
                    js |= (uint32_t)jb[k] << (8 * k);
                }
            }
            if (!have || Gp < bGp) {        // same b: a later t has a larger t-b and loses ties
                have = true; bGp = Gp; bG = Gv; bK = K; bt = t; bjs = js;
            }
        }
        ps.Gp[p] = bGp; ps.G[p] = bG; ps.K[p] = bK; ps.js[p] = bjs;
        ps.t[p] = have ? (uint8_t)bt : (uint8_t)255;
    }
    __syncwarp();
    if (cnt > 0) {
        const int l = lane, g0 = inc - cnt;
        int best = -1;
        for (int q = g0; q < g0 + cnt; ++q) {
            if (ps.t[q] == 255) continue;
            if (best < 0) { best = q; continue; }
            const double a = ps.Gp[q], c = ps.Gp[best];
            const int sq = ps.t[q] - ps.b[q], sbst = ps.t[best] - ps.b[best];
            if (a < c || (a == c && (sq < sbst || (sq == sbst && ps.b[q] < ps.b[best])))) best = q;
        }
        if (best >= 0)
            finish_layer(v, sh, G, i, root, l, true, ps.G[best], ps.K[best], ps.b[best], ps.t[best], ps.js[best],
                         froot);
        else
            finish_layer(v, sh, G, i, root, l, false, 0.0, 0.0, 0, 0, 0u, froot);
    }
}

// Congestion sum S of node i's parent run on the layer with slot s of its direction:
// ((m1 + m2) + ...) + m_len in ascending coordinate, loads issued 4 at a time.
__device__ __forceinline__ double run_sum(const DevGrid &G, int dtype, int lslot, int x, int y, int edir, int len) {
    const int a = run_lo(edir, x, y, len);
    const int32_t *wp;
    int64_t stride;
    if (dtype == 0) { wp = G.wH + ((int64_t)y * (G.X - 1) + a) * G.LH + lslot; stride = G.LH; }
    else { wp = G.wV + ((int64_t)x * (G.Y - 1) + a) * G.LV + lslot; stride = G.LV; }
    double Sc = 0.0;
    int e = 0;
    for (; e + 4 <= len; e += 4) {
        const int32_t w0 = __ldcg(wp + (e + 0) * stride), w1 = __ldcg(wp + (e + 1) * stride);
        const int32_t w2 = __ldcg(wp + (e + 2) * stride), w3 = __ldcg(wp + (e + 3) * stride);
        const double m0 = marginal(G, w0), m1 = marginal(G, w1), m2 = marginal(G, w2), m3 = marginal(G, w3);
        Sc = Sc + m0; Sc = Sc + m1; Sc = Sc + m2; Sc = Sc + m3;
    }
    for (; e < len; ++e) Sc = Sc + marginal(G, __ldcg(wp + e * stride));
    return Sc;
}

__device__ __forceinline__ double via_kappa(const DevGrid &G, const Shared &sh, uint32_t xy, int k) {
    const int x = xy & 0xffff, y = xy >> 16;
    const int32_t w = __ldcg(G.via + ((int64_t)y * G.X + x) * (G.L - 1) + k);
    return G.W_VIA + (G.W_CONG * sh.T.ofw[k]) * marginal(G, w);   // ViaCong, reading R11
}

// Fused K8 for node n: +1 per unit edge of its parent run on its layer, +1 per via cut.
__device__ __forceinline__ void commit_node(const DevGrid &G, uint32_t xy, int edir, int len, int l, int b, int t) {
    const int x = xy & 0xffff, y = xy >> 16;
    if (edir != NO_DIR) {
        const int a = run_lo(edir, x, y, len);
        if (edir <= 1) {
            int32_t *wp = G.wH + ((int64_t)y * (G.X - 1) + a) * G.LH + G.lidx[l];
            for (int e = 0; e < len; ++e) atomicAdd(wp + (int64_t)e * G.LH, 2);
        } else {
            int32_t *wp = G.wV + ((int64_t)x * (G.Y - 1) + a) * G.LV + G.lidx[l];
            for (int e = 0; e < len; ++e) atomicAdd(wp + (int64_t)e * G.LV, 2);
        }
    }
    int32_t *vp = G.via + ((int64_t)y * G.X + x) * (G.L - 1);
    for (int k = b; k < t; ++k) atomicAdd(vp + k, 2);
}

// ------------------------------------------------------------------ kernel --
__global__ void __launch_bounds__(ASSIGN_WARPS * 32) k_assign(DevGrid G, DevForest F, DevScratch S, AssignLaunch a) {
    __shared__ Shared sh;
    extern __shared__ __align__(16) char dyn[];
    stage_tab(sh.T, G.tab);
    if (threadIdx.x < MAXL) {
        sh.dir[threadIdx.x] = G.dir[threadIdx.x];
        sh.routable[threadIdx.x] = G.routable[threadIdx.x];
        sh.lidx[threadIdx.x] = (uint8_t)G.lidx[threadIdx.x];
    }
    __syncthreads();
    const int L = G.L, Lm1 = L - 1, LD = a.LD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const WLay wl = wlayout(L, LD, a.MP);
    char *wbase = dyn + warp * wl.bytes;
    const PairScratch ps = pair_scratch(wbase, wl);

    if ((int64_t)blockIdx.x < a.nbig) {
        // =========================== big path: one CTA per net ===========================
        const int64_t net = a.net_beg + blockIdx.x;
        const int64_t n0 = F.net_node0[net], n1 = F.net_node0[net + 1];
        const int nn = (int)(n1 - n0);
        const int pdrv = F.net_pdrv[net];
        const int64_t sbase = n0 - a.node_base;
        BigView v{&F, n0, S.bkap + sbase * Lm1, S.bA + sbase * LD, S.bB + sbase * LD, S.bC + sbase * LD,
                  S.bchoice + sbase * LD, S.bentry + sbase * LD, Lm1, LD};
        // gather kappa and S for all nodes (all loads of the net in flight)
        for (int idx = threadIdx.x; idx < nn * Lm1; idx += blockDim.x) {
            const int i = idx / Lm1, k = idx - i * Lm1;
            S.bkap[(sbase + i) * Lm1 + k] = via_kappa(G, sh, F.xy[n0 + i], k);
        }
        for (int idx = threadIdx.x; idx < nn * LD; idx += blockDim.x) {
            const int i = idx / LD, s = idx - i * LD;
            const int ed = F.edir[n0 + i];
            if (ed == NO_DIR) continue;
            const int dt = ed <= 1 ? 0 : 1;
            if (s >= (dt == 0 ? G.LH : G.LV)) continue;
            const uint32_t xy = F.xy[n0 + i];
            S.bA[(sbase + i) * LD + s] = run_sum(G, dt, s, xy & 0xffff, xy >> 16, ed, F.len[n0 + i]);
        }
        if (threadIdx.x == 0) {           // level boundaries (nodes are height-sorted)
            int nlv = 0, prev = -1;
            for (int i = 0; i < nn && nlv < MAX_LEVELS; ++i) {
                const int h = F.height[n0 + i];
                if (h != prev) { sh.lvl[nlv++] = (uint16_t)i; prev = h; }
            }
            sh.lvl[nlv] = (uint16_t)nn;
            sh.nlvl = nlv;
        }
        __syncthreads();
        const int nlv = sh.nlvl;
        for (int lv = 0; lv < nlv; ++lv) {
            for (int i = sh.lvl[lv] + warp; i < sh.lvl[lv + 1]; i += ASSIGN_WARPS)
                node_dp(v, sh, G, ps, i, i == nn - 1, pdrv, S.froot + net, lane);
            __syncthreads();
        }
        // Alg. 4, level-parallel from the root
        if (threadIdx.x == 0) S.lay[n1 - 1] = (uint8_t)pdrv;
        __syncthreads();
        for (int lv = nlv - 1; lv >= 0; --lv) {
            for (int i = sh.lvl[lv] + threadIdx.x; i < sh.lvl[lv + 1]; i += blockDim.x) {
                const int64_t n = n0 + i;
                const int l = S.lay[n];
                const int slot = (i == nn - 1) ? 0 : sh.lidx[l];
                const uint16_t ch = v.choice_[(int64_t)i * LD + slot];
                const int b = ch & 0xff, t = ch >> 8;
                S.sb[n] = (uint8_t)b;
                S.st[n] = (uint8_t)t;
                const uint32_t js = v.entry_[(int64_t)i * LD + slot];
                const int nk = F.nkid[n];
                for (int k = 0; k < nk; ++k) S.lay[F.kid[n * 4 + k]] = (uint8_t)((js >> (8 * k)) & 0xff);
                if (a.commit) commit_node(G, F.xy[n], F.edir[n], F.len[n], l, b, t);
            }
            __syncthreads();
        }
        return;
    }

    // ============================= small path: one warp per net =============================
    const int64_t net = a.net_beg + a.nbig + ((int64_t)blockIdx.x - a.nbig) * ASSIGN_WARPS + warp;
    if (net >= a.net_end) return;
    const int64_t n0 = F.net_node0[net], n1 = F.net_node0[net + 1];
    const int nn = (int)(n1 - n0);
    const int pdrv = F.net_pdrv[net];
    uint32_t *xy = reinterpret_cast<uint32_t *>(wbase + wl.xy);
    int32_t *len = reinterpret_cast<int32_t *>(wbase + wl.len);
    uint16_t *nsink = reinterpret_cast<uint16_t *>(wbase + wl.nsink), *sink0 = reinterpret_cast<uint16_t *>(wbase + wl.sink0);
    uint8_t *edir = reinterpret_cast<uint8_t *>(wbase + wl.edir), *nkid = reinterpret_cast<uint8_t *>(wbase + wl.nkid);
    uint8_t *nl = reinterpret_cast<uint8_t *>(wbase + wl.nl), *nh = reinterpret_cast<uint8_t *>(wbase + wl.nh);
    uint8_t *kid = reinterpret_cast<uint8_t *>(wbase + wl.kid), *height = reinterpret_cast<uint8_t *>(wbase + wl.height);
    uint8_t *lay = reinterpret_cast<uint8_t *>(wbase + wl.lay), *sb = reinterpret_cast<uint8_t *>(wbase + wl.sb);
    uint8_t *st = reinterpret_cast<uint8_t *>(wbase + wl.st), *player = reinterpret_cast<uint8_t *>(wbase + wl.player);
    double *wd = reinterpret_cast<double *>(wbase + wl.wd), *ur = reinterpret_cast<double *>(wbase + wl.ur);
    double *kap = reinterpret_cast<double *>(wbase + wl.kap);
    double *A = reinterpret_cast<double *>(wbase + wl.A), *B = reinterpret_cast<double *>(wbase + wl.B);
    double *C = reinterpret_cast<double *>(wbase + wl.C);
    double *pcap = reinterpret_cast<double *>(wbase + wl.pcap), *pw = reinterpret_cast<double *>(wbase + wl.pw);
    uint16_t *choice = reinterpret_cast<uint16_t *>(wbase + wl.choice);
    uint32_t *entry = reinterpret_cast<uint32_t *>(wbase + wl.entry);

    // ---- gather 1: node records and sinks
    const int q_base = F.sink0[n0];
    for (int i = lane; i < nn; i += 32) {
        const int64_t n = n0 + i;
        xy[i] = F.xy[n];
        len[i] = F.len[n];
        edir[i] = F.edir[n];
        nkid[i] = F.nkid[n];
        nl[i] = F.nl[n];
        nh[i] = F.nh[n];
        height[i] = F.height[n];
        nsink[i] = F.nsink[n];
        sink0[i] = (uint16_t)(F.sink0[n] - q_base);
        wd[i] = F.wd[n];
        ur[i] = F.ur[n];
        const int4 k4 = *reinterpret_cast<const int4 *>(F.kid + n * 4);
        kid[i * 4 + 0] = (uint8_t)(k4.x - n0);
        kid[i * 4 + 1] = (uint8_t)(k4.y - n0);
        kid[i * 4 + 2] = (uint8_t)(k4.z - n0);
        kid[i * 4 + 3] = (uint8_t)(k4.w - n0);
    }
    const int ns_net = F.sink0[n1 - 1] + F.nsink[n1 - 1] - q_base;
    for (int q = lane; q < ns_net; q += 32) {
        player[q] = F.p_layer[q_base + q];
        pcap[q] = F.p_cap[q_base + q];
        pw[q] = F.p_w[q_base + q];
    }
    __syncwarp();
    // ---- gather 2: kappa per (node, cut) and S per (non-root node, layer slot)
    for (int idx = lane; idx < nn * Lm1; idx += 32) {
        const int i = idx / Lm1, k = idx - i * Lm1;
        kap[idx] = via_kappa(G, sh, xy[i], k);
    }
    for (int idx = lane; idx < nn * LD; idx += 32) {
        const int i = idx / LD, s = idx - i * LD;
        const int ed = edir[i];
        if (ed == NO_DIR) continue;
        const int dt = ed <= 1 ? 0 : 1;
        if (s >= (dt == 0 ? G.LH : G.LV)) continue;
        A[idx] = run_sum(G, dt, s, xy[i] & 0xffff, xy[i] >> 16, ed, len[i]);
    }
    __syncwarp();
    // ---- Alg. 3, nodes in height order (children before parents)
    SmallView v{xy, len, sink0, nsink, edir, nkid, nl, nh, kid, wd, ur, kap, A, B, C, choice, entry,
                player, pcap, pw, Lm1, LD};
    double froot = 0.0;
    for (int i = 0; i < nn; ++i) {
        node_dp(v, sh, G, ps, i, i == nn - 1, pdrv, &froot, lane);
        __syncwarp();
    }
    // root entry layer has a single lane; broadcast its f
    {
        const int src = pdrv;   // lane that finished the root's only entry layer
        froot = __shfl_sync(FULL_MASK, froot, src);
        if (lane == 0) S.froot[net] = froot;
    }
    // ---- Alg. 4, level-parallel from the root (root entry = driver pin layer, R13)
    if (lane == 0) lay[nn - 1] = (uint8_t)pdrv;
    __syncwarp();
    int hi = nn - 1;
    while (hi >= 0) {
        const int h = height[hi];
        int lo = hi;
        while (lo > 0 && height[lo - 1] == h) --lo;
        for (int i = lo + lane; i <= hi; i += 32) {
            const int l = lay[i];
            const int slot = (i == nn - 1) ? 0 : sh.lidx[l];
            const uint16_t ch = choice[i * LD + slot];
            sb[i] = (uint8_t)(ch & 0xff);
            st[i] = (uint8_t)(ch >> 8);
            const uint32_t js = entry[i * LD + slot];
            for (int k = 0; k < nkid[i]; ++k) lay[kid[i * 4 + k]] = (uint8_t)((js >> (8 * k)) & 0xff);
        }
        __syncwarp();
        hi = lo - 1;
    }
    for (int i = lane; i < nn; i += 32) {
        S.lay[n0 + i] = lay[i];
        S.sb[n0 + i] = sb[i];
        S.st[n0 + i] = st[i];
        if (a.commit) commit_node(G, xy[i], edir[i], len[i], lay[i], sb[i], st[i]);
    }
}

}  // namespace

size_t assign_smem_bytes(int L, int LD, int MP) { return (size_t)ASSIGN_WARPS * wlayout(L, LD, MP).bytes; }

cudaError_t launch_assign(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a,
                          cudaStream_t s) {
    const int64_t n = a.net_end - a.net_beg;
    if (n <= 0) return cudaSuccess;
    const size_t smem = assign_smem_bytes(G.L, a.LD, a.MP);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    const int64_t nsmall = n - a.nbig;
    const int64_t grid = a.nbig + (nsmall + ASSIGN_WARPS - 1) / ASSIGN_WARPS;
    k_assign<<<(unsigned)grid, ASSIGN_WARPS * 32, smem, s>>>(G, F, S, a);
    return cudaGetLastError();
}

}  // namespace gapla
