// K4 + K5 + fused K8: Alg. 3 getSubtreeCandidate + Alg. 4 traceBackSolution
// and the demand commit, for every net, as ONE kernel.
//
// Design (DESIGN §5 "k_assign", §2):
//   * Work items.  The forest is batch-major; items are, in that
//     order, either ONE big net (more than NS nodes or NP sinks) run by the whole
//     CTA, or up to ASSIGN_WARPS consecutive small nets, one warp each.  CTAs are
//     persistent and grab items with an atomic ticket.
//   * Batch mode (la_assign_batch): the items of one conflict-free batch.
//     Dataflow mode (la_assign_all, one GPU): ALL items in one cooperative launch;
//     a net waits until its per-net count of unfinished predecessors (the
//     conflict DAG) is 0, and after its commit releases its
//     successors.  Items are taken in a topological order, so every waited-on
//     net is held by a running CTA: no deadlock.
//   * Per net: (1) gather everything the DP reads from HBM -- node records,
//     sinks, the via-cut words of every node GCell and the congestion sum S of
//     every parent run on every legal layer -- with all loads in flight at once,
//     into shared memory; (2) leaves, all at once, lanes over (leaf, entry
//     layer); (3) internal nodes in height order, one warp per node: per-son
//     candidate table cost'(l; s, j) for all (entry layer, son layer) pairs,
//     lanes over (entry layer l, span-bottom group) sweep the span top t upward
//     with each son's running argmin (Alg. 3 l.370-395), a segmented shuffle
//     argmin by the key (G', t-b, b) (l.404, reading R21) picks each entry
//     layer's span; (4) level-parallel backtrack (Alg. 4); (5) decisions to HBM
//     and the integer-atomic demand commit (O8).
// Bit-exactness: compiled with --fmad=false; every fp64 value is the DESIGN §3
// expression tree in operand order; cross-lane reductions are min/argmin only.
#include <cuda_runtime.h>

#include "la_device.cuh"
#include "la_internal.h"

namespace gapla {
namespace {

// ---------------------------------------------------------------- layouts --
// One net's DP state (NS nodes, NP sinks), as byte offsets from a base.
struct NetLay {
    int wd, ur, A, C, pcap, pw, froot;                      // double
    int xy, vw;                                              // 32-bit
    int len, height, nsink, sink0, kid, entry;               // 16-bit
    int edir, nkid, nl, nh, choice, lay, sb, st, player;     // 8-bit
    int bytes;
};

__host__ __device__ inline NetLay net_layout(int NS, int NP, int L, int LD) {
    NetLay w;
    int o = 0;
    auto take = [&](int bytes) { int r = o; o += (bytes + 7) & ~7; return r; };
    w.wd = take(8 * NS); w.ur = take(8 * NS); w.A = take(8 * NS * LD); w.C = take(8 * NS * LD);
    w.pcap = take(8 * NP); w.pw = take(8 * NP); w.froot = take(8);
    w.xy = take(4 * NS); w.vw = take(4 * NS * (L - 1));
    w.len = take(2 * NS); w.height = take(2 * NS); w.nsink = take(2 * NS); w.sink0 = take(2 * NS);
    w.kid = take(2 * NS * MAXKIDS); w.entry = take(2 * NS * LD);
    w.edir = take(NS); w.nkid = take(NS); w.nl = take(NS); w.nh = take(NS); w.choice = take(NS * LD);
    w.lay = take(NS); w.sb = take(NS); w.st = take(NS); w.player = take(NP);
    w.bytes = (o + 15) & ~15;
    return w;
}

// Per-warp scratch of the node routine.
struct WarpLay {
    int CP, kap, map, bytes;
};

__host__ __device__ inline WarpLay warp_layout(int L, int LD) {
    WarpLay w;
    w.CP = 0;
    w.kap = w.CP + 8 * MAXKIDS * LD * LD;
    w.map = w.kap + 8 * (L - 1);
    w.bytes = (w.map + 2 * 32 + 15) & ~15;
    return w;
}

struct NetBuf {
    double *wd, *ur, *A, *C, *pcap, *pw, *froot;
    uint32_t *xy;
    int32_t *vw;
    uint16_t *len, *height, *nsink, *sink0, *kid, *entry;
    uint8_t *edir, *nkid, *nl, *nh, *choice, *lay, *sb, *st, *player;
};

__device__ __forceinline__ NetBuf net_buf(char *b, const NetLay &w) {
    NetBuf n;
    n.wd = (double *)(b + w.wd); n.ur = (double *)(b + w.ur); n.A = (double *)(b + w.A); n.C = (double *)(b + w.C);
    n.pcap = (double *)(b + w.pcap); n.pw = (double *)(b + w.pw); n.froot = (double *)(b + w.froot);
    n.xy = (uint32_t *)(b + w.xy); n.vw = (int32_t *)(b + w.vw);
    n.len = (uint16_t *)(b + w.len); n.height = (uint16_t *)(b + w.height); n.nsink = (uint16_t *)(b + w.nsink);
    n.sink0 = (uint16_t *)(b + w.sink0); n.kid = (uint16_t *)(b + w.kid); n.entry = (uint16_t *)(b + w.entry);
    n.edir = (uint8_t *)(b + w.edir); n.nkid = (uint8_t *)(b + w.nkid); n.nl = (uint8_t *)(b + w.nl);
    n.nh = (uint8_t *)(b + w.nh); n.choice = (uint8_t *)(b + w.choice); n.lay = (uint8_t *)(b + w.lay);
    n.sb = (uint8_t *)(b + w.sb); n.st = (uint8_t *)(b + w.st); n.player = (uint8_t *)(b + w.player);
    return n;
}

struct WarpBuf {
    double *CP, *kap;
    uint16_t *map;
};

struct Shared {          // per-CTA static shared memory
    TechTab T;
    uint8_t dir[MAXL], routable[MAXL], lidx[MAXL];
    uint8_t lay_of[2][MAXL];   // layer of slot s in direction d
    int ndir[2];               // legal layers per direction
    int64_t item;
    int lo, hi;                // big path: current level [lo, hi)
};

// Context of one net inside the node routines.
struct NetCtx {
    NetBuf nb;
    int L, LD, nn;
};

__device__ __forceinline__ double kappa_w(const DevGrid &G, const Shared &sh, int32_t w, int k) {
    return G.W_VIA + (G.W_CONG * sh.T.ofw[k]) * marginal(G, w);    // ViaCong, reading R11
}

// -------------------------------------------------------- node finishing --
// Entry layer l (slot `slot`) of node i once its span is chosen: pin terms
// (Alg. 3 l.4-7), f and dlc (l.405), choice / entry (l.406-408); for a non-root
// node also the O5 parent-edge terms A and capb on layer l (its edge layer).
__device__ __forceinline__ void finish_layer(const NetCtx &c, const Shared &sh, const DevGrid &G, int i, bool root,
                                             int l, int slot, bool have, double Gv, double K, int b, int t,
                                             uint32_t ent) {
    const NetBuf &nb = c.nb;
    const int at = i * c.LD + slot;
    if (!have) {
        if (root) *nb.froot = dinf();
        else nb.A[at] = dinf();
        return;
    }
    double F0 = 0.0, C0 = 0.0;
    const int q0 = nb.sink0[i], qn = nb.nsink[i];
    for (int q = q0; q < q0 + qn; ++q) {
        const double cq = nb.pcap[q];
        F0 = F0 + nb.pw[q] * (cq * sh.T.VR[nb.player[q] * MAXL + l]);
        C0 = C0 + cq;
    }
    const double f = F0 + Gv;
    const double dlc = C0 + K;
    nb.choice[at] = (uint8_t)(b | (t << 4));
    nb.entry[at] = (uint16_t)ent;
    if (root) {
        *nb.froot = f;
        return;
    }
    const double Sc = nb.A[at];                 // congestion sum gathered up front
    const double len = (double)nb.len[i];
    const double Rw = sh.T.r[l] * len;
    const double Cw = sh.T.c[l] * len;
    const double wd = nb.wd[i];
    nb.A[at] = ((f + wd * (Rw * (0.5 * Cw + dlc))) + G.W_CAP * Cw) + (G.W_CONG * sh.T.ofw[l]) * Sc;
    nb.C[at] = Cw + dlc;
}

// ----------------------------------------------------------------- leaves --
// Every non-root leaf i < nleaf, all entry layers, threads over (leaf, slot).
// A leaf has no son terms, G' = V(b, t) >= V(b0, t0) for every admissible span
// (kappa >= 0, rounded addition is monotone) and the key prefers the smaller
// span on ties, so the choice is (b0, t0) with G = V(b0, t0).
__device__ void leaves_dp(const NetCtx &c, const Shared &sh, const DevGrid &G, int nleaf, int tid, int nthr) {
    const NetBuf &nb = c.nb;
    const int LD = c.LD, Lm1 = c.L - 1;
    for (int idx = tid; idx < nleaf * LD; idx += nthr) {
        const int i = idx / LD, s = idx - i * LD;
        const int dt = nb.edir[i] <= 1 ? 0 : 1;
        if (s >= sh.ndir[dt]) continue;
        const int l = sh.lay_of[dt][s];
        if (!sh.routable[l]) continue;           // illegal entry layer (R15): A keeps +inf
        const int nl = nb.nl[i], nh = nb.nh[i];
        const bool pins = nl != 255;
        const int b0 = pins ? min(l, nl) : l, t0 = pins ? max(l, nh) : l;
        double V = 0.0;
        for (int k = b0; k < t0; ++k) V = V + kappa_w(G, sh, nb.vw[i * Lm1 + k], k);
        finish_layer(c, sh, G, i, false, l, s, true, V, 0.0, b0, t0, 0u);
    }
}

// -------------------------------------------------------------- node DP --
// Alg. 3 for node i (internal, or the root), all entry layers, one warp.
__device__ void node_dp(const NetCtx &c, const WarpBuf &wb, const Shared &sh, const DevGrid &G, int i, bool root,
                        int pdrv, int lane) {
    const NetBuf &nb = c.nb;
    const int L = c.L, LD = c.LD, Lm1 = L - 1;
    const int nk = nb.nkid[i];
    const int nl = nb.nl[i], nh = nb.nh[i];
    const bool pins = nl != 255;
    const int dt = root ? 0 : (nb.edir[i] <= 1 ? 0 : 1);
    const int nE = root ? 1 : sh.ndir[dt];
    const double urn = nb.ur[i];
    int kid[MAXKIDS], kdt[MAXKIDS];
#pragma unroll
    for (int k = 0; k < MAXKIDS; ++k) {
        kid[k] = k < nk ? nb.kid[i * MAXKIDS + k] : 0;
        kdt[k] = k < nk ? (nb.edir[kid[k]] <= 1 ? 0 : 1) : 0;
    }
    // ViaCong per cut of this node's GCell
    if (lane < Lm1) wb.kap[lane] = kappa_w(G, sh, nb.vw[i * Lm1 + lane], lane);
    // candidate table CP[k][e][js] = cost'(l_e; s_k, j) (O5): +inf where the son is infeasible
    const int per_k = nE * LD;
    for (int idx = lane; idx < nk * per_k; idx += 32) {
        const int k = idx / per_k, r = idx - k * per_k;
        const int e = r / LD, js = r - e * LD;
        int kk = 0, dk = 0;
#pragma unroll
        for (int q = 0; q < MAXKIDS; ++q) if (q == k) { kk = kid[q]; dk = kdt[q]; }
        if (js >= sh.ndir[dk]) continue;
        const int l = root ? pdrv : sh.lay_of[dt][e];
        const int j = sh.lay_of[dk][js];
        const int at = kk * LD + js;
        const double A = nb.A[at];
        double cp = dinf();
        if (A < dinf()) {
            const double Bv = nb.wd[kk] * nb.C[at];          // B = wd_s (Cw + D)
            const double cost = A + Bv * sh.T.VR[l * MAXL + j];
            cp = cost + Bv * urn;
        }
        wb.CP[(k * LD + e) * LD + js] = cp;
    }
    // span-bottom tasks: entry e has b in [0, b0(e)]; a lane owns up to m of them
    int cnt = 0;
    if (lane < nE) {
        const int l = root ? pdrv : sh.lay_of[dt][lane];
        if (root || sh.routable[l]) cnt = (pins ? min(l, nl) : l) + 1;   // R13, R15
    }
    int m = 1, g = cnt, P = 0;
    for (;;) {
        g = (cnt + m - 1) / m;
        P = g;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) P += __shfl_xor_sync(FULL_MASK, P, o);
        if (P <= 32) break;
        ++m;
    }
    int inc = g;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(FULL_MASK, inc, o);
        if (lane >= o) inc += x;
    }
    for (int q = 0; q < g; ++q) wb.map[inc - g + q] = (uint16_t)(lane | (q << 8));
    __syncwarp();

    bool have = false;
    double bGp = 0.0, bV = 0.0;
    int bt = 0, bb = 0;
    uint32_t bjs = 0;
    int e = 0, seg_end = 0;
    if (lane < P) {
        const uint16_t mp = wb.map[lane];
        e = mp & 0xff;
        const int q = mp >> 8;
        const int l = root ? pdrv : sh.lay_of[dt][e];
        const int b0 = pins ? min(l, nl) : l, t0 = pins ? max(l, nh) : l;
        const double *CPe = wb.CP + e * LD;
        const int bend = min(q * m + m, b0 + 1);
        for (int b = q * m; b < bend; ++b) {
            double V = 0.0;
            for (int k = b; k < t0; ++k) V = V + wb.kap[k];
            double mv[MAXKIDS];
            int jb[MAXKIDS];
#pragma unroll
            for (int k = 0; k < MAXKIDS; ++k) { mv[k] = dinf(); jb[k] = -1; }
            // son argmin of cost' over j in [b, t], ties -> lowest j (ascending j, strict <)
            auto consider = [&](int j) {
                if (!sh.routable[j]) return;
                const int dj = sh.dir[j], sj = sh.lidx[j];
#pragma unroll
                for (int k = 0; k < MAXKIDS; ++k) {
                    if (k < nk && kdt[k] == dj) {
                        const double cp = CPe[k * LD * LD + sj];
                        if (cp < mv[k]) { mv[k] = cp; jb[k] = j; }
                    }
                }
            };
            for (int j = b; j <= t0; ++j) consider(j);
            for (int t = t0; t < L; ++t) {
                if (t > t0) {
                    V = V + wb.kap[t - 1];
                    consider(t);
                }
                bool feas = true;
                double Gp = V;
                uint32_t js = 0;
#pragma unroll
                for (int k = 0; k < MAXKIDS; ++k) {
                    if (k < nk) {
                        feas = feas && jb[k] >= 0;
                        Gp = Gp + mv[k];
                        js |= (uint32_t)(jb[k] & 0xf) << (4 * k);
                    }
                }
                if (!feas) continue;
                // key (G', t - b, b), lexicographic (reading R21)
                const bool better = !have || Gp < bGp ||
                                    (Gp == bGp && ((t - b) < (bt - bb) || ((t - b) == (bt - bb) && b < bb)));
                if (better) { have = true; bGp = Gp; bt = t; bb = b; bjs = js; bV = V; }
            }
        }
    }
    // segmented argmin over the lanes of one entry layer (contiguous lanes)
    seg_end = __shfl_sync(FULL_MASK, inc, e);
    if (lane >= P) seg_end = 0;
    uint32_t key = (have ? 1u << 16 : 0u) | ((uint32_t)bt << 8) | ((uint32_t)bb << 4) | 0u;
    int src = lane;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double oG = __shfl_down_sync(FULL_MASK, bGp, o);
        const uint32_t ok = __shfl_down_sync(FULL_MASK, key, o);
        const int os = __shfl_down_sync(FULL_MASK, src, o);
        if (lane + o < seg_end && (ok >> 16)) {
            const int ot = (ok >> 8) & 0xff, ob = (ok >> 4) & 0xf;
            const int mt = (key >> 8) & 0xff, mb = (key >> 4) & 0xf;
            const bool better = !(key >> 16) || oG < bGp ||
                                (oG == bGp && ((ot - ob) < (mt - mb) || ((ot - ob) == (mt - mb) && ob < mb)));
            if (better) { bGp = oG; key = ok; src = os; }
        }
    }
    const uint32_t wjs = __shfl_sync(FULL_MASK, bjs, src);
    const double wV = __shfl_sync(FULL_MASK, bV, src);
    if (lane < P && (wb.map[lane] >> 8) == 0) {      // head lane of entry e
        const int l = root ? pdrv : sh.lay_of[dt][e];
        const int slot = root ? 0 : e;
        if (!(key >> 16)) {
            finish_layer(c, sh, G, i, root, l, slot, false, 0.0, 0.0, 0, 0, 0u);
        } else {
            const int t = (key >> 8) & 0xff, b = (key >> 4) & 0xf;
            double Gv = wV, K = 0.0;
#pragma unroll
            for (int k = 0; k < MAXKIDS; ++k) {
                if (k < nk) {
                    const int j = (wjs >> (4 * k)) & 0xf;
                    const int at = kid[k] * LD + sh.lidx[j];
                    const double A = nb.A[at], Cc = nb.C[at];
                    const double Bv = nb.wd[kid[k]] * Cc;
                    Gv = Gv + (A + Bv * sh.T.VR[l * MAXL + j]);
                    K = K + Cc;
                }
            }
            finish_layer(c, sh, G, i, root, l, slot, true, Gv, K, b, t, wjs);
        }
    }
    __syncwarp();
}

// ------------------------------------------------------------- gathering --
// Congestion sum S of a parent run on the layer with slot s of its direction:
// ((m1 + m2) + ...) + m_len in ascending coordinate (reading R23).
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

// Node records and sinks of net [n0, n0+nn) into nb (threads tid of nthr).
__device__ __forceinline__ void gather_nodes(const NetBuf &nb, const DevForest &F, int64_t n0, int nn, int tid,
                                             int nthr) {
    const int q_base = F.sink0[n0];
    for (int i = tid; i < nn; i += nthr) {
        const int64_t n = n0 + i;
        nb.xy[i] = F.xy[n];
        nb.len[i] = (uint16_t)F.len[n];
        nb.edir[i] = F.edir[n];
        nb.nkid[i] = F.nkid[n];
        nb.nl[i] = F.nl[n];
        nb.nh[i] = F.nh[n];
        nb.height[i] = F.height[n];
        nb.nsink[i] = F.nsink[n];
        nb.sink0[i] = (uint16_t)(F.sink0[n] - q_base);
        nb.wd[i] = F.wd[n];
        nb.ur[i] = F.ur[n];
        const int4 k4 = *reinterpret_cast<const int4 *>(F.kid + n * 4);
        nb.kid[i * 4 + 0] = (uint16_t)(k4.x - n0);
        nb.kid[i * 4 + 1] = (uint16_t)(k4.y - n0);
        nb.kid[i * 4 + 2] = (uint16_t)(k4.z - n0);
        nb.kid[i * 4 + 3] = (uint16_t)(k4.w - n0);
    }
    const int64_t nlast = n0 + nn - 1;
    const int ns = F.sink0[nlast] + F.nsink[nlast] - q_base;
    for (int q = tid; q < ns; q += nthr) {
        nb.player[q] = F.p_layer[q_base + q];
        nb.pcap[q] = F.p_cap[q_base + q];
        nb.pw[q] = F.p_w[q_base + q];
    }
}

// Via-cut words per (node, cut) and S per (non-root node, layer slot).
__device__ __forceinline__ void gather_state(const NetBuf &nb, const DevGrid &G, const Shared &sh, int nn, int LD,
                                             int tid, int nthr) {
    const int Lm1 = G.L - 1;
    for (int idx = tid; idx < nn * Lm1; idx += nthr) {
        const int i = idx / Lm1, k = idx - i * Lm1;
        const uint32_t xy = nb.xy[i];
        nb.vw[idx] = __ldcg(G.via + ((int64_t)(xy >> 16) * G.X + (xy & 0xffff)) * Lm1 + k);
    }
    for (int idx = tid; idx < nn * LD; idx += nthr) {
        const int i = idx / LD, s = idx - i * LD;
        const int ed = nb.edir[i];
        if (ed == NO_DIR) continue;
        const int dt = ed <= 1 ? 0 : 1;
        if (s >= sh.ndir[dt]) continue;
        if (!sh.routable[sh.lay_of[dt][s]]) { nb.A[idx] = dinf(); continue; }
        const uint32_t xy = nb.xy[i];
        nb.A[idx] = run_sum(G, dt, s, xy & 0xffff, xy >> 16, ed, nb.len[i]);
    }
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

// Backtrack of node i (Alg. 4): its span from choice[i][l_i], its sons' layers from entry.
__device__ __forceinline__ void backtrack_node(const NetCtx &c, const Shared &sh, int i) {
    const NetBuf &nb = c.nb;
    const int l = nb.lay[i];
    const int slot = (i == c.nn - 1) ? 0 : sh.lidx[l];
    const uint8_t ch = nb.choice[i * c.LD + slot];
    nb.sb[i] = ch & 0xf;
    nb.st[i] = ch >> 4;
    const uint32_t js = nb.entry[i * c.LD + slot];
    const int nk = nb.nkid[i];
    for (int k = 0; k < nk; ++k) nb.lay[nb.kid[i * 4 + k]] = (uint8_t)((js >> (4 * k)) & 0xf);
}

// CTA barrier that is correct when a warp arrives diverged (e.g. one lane
// spinning on a dependency counter while the others wait): the NON-aligned
// barrier.sync counts threads, whereas __syncthreads (bar.sync, .aligned)
// requires every warp to arrive converged.
__device__ __forceinline__ void cta_sync() { asm volatile("barrier.sync 0;" ::: "memory"); }

__device__ __forceinline__ int32_t ld_acquire(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ------------------------------------------------------------------ kernel --
__global__ void __launch_bounds__(ASSIGN_WARPS * 32, 5) k_assign(DevGrid G, DevForest F, DevScratch S, AssignLaunch a) {
    __shared__ Shared sh;
    extern __shared__ __align__(16) char dyn[];
    stage_tab(sh.T, G.tab);
    if (threadIdx.x < MAXL) {
        const int l = threadIdx.x;
        sh.dir[l] = G.dir[l];
        sh.routable[l] = G.routable[l];
        sh.lidx[l] = (uint8_t)G.lidx[l];
        if (l < G.L) sh.lay_of[G.dir[l]][G.lidx[l]] = (uint8_t)l;
    }
    if (threadIdx.x == 0) { sh.ndir[0] = G.LH; sh.ndir[1] = G.LV; }
    const int L = G.L, LD = a.LD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const WarpLay wlay = warp_layout(L, LD);
    const NetLay slay = net_layout(a.NS, a.NP, L, LD);
    char *wscr = dyn + warp * wlay.bytes;
    char *nets = dyn + ASSIGN_WARPS * wlay.bytes;
    const WarpBuf wb{reinterpret_cast<double *>(wscr + wlay.CP), reinterpret_cast<double *>(wscr + wlay.kap),
                     reinterpret_cast<uint16_t *>(wscr + wlay.map)};
    const bool flow = a.wait != nullptr;

    for (;;) {
        cta_sync();
        if (threadIdx.x == 0) {
            const unsigned long long t = atomicAdd(a.ticket, 1ull);
            sh.item = (int64_t)t < a.item_end - a.item_beg ? a.item_beg + (int64_t)t : -1;
        }
        cta_sync();
        const int64_t item = sh.item;
        if (item < 0) return;
        const uint64_t it = a.items[item];
        const int64_t net_first = (int64_t)(it & 0xffffffffull);
        const int cnt = (int)((it >> 32) & 0xff);
        const bool big = (it >> 40) & 1;

        if (big) {
            // ======================= big net: the whole CTA =======================
            const int64_t net = net_first;
            const int64_t n0 = F.net_node0[net], n1 = F.net_node0[net + 1];
            const int nn = (int)(n1 - n0);
            const int ns = F.sink0[n1 - 1] + F.nsink[n1 - 1] - F.sink0[n0];
            const NetLay blay = net_layout(nn, ns, L, LD);
            char *base = blay.bytes <= a.big_smem ? nets : a.gscratch + (int64_t)blockIdx.x * a.gslot_bytes;
            const NetCtx c{net_buf(base, blay), L, LD, nn};
            const int pdrv = F.net_pdrv[net];
            if (flow) {
                if (threadIdx.x == 0) while (ld_acquire(a.wait + net) > 0) __nanosleep(100);
                cta_sync();
                __threadfence();
            }
            gather_nodes(c.nb, F, n0, nn, threadIdx.x, blockDim.x);
            cta_sync();
            gather_state(c.nb, G, sh, nn, LD, threadIdx.x, blockDim.x);
            if (threadIdx.x == 0) {
                int hi = 0;
                while (hi < nn - 1 && c.nb.height[hi] == 0) ++hi;
                sh.lo = 0;
                sh.hi = hi;
            }
            cta_sync();
            leaves_dp(c, sh, G, sh.hi, threadIdx.x, blockDim.x);
            for (;;) {
                cta_sync();
                if (threadIdx.x == 0) {
                    int lo = sh.hi, hi = lo;
                    if (lo < nn) {
                        const int h = c.nb.height[lo];
                        while (hi < nn && c.nb.height[hi] == h) ++hi;
                    }
                    sh.lo = lo;
                    sh.hi = hi;
                }
                cta_sync();
                const int lo = sh.lo, hi = sh.hi;
                if (lo >= nn) break;
                for (int i = lo + warp; i < hi; i += ASSIGN_WARPS) node_dp(c, wb, sh, G, i, i == nn - 1, pdrv, lane);
            }
            // Alg. 4, level-parallel from the root (root entry = driver pin layer, R13)
            if (threadIdx.x == 0) {
                c.nb.lay[nn - 1] = (uint8_t)pdrv;
                S.froot[net] = *c.nb.froot;
                sh.lo = nn;
            }
            for (;;) {
                cta_sync();
                if (threadIdx.x == 0) {
                    const int hi = sh.lo;
                    int lo = hi;
                    if (hi > 0) {
                        const int h = c.nb.height[hi - 1];
                        while (lo > 0 && c.nb.height[lo - 1] == h) --lo;
                    }
                    sh.hi = hi;
                    sh.lo = lo;
                }
                cta_sync();
                const int lo = sh.lo, hi = sh.hi;
                if (hi <= 0) break;
                for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) backtrack_node(c, sh, i);
            }
            cta_sync();
            for (int i = threadIdx.x; i < nn; i += blockDim.x) {
                S.lay[n0 + i] = c.nb.lay[i];
                S.sb[n0 + i] = c.nb.sb[i];
                S.st[n0 + i] = c.nb.st[i];
                if (a.commit) commit_node(G, c.nb.xy[i], c.nb.edir[i], c.nb.len[i], c.nb.lay[i], c.nb.sb[i], c.nb.st[i]);
            }
            if (flow) {
                __threadfence();
                cta_sync();
                for (int64_t e = a.succ_off[net] + threadIdx.x; e < a.succ_off[net + 1]; e += blockDim.x)
                    atomicSub(a.wait + a.succ[e], 1);
            }
            continue;
        }

        // ========================= small nets: one warp each =========================
        if (warp >= cnt) continue;
        const int64_t net = net_first + warp;
        const int64_t n0 = F.net_node0[net], n1 = F.net_node0[net + 1];
        const int nn = (int)(n1 - n0);
        const NetCtx c{net_buf(nets + warp * slay.bytes, slay), L, LD, nn};
        const int pdrv = F.net_pdrv[net];
        if (flow) {
            while (ld_acquire(a.wait + net) > 0) __nanosleep(64);
            __syncwarp();
        }
        gather_nodes(c.nb, F, n0, nn, lane, 32);
        __syncwarp();
        gather_state(c.nb, G, sh, nn, LD, lane, 32);
        __syncwarp();
        int nleaf = 0;
        while (nleaf < nn - 1 && c.nb.height[nleaf] == 0) ++nleaf;
        leaves_dp(c, sh, G, nleaf, lane, 32);
        __syncwarp();
        for (int i = nleaf; i < nn; ++i) node_dp(c, wb, sh, G, i, i == nn - 1, pdrv, lane);
        if (lane == 0) {
            S.froot[net] = *c.nb.froot;
            c.nb.lay[nn - 1] = (uint8_t)pdrv;
        }
        __syncwarp();
        int hi = nn;
        while (hi > 0) {
            const int h = c.nb.height[hi - 1];
            int lo = hi - 1;
            while (lo > 0 && c.nb.height[lo - 1] == h) --lo;
            for (int i = lo + lane; i < hi; i += 32) backtrack_node(c, sh, i);
            __syncwarp();
            hi = lo;
        }
        for (int i = lane; i < nn; i += 32) {
            S.lay[n0 + i] = c.nb.lay[i];
            S.sb[n0 + i] = c.nb.sb[i];
            S.st[n0 + i] = c.nb.st[i];
            if (a.commit) commit_node(G, c.nb.xy[i], c.nb.edir[i], c.nb.len[i], c.nb.lay[i], c.nb.sb[i], c.nb.st[i]);
        }
        if (flow) {
            __threadfence();
            __syncwarp();
            for (int64_t e = a.succ_off[net] + lane; e < a.succ_off[net + 1]; e += 32) atomicSub(a.wait + a.succ[e], 1);
        }
    }
}

}  // namespace

size_t assign_smem_bytes(int L, int LD, int NS, int NP) {
    return (size_t)ASSIGN_WARPS * (warp_layout(L, LD).bytes + net_layout(NS, NP, L, LD).bytes);
}

size_t assign_net_bytes(int nodes, int sinks, int L, int LD) { return (size_t)net_layout(nodes, sinks, L, LD).bytes; }

cudaError_t assign_resident_ctas(int L, int LD, int NS, int NP, int *per_sm, int *n_sm) {
    const size_t smem = assign_smem_bytes(L, LD, NS, NP);
    cudaError_t e = cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_assign, ASSIGN_WARPS * 32, smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    return cudaDeviceGetAttribute(n_sm, cudaDevAttrMultiProcessorCount, dev);
}

cudaError_t launch_assign(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a, int grid,
                          cudaStream_t s) {
    if (a.item_end <= a.item_beg || grid <= 0) return cudaSuccess;
    const size_t smem = assign_smem_bytes(G.L, a.LD, a.NS, a.NP);
    if (a.wait) {
        // dataflow mode: every CTA must be co-resident (nets wait on each other)
        void *args[] = {(void *)&G, (void *)&F, (void *)&S, (void *)&a};
        return cudaLaunchCooperativeKernel((const void *)k_assign, dim3(grid), dim3(ASSIGN_WARPS * 32), args, smem, s);
    }
    k_assign<<<(unsigned)grid, ASSIGN_WARPS * 32, smem, s>>>(G, F, S, a);
    return cudaGetLastError();
}

}  // namespace gapla
