// K4 + K5 + fused K8: Alg. 3 getSubtreeCandidate + Alg. 4 traceBackSolution
// and the demand commit, for every net, as ONE kernel.
//
// Design (DESIGN §5 "k_assign", §2):
//   * Work.  The forest is batch-major.  CTAs are persistent and have
//     one of two roles.  SMALL nets (at most NS nodes and NP sinks; ~99%): every
//     warp takes the next one with its own atomic ticket and runs it alone, DP
//     state in the warp's shared-memory slot.  BIG nets: the first n_big_ctas CTAs
//     take one at a time and spread each height level's nodes over their warps,
//     DP state in the CTA's whole shared memory (a global slot beyond that).  Big
//     nets are few but long, and sit on the critical path of the conflict DAG.
//   * Batch mode (la_assign_batch): the nets of one conflict-free batch.
//     Dataflow mode (la_assign_all, one GPU): ALL nets in one cooperative launch;
//     a net waits until its per-net count of unfinished predecessors (the
//     conflict DAG) is 0, and after its commit releases its
//     successors.  Each role takes its nets in a topological priority order and
//     waits only for the net it holds, so the earliest unfinished net is always
//     held or next in its role's line: no deadlock.
//   * Per net: (1) gather everything the DP reads from HBM -- node records,
//     sinks, the ViaCong kappa of every cut of every node GCell and the
//     congestion sum S of every parent run on every legal layer -- with all
//     loads in flight at once; (2) all leaves at once, lanes over (leaf, entry
//     layer); (3) internal nodes in height order, one WARP per node ("wide
//     node", below); (4) level-parallel backtrack (Alg. 4); (5) decisions to HBM
//     and the integer-atomic demand commit (O8).
//
// Wide node (Alg. 3 l.360-409 for one node, all entry layers).  Tables first,
// lanes in parallel: V(b, t) for every b <= t (R10, each row summed ascending
// from b), cost'(l_e; s_k, j) for every (entry, son, son layer) (O5).  Then the
// CANDIDATE spans of every entry are tasks spread over the lanes; each task
// takes every son's window argmin from the table and its G', and a segmented
// warp argmin by the key (G', t-b, b) (R21) keeps each entry's best; the entry's
// lane then recomputes G, K and the son layers of the winner and finishes.
//
// Candidate spans (exact; DESIGN §5 "minimal covers").  Alg. 3 enumerates every
// span (b, t) with b <= b0 = min(l, nl), t >= t0 = max(l, nh).  Let S* be the
// winner under the key and J* its per-son argmins (lowest j on ties).  The
// smallest span S' covering {b0, t0} and J* lies inside S*; since kappa >= 0 and
// rounded addition is monotone, V(S') <= V(S*), and every son keeps its argmin
// (m_s(S') = cost'(j*_s)), so G'(S') <= G'(S*) with t'-b' <= t*-b*: the key
// forces S' = S*.  Hence S* is the minimal cover of its own argmins, so
//   b* in {b0} U {legal son layers < b0},  t* in {t0} U {legal son layers > t0},
// and with ONE son (83% of internal nodes) also b* == b0 or t* == t0.  The
// kernel evaluates exactly those spans, each with the oracle's expression
// tree, so the argmin equals the full enumeration's.
//
// Bit-exactness: compiled with --fmad=false; every fp64 value is the DESIGN §3
// expression tree in operand order; cross-lane reductions are argmins only.
#include <cuda_runtime.h>

#include "la_device.cuh"
#include "la_internal.h"

namespace gapla {
namespace {

constexpr int MAXE = 8;                               // entry layer slots per direction (L <= 16)

// ---------------------------------------------------------------- layouts --
// One net's DP state in a warp's slot (shared memory; a big net: the CTA's
// slots, or a global slot): node records, (node, entry slot) records, kappa of
// every (node, cut), sinks, decisions.
struct NodeRec {
    double wd, ur;                    // W_D w_n (Eq. 5), ur (O3)
    uint32_t xy;                      // x | y << 16
    uint16_t len, height, nsink, sink0;
    uint16_t kid[MAXKIDS];            // children (net-local), E W N S order
    uint8_t edir, nkid, nl, nh, lay, sb, st, pad;
};
static_assert(sizeof(NodeRec) == 48, "NodeRec layout");
struct SlotRec {                      // node i, entry layer slot e
    double A, C;                      // gathered S, then O5 A(l) and capb(l) of the parent edge
};
struct SinkRec {
    double cap, w;                    // C_q, weight of its pin-via delay term
};

struct NetLay {
    int node, slot, sink, kap, dec, player, froot, bytes;
};

__host__ __device__ inline NetLay net_layout(int NS, int NP, int L, int LD) {
    NetLay w;
    int o = 0;
    auto take = [&](int bytes) { int r = o; o += (bytes + 15) & ~15; return r; };
    w.node = take(48 * NS);
    w.slot = take(16 * NS * LD);
    w.sink = take(16 * NP);
    w.kap = take(8 * NS * (L - 1));
    w.dec = take(4 * NS * LD);        // (choice | entry << 8) per (node, slot)
    w.player = take(NP);
    w.froot = take(8);
    w.bytes = o;
    return w;
}

struct NetBuf {
    NodeRec *nd;
    SlotRec *sl;
    SinkRec *sk;
    double *kap;
    uint32_t *dec;
    uint8_t *player;
    double *froot;
};

__device__ __forceinline__ NetBuf net_buf(char *b, const NetLay &w) {
    NetBuf n;
    n.nd = (NodeRec *)(b + w.node); n.sl = (SlotRec *)(b + w.slot); n.sk = (SinkRec *)(b + w.sink);
    n.kap = (double *)(b + w.kap); n.dec = (uint32_t *)(b + w.dec); n.player = (uint8_t *)(b + w.player);
    n.froot = (double *)(b + w.froot);
    return n;
}

// Per-warp scratch of the wide node routine, sized for the grid's L (rows of V) and LD (son
// layer slots): V(b, t) [L][L]; cost'(l_e; s_k, slot) [LD][MAXKIDS][LD]; per entry best G',
// key and layer.
struct WarpScr {
    double *Vt, *cpt, *bestG;
    uint32_t *bestK;                      // (t - b) << 4 | b, bit 8 = none
    uint8_t *el;
    int vs, cs;                           // row strides: V (L), cost' (LD)
};

__host__ __device__ inline int scr_bytes(int L, int LD) {
    return ((8 * L * L + 8 * LD * MAXKIDS * LD + 8 * MAXE + 4 * MAXE + MAXE) + 15) & ~15;
}

__device__ __forceinline__ WarpScr warp_scr(char *b, int L, int LD) {
    WarpScr w;
    w.Vt = (double *)b;
    w.cpt = w.Vt + L * L;
    w.bestG = w.cpt + LD * MAXKIDS * LD;
    w.bestK = (uint32_t *)(w.bestG + MAXE);
    w.el = (uint8_t *)(w.bestK + MAXE);
    w.vs = L;
    w.cs = LD;
    return w;
}

struct Shared {          // per-CTA static shared memory
    TechTab T;
    uint8_t dir[MAXL], routable[MAXL], lidx[MAXL];
    uint8_t lay_of[2][MAXL];   // layer of slot s in direction d
    int ndir[2];               // legal layers per direction
    uint32_t legal[2];         // bit j: layer j is routable and of direction d
};

// Context of one net inside the node routines.
struct NetCtx {
    NetBuf nb;
    int L, LD, nn;
};

__device__ __forceinline__ double kappa_w(const DevGrid &G, const Shared &sh, int32_t w, int k) {
    return G.W_VIA + (G.W_CONG * sh.T.ofw[k]) * marginal(G, w);    // ViaCong, reading R11
}

// n-th (1-based) set bit of m
__device__ __forceinline__ int nth_bit(uint32_t m, int n) {
#pragma unroll 1
    for (int k = 1; k < n; ++k) m &= m - 1;
    return __ffs(m) - 1;
}

// -------------------------------------------------------- node finishing --
// Entry layer l (slot `slot`) of node i once its span is chosen: pin terms
// (Alg. 3 l.4-7), f and dlc (l.405), choice / entry (l.406-408); for a non-root
// node also the O5 parent-edge terms A and capb on layer l (its edge layer).
__device__ __forceinline__ void finish_layer(const NetCtx &c, const Shared &sh, const DevGrid &G, int i, bool root,
                                             int l, int slot, double Gv, double K, int b, int t, uint32_t ent) {
    const NetBuf &nb = c.nb;
    const int at = i * c.LD + slot;
    const NodeRec &nd = nb.nd[i];
    double F0 = 0.0, C0 = 0.0;
    const int q0 = nd.sink0, qn = nd.nsink;
#pragma unroll 1
    for (int q = q0; q < q0 + qn; ++q) {
        const double cq = nb.sk[q].cap;
        F0 = F0 + nb.sk[q].w * (cq * sh.T.VR[nb.player[q] * MAXL + l]);
        C0 = C0 + cq;
    }
    const double f = F0 + Gv;
    const double dlc = C0 + K;
    nb.dec[at] = (uint32_t)(b | (t << 4)) | (ent << 8);
    if (root) {
        *nb.froot = f;
        return;
    }
    const double Sc = nb.sl[at].A;              // congestion sum gathered up front
    const double len = (double)nd.len;
    const double Rw = sh.T.r[l] * len;
    const double Cw = sh.T.c[l] * len;
    const double wd = nd.wd;
    nb.sl[at].A = ((f + wd * (Rw * (0.5 * Cw + dlc))) + G.W_CAP * Cw) + (G.W_CONG * sh.T.ofw[l]) * Sc;
    nb.sl[at].C = Cw + dlc;
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
        const NodeRec &nd = nb.nd[i];
        const int dt = nd.edir <= 1 ? 0 : 1;
        if (s >= sh.ndir[dt]) continue;
        const int l = sh.lay_of[dt][s];
        if (!sh.routable[l]) continue;           // illegal entry layer (R15): A keeps +inf
        const int nl = nd.nl, nh = nd.nh;
        const bool pins = nl != 255;
        const int b0 = pins ? min(l, nl) : l, t0 = pins ? max(l, nh) : l;
        double V = 0.0;
#pragma unroll 1
        for (int k = b0; k < t0; ++k) V = V + nb.kap[i * Lm1 + k];
        finish_layer(c, sh, G, i, false, l, s, V, 0.0, b0, t0, 0u);
    }
}

// -------------------------------------------------------------- wide node --
// Son k's window argmin over [b, t] on entry e: lowest layer among the minima
// of the finite cost' values (ascending slots = ascending layers, strict <).
__device__ __forceinline__ int window_argmin(const WarpScr &w, const Shared &sh, int e, int k, int dk, int b, int t,
                                             double *mv) {
    double m = dinf();
    int jb = -1;
    const double *row = w.cpt + (e * MAXKIDS + k) * w.cs;
    const int nd = sh.ndir[dk];
#pragma unroll 1
    for (int s = 0; s < nd; ++s) {
        {
            const int j = sh.lay_of[dk][s];
            if (j >= b && j <= t) {
                const double cp = row[s];
                if (cp < m) { m = cp; jb = j; }
            }
        }
    }
    *mv = m;
    return jb;
}

// Alg. 3 for a node with ONE son (83% of internal nodes), all entries, by one
// warp: 8-lane segments, one per entry layer, lane s of a segment = son layer
// slot s.  Candidates (header: minimal covers): (b0, t0), (b0, j) for son layers
// j > t0 and (j, t0) for son layers j < b0; the window minima come from two
// segmented scans -- upward from b0 (strict <: the lower layer keeps ties) and
// downward from t0 (the lower layer wins ties) -- and a butterfly argmin by the
// key (G', t-b, b) picks each entry's span.
__device__ __forceinline__ void node_dp_1son(const NetCtx &c, WarpScr &w, const Shared &sh, const DevGrid &G,
                                             int i, bool root, int pdrv, int dt, int nE, int kk, int dk, int lane) {
    const NetBuf &nb = c.nb;
    const NodeRec &nd = nb.nd[i];
    const int LD = c.LD, ndk = sh.ndir[dk], s = lane & 7;
    const double urn = nd.ur, wdk = nb.nd[kk].wd;
    const int nl = nd.nl, nh = nd.nh;
    const bool pins = nl != 255;
    const int j = s < ndk ? sh.lay_of[dk][s] : MAXL;
    const int jnext = s + 1 < ndk ? sh.lay_of[dk][s + 1] : MAXL;
    for (int e0 = 0; e0 < nE; e0 += 4) {
        const int e = e0 + (lane >> 3);
        const int l = root ? pdrv : sh.lay_of[dt][e < nE ? e : 0];
        const bool eok = e < nE && (root || sh.routable[l]);
        const int b0 = pins ? min(l, nl) : l, t0 = pins ? max(l, nh) : l;
        double cp = dinf();
        if (eok && s < ndk) {
            const SlotRec &rr = nb.sl[kk * LD + s];
            const double A = rr.A;
            if (A < dinf()) {
                const double Bv = wdk * rr.C;                // B = wd_s (Cw + D)
                const double cost = A + Bv * sh.T.VR[l * MAXL + j];
                cp = cost + Bv * urn;
            }
        }
        // windows [b0, j]: inclusive prefix min over layers >= b0, lowest layer on ties
        double pu = (j >= b0 && cp < dinf()) ? cp : dinf();
        int ju = pu < dinf() ? j : -1;
        // windows [j, t0]: inclusive suffix min over layers <= t0, lowest layer on ties
        double pd = (j <= t0 && cp < dinf()) ? cp : dinf();
        int jd = pd < dinf() ? j : -1;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const double ou = __shfl_up_sync(FULL_MASK, pu, o, 8);
            const int oju = __shfl_up_sync(FULL_MASK, ju, o, 8);
            const double od = __shfl_down_sync(FULL_MASK, pd, o, 8);
            const int ojd = __shfl_down_sync(FULL_MASK, jd, o, 8);
            if (s >= o && ou <= pu && oju >= 0) { pu = ou; ju = oju; }
            if (s + o < 8 && od < pd) { pd = od; jd = ojd; }
        }
        double Gp = dinf();
        uint32_t key = 0x1ffu;
        int jm = -1;
        if (eok && s < ndk) {
            int b = b0, t = t0;
            double m = dinf();
            if (j > t0) { t = j; m = pu; jm = ju; }
            else if (j < b0) { b = j; m = pd; jm = jd; }
            else if (jnext > t0) { m = pu; jm = ju; }        // last son layer inside [b0, t0]: the base span
            if (jm >= 0) {
                Gp = w.Vt[b * w.vs + t] + m;
                key = (uint32_t)(((t - b) << 4) | b);
            }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            const double oG = __shfl_xor_sync(FULL_MASK, Gp, o, 8);
            const uint32_t ok = __shfl_xor_sync(FULL_MASK, key, o, 8);
            const int oj = __shfl_xor_sync(FULL_MASK, jm, o, 8);
            if (oG < Gp || (oG == Gp && ok < key)) { Gp = oG; key = ok; jm = oj; }
        }
        if (s == 0 && e < nE) {
            w.el[e] = (uint8_t)l;
            w.bestK[e] = eok ? (key | ((uint32_t)(jm & 0xf) << 12)) : 0x1ffu;
        }
    }
    __syncwarp();
    // entry lanes finish in parallel: G (cost, not cost'), K = capb (O6)
    if (lane < nE) {
        const int e = lane, l = w.el[e];
        const uint32_t key = w.bestK[e];
        if (root || sh.routable[l]) {
            const int slot = root ? 0 : e;
            if (key & 0x100u) {
                if (root) *nb.froot = dinf();
                else nb.sl[i * LD + slot].A = dinf();
            } else {
                const int b = key & 0xf, t = b + (int)((key >> 4) & 0xf), jm = (int)(key >> 12);
                const SlotRec &rr = nb.sl[kk * LD + sh.lidx[jm]];
                const double Bv = wdk * rr.C;
                const double Gv = w.Vt[b * w.vs + t] + (rr.A + Bv * sh.T.VR[l * MAXL + jm]);
                finish_layer(c, sh, G, i, root, l, slot, Gv, 0.0 + rr.C, b, t, (uint32_t)jm);
            }
        }
    }
}

// Alg. 3 for internal node (or root) i by one warp.
__device__ void node_dp_wide(const NetCtx &c, WarpScr &w, const Shared &sh, const DevGrid &G, int i, int pdrv,
                             int lane) {
    const NetBuf &nb = c.nb;
    const int L = c.L, LD = c.LD, Lm1 = L - 1;
    const bool root = i == c.nn - 1;
    const NodeRec &nd = nb.nd[i];
    const int nk = nd.nkid;
    const int dt = root ? 0 : (nd.edir <= 1 ? 0 : 1);
    const int nE = root ? 1 : sh.ndir[dt];
    const double urn = nd.ur;
    int kid[MAXKIDS], kdt[MAXKIDS];
    uint32_t legal_any = 0;
#pragma unroll
    for (int k = 0; k < MAXKIDS; ++k) {
        kid[k] = k < nk ? nd.kid[k] : 0;
        kdt[k] = k < nk ? (nb.nd[kid[k]].edir <= 1 ? 0 : 1) : 0;
        if (k < nk) legal_any |= sh.legal[kdt[k]];
    }
    const double *kap = nb.kap + i * Lm1;
    // (1) V table: lane b sums its row ascending from b (R10, R23)
    if (lane < L) {
        double V = 0.0;
        w.Vt[lane * w.vs + lane] = 0.0;
#pragma unroll 1
        for (int t = lane + 1; t < L; ++t) {
            V = V + kap[t - 1];
            w.Vt[lane * w.vs + t] = V;
        }
    }
    if (nk == 1) {
        __syncwarp();
        node_dp_1son(c, w, sh, G, i, root, pdrv, dt, nE, kid[0], kdt[0], lane);
        __syncwarp();
        return;
    }
    // (2) cost' table (O5, R16-R17): +inf where the son is infeasible on the layer
    const int ncp = nE * nk * LD;
    for (int idx = lane; idx < ncp; idx += 32) {
        const int e = idx / (nk * LD), r = idx - e * (nk * LD);
        const int k = r / LD, s = r - k * LD;
        int kk = 0, dk = 0;
#pragma unroll
        for (int q = 0; q < MAXKIDS; ++q) if (q == k) { kk = kid[q]; dk = kdt[q]; }
        if (s >= sh.ndir[dk]) continue;
        const int l = root ? pdrv : sh.lay_of[dt][e];
        const int j = sh.lay_of[dk][s];
        const SlotRec &rr = nb.sl[kk * LD + s];
        const double A = rr.A;
        double cp = dinf();
        if (A < dinf()) {
            const double Bv = nb.nd[kk].wd * rr.C;           // B = wd_s (Cw + D)
            const double cost = A + Bv * sh.T.VR[l * MAXL + j];
            cp = cost + Bv * urn;
        }
        w.cpt[(e * MAXKIDS + k) * w.cs + s] = cp;
    }
    __syncwarp();
    // (3) lanes over (entry e, span bottom b): 8-lane segments, one per entry, lane s8 takes
    //     the bottoms b = B[s8], B[s8 + 8], ...; each sweeps the candidate tops t upward with
    //     the running son minima (strict <: the lowest layer keeps ties), then a butterfly
    //     argmin by the key (G', t-b, b) (R21) leaves the entry's best span in its segment
    const int nl = nd.nl, nh = nd.nh;
    const bool pins = nl != 255;
    const int s8 = lane & 7;
    for (int e0 = 0; e0 < nE; e0 += 4) {
        const int e = e0 + (lane >> 3);
        const int l = root ? pdrv : sh.lay_of[dt][e < nE ? e : 0];
        const bool eok = e < nE && (root || sh.routable[l]);
        const int b0 = pins ? min(l, nl) : l, t0 = pins ? max(l, nh) : l;
        const uint32_t mB = legal_any & ((1u << b0) - 1u);
        const int nB = 1 + __popc(mB);
        double Gb = dinf();
        uint32_t kb = 0x1ffu;
        for (int bi = s8; eok && bi < nB; bi += 8) {
            const int b = bi == 0 ? b0 : nth_bit(mB, bi);
            double m[MAXKIDS];
#pragma unroll
            for (int k = 0; k < MAXKIDS; ++k) {
                m[k] = dinf();
                if (k < nk) window_argmin(w, sh, e, k, kdt[k], b, t0, &m[k]);
            }
            auto evaluate = [&](int t) {
                double g = w.Vt[b * w.vs + t];
                bool feas = true;
#pragma unroll
                for (int k = 0; k < MAXKIDS; ++k)
                    if (k < nk) {
                        feas = feas && m[k] < dinf();
                        g = g + m[k];
                    }
                const uint32_t key = (uint32_t)(((t - b) << 4) | b);
                if (feas && (g < Gb || (g == Gb && key < kb))) { Gb = g; kb = key; }
            };
            evaluate(t0);
            for (int t = t0 + 1; t < L; ++t) {
                if (!((legal_any >> t) & 1)) continue;
                const int dtt = sh.dir[t], st = sh.lidx[t];
#pragma unroll
                for (int k = 0; k < MAXKIDS; ++k)
                    if (k < nk && kdt[k] == dtt) {
                        const double cp = w.cpt[(e * MAXKIDS + k) * w.cs + st];
                        if (cp < m[k]) m[k] = cp;
                    }
                evaluate(t);
            }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            const double oG = __shfl_xor_sync(FULL_MASK, Gb, o, 8);
            const uint32_t ok = __shfl_xor_sync(FULL_MASK, kb, o, 8);
            if (oG < Gb || (oG == Gb && ok < kb)) { Gb = oG; kb = ok; }
        }
        if (s8 == 0 && e < nE) {
            w.el[e] = (uint8_t)l;
            w.bestG[e] = Gb;
            w.bestK[e] = kb;
        }
    }
    __syncwarp();
    // (5) entry lanes: winner's son layers, G (cost, not cost'), K; finish
    if (lane < nE && (root || sh.routable[w.el[lane]])) {
        const int e = lane, l = w.el[e];
        const uint32_t key = w.bestK[e];
        if (key & 0x100u) {
            if (root) *nb.froot = dinf();
            else nb.sl[i * LD + e].A = dinf();
        } else {
            const int b = key & 0xf, t = b + (int)(key >> 4);
            double Gv = w.Vt[b * w.vs + t], K = 0.0;
            uint32_t js = 0;
#pragma unroll
            for (int k = 0; k < MAXKIDS; ++k) {
                if (k < nk) {
                    double mv;
                    const int j = window_argmin(w, sh, e, k, kdt[k], b, t, &mv);
                    js |= (uint32_t)j << (4 * k);
                    const SlotRec &rr = nb.sl[kid[k] * LD + sh.lidx[j]];
                    const double A = rr.A, Cc = rr.C;
                    const double Bv = nb.nd[kid[k]].wd * Cc;
                    Gv = Gv + (A + Bv * sh.T.VR[l * MAXL + j]);
                    K = K + Cc;
                }
            }
            finish_layer(c, sh, G, i, root, l, root ? 0 : e, Gv, K, b, t, js);
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
__device__ __forceinline__ void gather_nodes(const NetBuf &nb, const DevForest &F, int64_t n0, int nn, int q_base,
                                             int ns, int tid, int nthr) {
    for (int i = tid; i < nn; i += nthr) {
        const int64_t n = n0 + i;
        NodeRec r;
        r.wd = F.wd[n];
        r.ur = F.ur[n];
        r.xy = F.xy[n];
        r.len = (uint16_t)F.len[n];
        r.height = F.height[n];
        r.nsink = F.nsink[n];
        r.sink0 = (uint16_t)(F.sink0[n] - q_base);
        const int4 k4 = *reinterpret_cast<const int4 *>(F.kid + n * 4);
        r.kid[0] = (uint16_t)(k4.x - n0);
        r.kid[1] = (uint16_t)(k4.y - n0);
        r.kid[2] = (uint16_t)(k4.z - n0);
        r.kid[3] = (uint16_t)(k4.w - n0);
        r.edir = F.edir[n];
        r.nkid = F.nkid[n];
        r.nl = F.nl[n];
        r.nh = F.nh[n];
        r.lay = r.sb = r.st = r.pad = 0;
        nb.nd[i] = r;
    }
    for (int q = tid; q < ns; q += nthr) {
        nb.player[q] = F.p_layer[q_base + q];
        nb.sk[q].cap = F.p_cap[q_base + q];
        nb.sk[q].w = F.p_w[q_base + q];
    }
}

// kappa per (node, cut) and S per (non-root node, layer slot).
__device__ __forceinline__ void gather_state(const NetBuf &nb, const DevGrid &G, const Shared &sh, int nn, int LD,
                                             int tid, int nthr) {
    const int Lm1 = G.L - 1;
    for (int idx = tid; idx < nn * Lm1; idx += nthr) {
        const int i = idx / Lm1, k = idx - i * Lm1;
        const uint32_t xy = nb.nd[i].xy;
        nb.kap[idx] = kappa_w(G, sh, __ldcg(G.via + ((int64_t)(xy >> 16) * G.X + (xy & 0xffff)) * Lm1 + k), k);
    }
    for (int idx = tid; idx < nn * LD; idx += nthr) {
        const int i = idx / LD, s = idx - i * LD;
        const int ed = nb.nd[i].edir;
        if (ed == NO_DIR) continue;
        const int dt = ed <= 1 ? 0 : 1;
        if (s >= sh.ndir[dt]) continue;
        if (!sh.routable[sh.lay_of[dt][s]]) { nb.sl[idx].A = dinf(); continue; }
        const uint32_t xy = nb.nd[i].xy;
        nb.sl[idx].A = run_sum(G, dt, s, xy & 0xffff, xy >> 16, ed, nb.nd[i].len);
    }
}

// Fused K8 for node n: +1 per unit edge of its parent run on its layer, +1 per via cut.
__device__ __forceinline__ void commit_node(const DevGrid &G, uint32_t xy, int edir, int len, int l, int b, int t) {
    const int x = xy & 0xffff, y = xy >> 16;
    if (edir != NO_DIR) {
        const int a = run_lo(edir, x, y, len);
        if (edir <= 1) {
            int32_t *wp = G.wH + ((int64_t)y * (G.X - 1) + a) * G.LH + G.lidx[l];
#pragma unroll 1
            for (int e = 0; e < len; ++e) red_add(wp + (int64_t)e * G.LH, 2);
        } else {
            int32_t *wp = G.wV + ((int64_t)x * (G.Y - 1) + a) * G.LV + G.lidx[l];
#pragma unroll 1
            for (int e = 0; e < len; ++e) red_add(wp + (int64_t)e * G.LV, 2);
        }
    }
    int32_t *vp = G.via + ((int64_t)y * G.X + x) * (G.L - 1);
#pragma unroll 1
    for (int k = b; k < t; ++k) red_add(vp + k, 2);
}

// Backtrack of node i (Alg. 4): its span from choice[i][l_i], its sons' layers from entry.
__device__ __forceinline__ void backtrack_node(const NetCtx &c, const Shared &sh, int i) {
    const NetBuf &nb = c.nb;
    NodeRec &nd = nb.nd[i];
    const int l = nd.lay;
    const int slot = (i == c.nn - 1) ? 0 : sh.lidx[l];
    const uint32_t dec = nb.dec[i * c.LD + slot];
    nd.sb = dec & 0xf;
    nd.st = (dec >> 4) & 0xf;
    const uint32_t js = dec >> 8;
    const int nk = nd.nkid;
#pragma unroll 1
    for (int k = 0; k < nk; ++k) nb.nd[nd.kid[k]].lay = (uint8_t)((js >> (4 * k)) & 0xf);
}

__device__ __forceinline__ int64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}

__device__ __forceinline__ int32_t ld_acquire(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// CTA barriers are the NON-aligned barrier.sync (it counts threads; __syncthreads =
// barrier.sync.aligned requires converged warps, and a group's warps reach it diverged: one thread
// spins on a dependency counter, warps leave a level's node loop at different times).
// Over the `n` threads of named barrier `id` (0: the whole CTA; 1 / 2: a half-CTA running one big net).
// Immediate barrier ids keep ptxas from reserving all 16 (id 0: whole CTA, 1 / 2: halves).
__device__ __forceinline__ void bar_sync(int id, int n) {
    if (id == 1) asm volatile("barrier.sync 1, %0;" ::"r"(n) : "memory");
    else if (id == 2) asm volatile("barrier.sync 2, %0;" ::"r"(n) : "memory");
    else asm volatile("barrier.sync 0, %0;" ::"r"(n) : "memory");
}

// Wait until net `net` has no unfinished predecessor (dataflow mode), with a
// growing back-off so waiting warps leave the issue slots to working ones.
__device__ __forceinline__ void wait_ready(const int32_t *wait, int64_t net) {
    unsigned ns = 32;
    while (ld_acquire(wait + net) > 0) {
        __nanosleep(ns);
        ns = min(ns * 2, 512u);
    }
}

__device__ __forceinline__ void trace_end(int64_t *tr) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[3] = gtimer();
    tr[4] = smid;
}

// One net, start to finish, by `nthr` threads (one warp for a small net, the
// CTA for a big net): wait for its predecessors (dataflow mode), gather,
// leaves, internal nodes level by level (one warp per node), backtrack,
// decisions and the fused commit, then release its successors.
template <bool CTA>
__device__ __forceinline__ void run_net(const NetCtx &c, WarpScr &w, const Shared &sh, const DevGrid &G,
                                        const DevForest &F, const DevScratch &S, const AssignLaunch &a, int64_t net,
                                        int64_t n0, int q_base, int ns, int tid, int nthr, int bar = 0) {
    auto sync = [bar, nthr] { if (CTA) bar_sync(bar, nthr); else __syncwarp(); };
    const int nn = c.nn, lane = threadIdx.x & 31, warp = tid >> 5, nwarps = nthr >> 5;
    const bool flow = a.wait != nullptr;
    const int pdrv = F.net_pdrv[net];
    int64_t *tr = a.trace ? a.trace + 5 * net : nullptr;
    if (tr && tid == 0) tr[0] = gtimer();
    if (flow) {
        if (!CTA || tid == 0) wait_ready(a.wait, net);
        sync();
    }
    if (tr && tid == 0) tr[1] = gtimer();
    gather_nodes(c.nb, F, n0, nn, q_base, ns, tid, nthr);
    sync();
    gather_state(c.nb, G, sh, nn, c.LD, tid, nthr);
    sync();
    if (tr && tid == 0) tr[2] = gtimer();
    int lo = 0;
    while (lo < nn - 1 && c.nb.nd[lo].height == 0) ++lo;
    leaves_dp(c, sh, G, lo, tid, nthr);
    sync();
    while (lo < nn) {
        const int h = c.nb.nd[lo].height;
        int hi = lo + 1;
        while (hi < nn && c.nb.nd[hi].height == h) ++hi;
        for (int i = lo + warp; i < hi; i += nwarps) node_dp_wide(c, w, sh, G, i, pdrv, lane);
        if (CTA) bar_sync(bar, nthr);
        lo = hi;
    }
    if (tid == 0) {
        S.froot[net] = *c.nb.froot;
        c.nb.nd[nn - 1].lay = (uint8_t)pdrv;
    }
    sync();
    // Alg. 4, level-parallel from the root (root entry = driver pin layer, R13)
    for (int hi = nn; hi > 0;) {
        const int h = c.nb.nd[hi - 1].height;
        int l0 = hi - 1;
        while (l0 > 0 && c.nb.nd[l0 - 1].height == h) --l0;
        for (int i = l0 + tid; i < hi; i += nthr) backtrack_node(c, sh, i);
        sync();
        hi = l0;
    }
    for (int i = tid; i < nn; i += nthr) {
        const NodeRec &nd = c.nb.nd[i];
        S.lay[n0 + i] = nd.lay;
        S.sb[n0 + i] = nd.sb;
        S.st[n0 + i] = nd.st;
        if (a.commit) commit_node(G, nd.xy, nd.edir, nd.len, nd.lay, nd.sb, nd.st);
    }
    if (flow) __threadfence();
    sync();
    if (tr && tid == 0) trace_end(tr);
    if (flow)
        for (int64_t e = a.succ_off[net] + tid; e < a.succ_off[net + 1]; e += nthr) atomicSub(a.wait + a.succ[e], 1);
}

// A global slot for a big net that does not fit shared memory: a small pool of slots, each
// guarded by a lock word (the pool is sized by the host budget, not by the grid).
__device__ __forceinline__ int gslot_acquire(const AssignLaunch &a, int hid) {
    int s = hid % a.n_gslots;
    unsigned ns = 64;
    while (atomicCAS(a.glock + s, 0, 1) != 0) {
        s = s + 1 == a.n_gslots ? 0 : s + 1;
        __nanosleep(ns);
        ns = min(ns * 2, 1024u);
    }
    __threadfence();
    return s;
}

__device__ __forceinline__ void gslot_release(const AssignLaunch &a, int s) {
    __threadfence();
    atomicExch(a.glock + s, 0);
}

// ------------------------------------------------------------- group path --
// Batch mode, every net that fits a warp's arena (DESIGN §5 "group path"): an 8-lane GROUP
// runs one net and a warp runs up to four nets side by side (a host-packed "job").  Lane e of
// a group owns entry layer slot e of the node being processed (Alg. 3 l.2-3: one thread per
// (node, layer)); the group walks the net's nodes in forest order (children before parents).
//
// Candidate spans by son-layer combinations (exact).  For a node with sons s_1..s_k and entry
// l, every choice of son layers (j_1..j_k) has a cover span S_c = [min(b0, j..), max(t0, j..)]
// and the value v_c = ((V(S_c) + cost'(j_1)) + ...).  For every span S, v_c >= G'(S_c) (a son's
// window minimum is <= its chosen value; rounded addition is monotone) and the combination of
// S's own window argmins has a cover inside S, hence a value <= G'(S) (V is monotone under
// inclusion because kappa >= 0).  So min_c v_c equals the minimum G' over all spans, bitwise, and
// the key winner (G', t-b, b) of Alg. 3's enumeration is the cover of a minimum-value combination
// with the smallest (t-b, b): the lanes enumerate combinations (LD per son: L-independent loops,
// uniform across the warp's four groups), then take each son's lowest-layer window argmin on the
// winning span (R21) and recompute G with cost (not cost') and K in son order (O6).  V(b, t)
// comes from a per-node table the group builds first, row b summed ascending from b (R10, R23).
// Nodes with three or more sons (rare) sweep the spans directly (group_sweep).
struct NodeG {
    double wd, ur;                    // W_D w_n (Eq. 5), ur (O3)
    uint32_t xy;                      // x | y << 16
    uint16_t len, sink0, nsink, height;
    uint16_t kid[MAXKIDS];            // children (net-local), E W N S order
    uint8_t edir, nkid, nl, nh, lay, sb, st;
};
static_assert(sizeof(NodeG) == 48, "NodeG layout");

struct GLay {
    int node, ac, kap, dec, sink, player, froot, vt, bytes;
};

// One net's DP state in a group's part of the warp arena: node records, (A, C) per (node,
// entry slot) (gathered S first, then O5's A and capb of the parent edge), kappa per (node,
// cut), decisions per (node, slot), sinks (C_q, weight), sink layers and the V(b, t) table of
// the node being processed (triangular, row b from t = b) -- one per group of the team running
// the net (nvt: 1 on the small-net path, 8 or 16 for a big net).
__host__ __device__ inline int vt_elems(int L) { return L * (L + 1) / 2; }

__host__ __device__ inline GLay group_layout(int nn, int ns, int L, int LD, int nvt = 1) {
    GLay w;
    int o = 0;
    auto take = [&](int bytes) { int r = o; o += (bytes + 15) & ~15; return r; };
    w.node = take(48 * nn);
    w.ac = take(16 * nn * LD);
    w.kap = take(8 * nn * (L - 1));
    w.dec = take(4 * nn * LD);
    w.sink = take(16 * ns);
    w.player = take(ns);
    w.froot = take(8);
    w.vt = take(8 * vt_elems(L) * nvt);
    w.bytes = o;
    return w;
}

struct GNet {
    NodeG *nd;
    double2 *AC;
    double *kap, *Vt, *froot;
    uint32_t *dec;
    double2 *sk;
    uint8_t *pl;
};

__device__ __forceinline__ int vtri(int b, int t, int L) { return ((b * (2 * L + 1 - b)) >> 1) + (t - b); }

// O5 cost'(l; s, j) of son s (A, C at its slot for layer j), +inf where the son is infeasible.
__device__ __forceinline__ double cost_p(const double2 ac, double wdk, double vr, double urn) {
    if (!(ac.x < dinf())) return dinf();
    const double Bv = wdk * ac.y;                     // B = wd_s (Cw + D)
    const double cost = ac.x + Bv * vr;
    return cost + Bv * urn;
}

// Nodes with 3 or 4 sons: bottoms b in {b0} U {legal son layers < b0}, descending, tops t in
// {t0} U {legal son layers > t0}, ascending; son k's window minimum is D_k over [b, b0-1]
// (descending, <=: the lower layer wins ties) then the layers [b0, t] (ascending, strict <).
// Returns the key (t-b) << 4 | b (bit 8: no feasible span) and the window argmins in *js.
__device__ __noinline__ uint32_t group_sweep(const Shared &sh, const GNet &n, int i, int l, int b0, int t0, int L,
                                             int LD, uint32_t *js) {
    const NodeG &r = n.nd[i];
    const int nk = r.nkid;
    const double urn = r.ur;
    const double *VRl = sh.T.VR + l * MAXL;
    int kid[MAXKIDS], kdt[MAXKIDS];
    double wdk[MAXKIDS];
    uint32_t legal_any = 0;
#pragma unroll
    for (int k = 0; k < MAXKIDS; ++k) {
        kid[k] = k < nk ? r.kid[k] : 0;
        kdt[k] = k < nk ? (n.nd[kid[k]].edir <= 1 ? 0 : 1) : 2;
        wdk[k] = n.nd[kid[k]].wd;
        if (k < nk) legal_any |= sh.legal[kdt[k]];
    }
    double D[MAXKIDS];
    uint32_t jD = 0;
#pragma unroll
    for (int k = 0; k < MAXKIDS; ++k) D[k] = dinf();
    double bestG = dinf();
    uint32_t bestK = 0x1ffu, bestJ = 0;
    uint32_t rem = legal_any & ((1u << b0) - 1u);
    int b = b0;
    for (;;) {
        double U[MAXKIDS];
        uint32_t jU = jD;
#pragma unroll
        for (int k = 0; k < MAXKIDS; ++k) U[k] = D[k];
#pragma unroll 1
        for (int t = b0; t < L; ++t) {
            const bool son_layer = (legal_any >> t) & 1;
            if (son_layer) {
                const int dtt = sh.dir[t], st = sh.lidx[t];
                const double vr = VRl[t];
#pragma unroll
                for (int k = 0; k < MAXKIDS; ++k)
                    if (kdt[k] == dtt) {
                        const double cp = cost_p(n.AC[kid[k] * LD + st], wdk[k], vr, urn);
                        if (cp < U[k]) {
                            U[k] = cp;
                            jU = (jU & ~(0xfu << (4 * k))) | ((uint32_t)t << (4 * k));
                        }
                    }
            }
            if (t >= t0 && (t == t0 || son_layer)) {
                bool feas = true;
                double g = n.Vt[vtri(b, t, L)];
#pragma unroll
                for (int k = 0; k < MAXKIDS; ++k)
                    if (k < nk) {
                        feas = feas && U[k] < dinf();
                        g = g + U[k];
                    }
                const uint32_t key = (uint32_t)(((t - b) << 4) | b);
                if (feas && (g < bestG || (g == bestG && key < bestK))) {
                    bestG = g;
                    bestK = key;
                    bestJ = jU;
                }
            }
        }
        if (!rem) break;
        b = 31 - __clz(rem);                        // next candidate bottom, descending
        rem &= ~(1u << b);
        const int dtb = sh.dir[b], sbb = sh.lidx[b];
        const double vr = VRl[b];
#pragma unroll
        for (int k = 0; k < MAXKIDS; ++k)
            if (kdt[k] == dtb) {
                const double cp = cost_p(n.AC[kid[k] * LD + sbb], wdk[k], vr, urn);
                if (cp < dinf() && cp <= D[k]) {
                    D[k] = cp;
                    jD = (jD & ~(0xfu << (4 * k))) | ((uint32_t)b << (4 * k));
                }
            }
    }
    *js = bestJ;
    return bestK;
}


// Reduction of a candidate (G', key) over the P parts of an entry (lanes part * 8 + e).
template <int P>
__device__ __forceinline__ void reduce_best(double &g, uint32_t &key) {
    if constexpr (P > 1) {
#pragma unroll
        for (int o = 8; o < 8 * P; o <<= 1) {
            const double og = __shfl_xor_sync(FULL_MASK, g, o);
            const uint32_t ok = __shfl_xor_sync(FULL_MASK, key, o);
            if (og < g || (og == g && ok < key)) { g = og; key = ok; }
        }
    }
}

// Reduction of a son's window argmin (value, layer) over the P parts: the lowest layer among the minima.
template <int P>
__device__ __forceinline__ void reduce_argmin(double &m, int &j) {
    if constexpr (P > 1) {
#pragma unroll
        for (int o = 8; o < 8 * P; o <<= 1) {
            const double om = __shfl_xor_sync(FULL_MASK, m, o);
            const int oj = __shfl_xor_sync(FULL_MASK, j, o);
            if (om < m || (om == m && oj < j)) { m = om; j = oj; }
        }
    }
}

// Node i, entry layer l (slot e; the root: l = p_drv, slot 0).  P = 1: one lane per entry (the
// small-net path; the caller passes only active lanes).  P = 4: a whole warp per node (big nets),
// lane = part * 8 + e; the parts split the son-layer slots of the combination search (slot s in
// part s % P) and reduce by the same total orders, so the choice is the P = 1 one; every lane
// calls (act = an entry of the node), part 0 writes.
template <int P>
__device__ __forceinline__ void group_node(const Shared &sh, const DevGrid &G, const GNet &n, int i, bool root,
                                           int l, int e, int part, bool act, int L, int LD, double *froot) {
    constexpr int NSP = MAXE / P;                       // son-layer slots per part
    const NodeG &r = n.nd[i];
    const int nk = r.nkid;
    // pin terms, sinks in input order (Alg. 3 l.4-7)
    double F0 = 0.0, C0 = 0.0;
#pragma unroll 1
    for (int q = r.sink0; q < r.sink0 + r.nsink; ++q) {
        const double2 c = n.sk[q];
        F0 = F0 + c.y * (c.x * sh.T.VR[n.pl[q] * MAXL + l]);
        C0 = C0 + c.x;
    }
    const int nl = r.nl, nh = r.nh;
    const bool pins = nl != 255;
    const int b0 = pins ? min(l, nl) : l, t0 = pins ? max(l, nh) : l;
    const double *kp = n.kap + i * (L - 1);
    const double *VRl = sh.T.VR + l * MAXL;
    double Gv, K = 0.0;
    int bw = b0, tw = t0;
    uint32_t js = 0;
    if (nk == 0) {
        // leaf: G' = V(b, t) >= V(b0, t0) on every admissible span (kappa >= 0), so (b0, t0)
        double V = 0.0;
#pragma unroll 1
        for (int k = 0; k < L - 1; ++k)
            if (k >= b0 && k < t0) V = V + kp[k];
        Gv = V;
    } else {
        const double urn = r.ur;
        uint32_t key = 0x1ffu;
        const int k0 = r.kid[0], k1 = nk > 1 ? r.kid[1] : 0;
        const int d0 = n.nd[k0].edir <= 1 ? 0 : 1, d1 = n.nd[k1].edir <= 1 ? 0 : 1;
        const double w0 = n.nd[k0].wd, w1 = n.nd[k1].wd;
        const double2 *ac0 = n.AC + k0 * LD, *ac1 = n.AC + k1 * LD;
        if (nk == 1) {
            // son-layer combinations (header): cost' per slot in registers, independent loads and
            // evaluations, then a compare chain in ascending slot order
            double c0[NSP];
            const int n0 = sh.ndir[d0];
            double bestG = dinf();
#pragma unroll
            for (int k = 0; k < NSP; ++k) {
                const int s = part + k * P;
                const int j = sh.lay_of[d0][s];
                c0[k] = s < n0 ? cost_p(ac0[s], w0, VRl[j], urn) : dinf();
                const int bb = min(b0, j), tt = max(t0, j);
                const double g = n.Vt[vtri(bb, tt, L)] + c0[k];
                const uint32_t kk = (uint32_t)(((tt - bb) << 4) | bb);
                if (c0[k] < dinf() && (g < bestG || (g == bestG && kk < key))) { bestG = g; key = kk; }
            }
            reduce_best<P>(bestG, key);
            bw = key & 0xf;
            tw = bw + (int)((key >> 4) & 0xf);
            double m = dinf();
            int jm = MAXL;
#pragma unroll
            for (int k = 0; k < NSP; ++k) {                 // the son's lowest-layer window argmin (R21)
                const int j = sh.lay_of[d0][part + k * P];
                if (j >= bw && j <= tw && c0[k] < m) { m = c0[k]; jm = j; }
            }
            reduce_argmin<P>(m, jm);
            js = (uint32_t)jm & 0xf;
        } else if (nk == 2) {
            // son-layer combinations; son 1's cost' per slot in registers, son 0 per outer step
            double c1[MAXE];
            const int n0 = sh.ndir[d0], n1 = sh.ndir[d1];
#pragma unroll
            for (int s = 0; s < MAXE; ++s) c1[s] = s < n1 ? cost_p(ac1[s], w1, VRl[sh.lay_of[d1][s]], urn) : dinf();
            double bestG = dinf();
#pragma unroll 1
            for (int s0 = part; s0 < n0; s0 += P) {
                const int j0 = sh.lay_of[d0][s0];
                const double c0 = cost_p(ac0[s0], w0, VRl[j0], urn);
                if (!(c0 < dinf())) continue;
                const int bb = min(b0, j0), tt = max(t0, j0);
#pragma unroll
                for (int s1 = 0; s1 < MAXE; ++s1) {
                    const int j1 = sh.lay_of[d1][s1];
                    const int b = min(bb, j1), t = max(tt, j1);
                    const double g = (n.Vt[vtri(b, t, L)] + c0) + c1[s1];
                    const uint32_t kk = (uint32_t)(((t - b) << 4) | b);
                    if (c1[s1] < dinf() && (g < bestG || (g == bestG && kk < key))) { bestG = g; key = kk; }
                }
            }
            reduce_best<P>(bestG, key);
            bw = key & 0xf;
            tw = bw + (int)((key >> 4) & 0xf);
            double m = dinf();
            int jm = MAXL;
#pragma unroll
            for (int k = 0; k < NSP; ++k) {                 // son 0's window argmin over this part's slots
                const int s = part + k * P;
                const int j = sh.lay_of[d0][s];
                if (s < n0 && j >= bw && j <= tw) {
                    const double cp = cost_p(ac0[s], w0, VRl[j], urn);
                    if (cp < m) { m = cp; jm = j; }
                }
            }
            reduce_argmin<P>(m, jm);
            js = (uint32_t)jm & 0xf;
            m = dinf();
            jm = 0;
#pragma unroll
            for (int s = 0; s < MAXE; ++s) {
                const int j = sh.lay_of[d1][s];
                if (j >= bw && j <= tw && c1[s] < m) { m = c1[s]; jm = j; }
            }
            js |= (uint32_t)jm << 4;
        } else {
            key = group_sweep(sh, n, i, l, b0, t0, L, LD, &js);
            bw = key & 0xf;
            tw = bw + (int)((key >> 4) & 0xf);
        }
        if (!act || part != 0) return;
        if (key & 0x100u) {                             // no feasible span (cannot happen when every
            if (root) *froot = dinf();                  // direction has a routable layer; kept exact)
            else n.AC[i * LD + e].x = dinf();
            return;
        }
        Gv = n.Vt[vtri(bw, tw, L)];
#pragma unroll
        for (int k = 0; k < MAXKIDS; ++k)
            if (k < nk) {
                const int kk = r.kid[k];
                const int j = (js >> (4 * k)) & 0xf;
                const double2 ac = n.AC[kk * LD + sh.lidx[j]];
                const double Bv = n.nd[kk].wd * ac.y;
                Gv = Gv + (ac.x + Bv * VRl[j]);
                K = K + ac.y;
            }
    }
    if (!act || part != 0) return;
    const double f = F0 + Gv;
    const double dlc = C0 + K;
    n.dec[i * LD + e] = (uint32_t)(bw | (tw << 4)) | (js << 8);
    if (root) {
        *froot = f;
        return;
    }
    double2 &o = n.AC[i * LD + e];
    const double Sc = o.x;                              // congestion sum gathered up front
    const double len = (double)r.len;
    const double Rw = sh.T.r[l] * len;
    const double Cw = sh.T.c[l] * len;
    o.x = ((f + r.wd * (Rw * (0.5 * Cw + dlc))) + G.W_CAP * Cw) + (G.W_CONG * sh.T.ofw[l]) * Sc;
    o.y = Cw + dlc;
}

__device__ __forceinline__ GNet group_net(char *base, const GLay &lay) {
    GNet n;
    n.nd = (NodeG *)(base + lay.node);
    n.AC = (double2 *)(base + lay.ac);
    n.kap = (double *)(base + lay.kap);
    n.dec = (uint32_t *)(base + lay.dec);
    n.sk = (double2 *)(base + lay.sink);
    n.pl = (uint8_t *)(base + lay.player);
    n.froot = (double *)(base + lay.froot);
    n.Vt = (double *)(base + lay.vt);
    return n;
}

// Gather (a3) by threads tid of nthr: node records, sinks, kappa per (node, cut) and the
// congestion sum S per (non-root node, entry slot) -- all loads of the net in flight at once.
__device__ __forceinline__ void group_gather(const GNet &n, const Shared &sh, const DevGrid &G, const DevForest &F,
                                             int64_t n0, int nn, int ns, int q_base, int LD, int tid, int nthr) {
    const int Lm1 = G.L - 1;
    for (int i = tid; i < nn; i += nthr) {
        const int64_t nid = n0 + i;
        NodeG r;
        r.wd = F.wd[nid];
        r.ur = F.ur[nid];
        r.xy = F.xy[nid];
        r.len = (uint16_t)F.len[nid];
        r.sink0 = (uint16_t)(F.sink0[nid] - q_base);
        r.nsink = F.nsink[nid];
        r.height = F.height[nid];
        const int4 k4 = *reinterpret_cast<const int4 *>(F.kid + nid * 4);
        r.kid[0] = (uint16_t)(k4.x - n0);
        r.kid[1] = (uint16_t)(k4.y - n0);
        r.kid[2] = (uint16_t)(k4.z - n0);
        r.kid[3] = (uint16_t)(k4.w - n0);
        r.edir = F.edir[nid];
        r.nkid = F.nkid[nid];
        r.nl = F.nl[nid];
        r.nh = F.nh[nid];
        r.lay = r.sb = r.st = 0;
        n.nd[i] = r;
    }
    for (int q = tid; q < ns; q += nthr) {
        n.pl[q] = F.p_layer[q_base + q];
        n.sk[q] = make_double2(F.p_cap[q_base + q], F.p_w[q_base + q]);
    }
    if (nthr >= 16) {
        // a team (big net, latency-bound): chunks of 4 items per thread, the chunk's via words all
        // in flight before the dependent Eq. (3) table lookups
        const int nk_items = nn * Lm1;
#pragma unroll 1
        for (int base = 0; base < nk_items; base += 4 * nthr) {
            int32_t wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int idx = base + tid + u * nthr;
                wv[u] = 0;
                if (idx < nk_items) {
                    const int i = idx / Lm1, k = idx - i * Lm1;
                    const uint32_t xy = __ldg(F.xy + n0 + i);
                    wv[u] = __ldcg(G.via + ((int64_t)(xy >> 16) * G.X + (xy & 0xffff)) * Lm1 + k);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int idx = base + tid + u * nthr;
                if (idx < nk_items) n.kap[idx] = kappa_w(G, sh, wv[u], idx % Lm1);
            }
        }
    } else {
        for (int idx = tid; idx < nn * Lm1; idx += nthr) {
            const int i = idx / Lm1, k = idx - i * Lm1;
            const uint32_t xy = __ldg(F.xy + n0 + i);
            n.kap[idx] = kappa_w(G, sh, __ldcg(G.via + ((int64_t)(xy >> 16) * G.X + (xy & 0xffff)) * Lm1 + k), k);
        }
    }
    for (int idx = tid; idx < (nn - 1) * LD; idx += nthr) {
        const int i = idx / LD, s = idx - i * LD;
        const int64_t nid = n0 + i;
        const int ed = __ldg(F.edir + nid);
        const int dt = ed <= 1 ? 0 : 1;
        if (s >= sh.ndir[dt]) continue;
        double Sc = dinf();
        if (sh.routable[sh.lay_of[dt][s]]) {
            const uint32_t xy = __ldg(F.xy + nid);
            Sc = run_sum(G, dt, s, xy & 0xffff, xy >> 16, ed, __ldg(F.len + nid));
        }
        n.AC[idx].x = Sc;
    }
}

// V(b, t) table of node i by the 8 lanes of a group: row b summed ascending from b (R10, R23).
__device__ __forceinline__ void group_vtable(const GNet &n, int i, int L, int gl) {
    const double *kp = n.kap + i * (L - 1);
    for (int b = gl; b < L; b += 8) {
        double *row = n.Vt + vtri(b, b, L);
        double V = 0.0;
        row[0] = V;
#pragma unroll 1
        for (int t = b + 1; t < L; ++t) {
            V = V + kp[t - 1];
            row[t - b] = V;
        }
    }
}

// Node i: P = 1, one group (lanes gl = entry slots); P = 4, a whole warp (lane = part * 8 + entry).
template <int P>
__device__ __forceinline__ void group_step(const GNet &n, const Shared &sh, const DevGrid &G, int i, int nn, int pdrv,
                                           int L, int LD, int lane) {
    const int e = lane & 7, part = P > 1 ? (lane >> 3) : 0;
    const bool root = i == nn - 1;
    const int ed = n.nd[i].edir;
    const int dt = ed <= 1 ? 0 : 1;
    const int nE = root ? 1 : sh.ndir[dt];
    const int l = root ? pdrv : sh.lay_of[dt][e];
    const bool act = e < nE && (root || sh.routable[l]);
    if (P == 1 && !act) return;
    group_node<P>(sh, G, n, i, root, act ? l : 0, e, part, act, L, LD, n.froot);
}

// Alg. 4 backtrack from the root (entry = driver pin layer, R13) by one thread: parents precede
// children in reverse forest order.
__device__ __forceinline__ void group_backtrack(const GNet &n, const Shared &sh, int nn, int pdrv, int LD) {
    n.nd[nn - 1].lay = (uint8_t)pdrv;
#pragma unroll 1
    for (int i = nn - 1; i >= 0; --i) {
        NodeG &r = n.nd[i];
        const int slot = i == nn - 1 ? 0 : sh.lidx[r.lay];
        const uint32_t d = n.dec[i * LD + slot];
        r.sb = d & 0xf;
        r.st = (d >> 4) & 0xf;
        const uint32_t jj = d >> 8;
#pragma unroll 1
        for (int k = 0; k < r.nkid; ++k) n.nd[r.kid[k]].lay = (uint8_t)((jj >> (4 * k)) & 0xf);
    }
}

// Decisions to HBM and the fused commit (O8), threads tid of nthr over the nodes.
__device__ __forceinline__ void group_emit(const GNet &n, const DevGrid &G, const DevScratch &S, const AssignLaunch &a,
                                           int64_t n0, int nn, int tid, int nthr) {
    for (int i = tid; i < nn; i += nthr) {
        const NodeG &r = n.nd[i];
        S.lay[n0 + i] = r.lay;
        S.sb[n0 + i] = r.sb;
        S.st[n0 + i] = r.st;
        if (a.commit) commit_node(G, r.xy, r.edir, r.len, r.lay, r.sb, r.st);
    }
}

// One small net by one group (lanes gl = 0..7; nn = 0: no net): gather, nodes in forest order
// (children before parents), backtrack, commit.  Called by all 32 lanes of the warp: the node
// loop runs to the largest node count of the warp's nets with a full-warp reconvergence point
// after every node, so the four groups execute each node step together (independent thread
// scheduling would otherwise let them drift apart for good).
__device__ __forceinline__ void run_net_group(char *base, const Shared &sh, const DevGrid &G, const DevForest &F,
                                              const DevScratch &S, const AssignLaunch &a, int64_t net, int64_t n0,
                                              int nn, int ns, int q_base, int gl) {
    const int L = G.L, LD = a.LD;
    const GNet n = group_net(base, group_layout(nn, ns, L, LD));
    int64_t *tr = (a.trace && nn > 0) ? a.trace + 5 * net : nullptr;
    if (tr && gl == 0) tr[0] = tr[1] = gtimer();
    const int pdrv = nn > 0 ? F.net_pdrv[net] : 0;
    group_gather(n, sh, G, F, n0, nn, ns, q_base, LD, gl, 8);
    const int nmax = __reduce_max_sync(FULL_MASK, (unsigned)nn);
    __syncwarp();
    if (tr && gl == 0) tr[2] = gtimer();
#pragma unroll 1
    for (int i = 0; i < nmax; ++i) {
        const bool act = i < nn;
        if (act && n.nd[i].nkid > 0) group_vtable(n, i, L, gl);
        __syncwarp();
        if (act) group_step<1>(n, sh, G, i, nn, pdrv, L, LD, gl);
        __syncwarp();
    }
    if (gl == 0 && nn > 0) {
        S.froot[net] = *n.froot;
        group_backtrack(n, sh, nn, pdrv, LD);
    }
    __syncwarp();
    group_emit(n, G, S, a, n0, nn, gl, 8);
    if (tr && gl == 0) trace_end(tr);
}

// One big net by a team (a half-CTA or the CTA: nthr threads = nthr / 32 warps, named barrier
// `bar`): gather, then each height level's nodes spread over the warps (a whole warp per node:
// group_node<4>, V table per warp), a team barrier between levels; backtrack by one thread; commit.
__device__ __forceinline__ void run_net_team(char *base, const Shared &sh, const DevGrid &G, const DevForest &F,
                                             const DevScratch &S, const AssignLaunch &a, int64_t net, int64_t n0,
                                             int nn, int ns, int q_base, int tid, int nthr, int bar) {
    const int L = G.L, LD = a.LD, T = nthr >> 5, wid = tid >> 5, lane = tid & 31;
    GNet n = group_net(base, group_layout(nn, ns, L, LD, T));
    n.Vt += wid * vt_elems(L);
    int64_t *tr = a.trace ? a.trace + 5 * net : nullptr;
    if (tr && tid == 0) tr[0] = gtimer();
    const int pdrv = F.net_pdrv[net];
    group_gather(n, sh, G, F, n0, nn, ns, q_base, LD, tid, nthr);
    bar_sync(bar, nthr);
    if (tr && tid == 0) tr[2] = gtimer();
    int lo = 0;
    while (lo < nn) {
        const int h = n.nd[lo].height;
        int hi = lo + 1;
        while (hi < nn && n.nd[hi].height == h) ++hi;
#pragma unroll 1
        for (int i = lo + wid; i < hi; i += T) {
            if (n.nd[i].nkid > 0) {        // V(b, t) table of node i, lane b sums row b ascending (R10, R23)
                if (lane < L) {
                    const double *kp = n.kap + i * (L - 1);
                    double *row = n.Vt + vtri(lane, lane, L);
                    double V = 0.0;
                    row[0] = V;
#pragma unroll 1
                    for (int t = lane + 1; t < L; ++t) {
                        V = V + kp[t - 1];
                        row[t - lane] = V;
                    }
                }
                __syncwarp();
            }
            group_step<4>(n, sh, G, i, nn, pdrv, L, LD, lane);
            __syncwarp();
        }
        bar_sync(bar, nthr);
        lo = hi;
    }
    if (tr && tid == 0) tr[1] = gtimer();             // team nets: [1] = end of the level loop
    // Alg. 4, level-parallel from the root: the nodes of one height level take their entry layer
    // from their parents (a level above) and set their sons'
    if (tid == 0) {
        S.froot[net] = *n.froot;
        n.nd[nn - 1].lay = (uint8_t)pdrv;
    }
    bar_sync(bar, nthr);
    for (int hi = nn; hi > 0;) {
        const int h = n.nd[hi - 1].height;
        int l0 = hi - 1;
        while (l0 > 0 && n.nd[l0 - 1].height == h) --l0;
        for (int i = l0 + tid; i < hi; i += nthr) {
            NodeG &r = n.nd[i];
            const int slot = i == nn - 1 ? 0 : sh.lidx[r.lay];
            const uint32_t d = n.dec[i * LD + slot];
            r.sb = d & 0xf;
            r.st = (d >> 4) & 0xf;
            const uint32_t jj = d >> 8;
#pragma unroll 1
            for (int k = 0; k < r.nkid; ++k) n.nd[r.kid[k]].lay = (uint8_t)((jj >> (4 * k)) & 0xf);
        }
        bar_sync(bar, nthr);
        hi = l0;
    }
    group_emit(n, G, S, a, n0, nn, tid, nthr);
    if (tr && tid == 0) trace_end(tr);
}

// ------------------------------------------------------------------ kernel --
// Two register budgets of the same kernel: MINB = ASSIGN_CTAS_LAT (6 CTAs/SM, 80 registers) for
// launches bound by their slowest net (fewer spills on the serial path), MINB = ASSIGN_CTAS_THR
// (7 CTAs/SM, 72 registers) for throughput-bound launches (more resident warps hide latency).
template <int MINB>
__global__ void __launch_bounds__(ASSIGN_WARPS * 32, MINB) k_assign(DevGrid G, DevForest F, DevScratch S, AssignLaunch a) {
    __shared__ Shared sh;
    __shared__ int64_t big_item[2];
    __shared__ int big_gslot[2];
    extern __shared__ __align__(16) char dyn[];
    stage_tab(sh.T, G.tab);
    if (threadIdx.x < 2 * MAXL) sh.lay_of[threadIdx.x / MAXL][threadIdx.x % MAXL] = 0;   // unused slots: layer 0
    __syncthreads();
    if (threadIdx.x < MAXL) {
        const int l = threadIdx.x;
        sh.dir[l] = G.dir[l];
        sh.routable[l] = G.routable[l];
        sh.lidx[l] = (uint8_t)G.lidx[l];
        if (l < G.L) sh.lay_of[G.dir[l]][G.lidx[l]] = (uint8_t)l;
    }
    if (threadIdx.x == 0) {
        sh.ndir[0] = G.LH;
        sh.ndir[1] = G.LV;
        uint32_t m0 = 0, m1 = 0;
        for (int l = 0; l < G.L; ++l)
            if (G.routable[l]) (G.dir[l] == 0 ? m0 : m1) |= 1u << l;
        sh.legal[0] = m0;
        sh.legal[1] = m1;
    }
    __syncthreads();
    const int L = G.L, LD = a.LD;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const NetLay slay = net_layout(a.NS, a.NP, L, LD);
    WarpScr w = warp_scr(dyn + ASSIGN_WARPS * slay.bytes + warp * scr_bytes(L, LD), L, LD);

    // hybrid (batch mode: no waits): every CTA first takes big nets, then small ones
    if (a.hybrid || (int)blockIdx.x < a.n_big_ctas) {
        // ---------------- big nets: each half-CTA (2 warps) per net ----------------
        // (a whole CTA idles at the level barriers of chain-like trees; two nets per CTA
        // halve that).  DP state in the half's two slots, a global slot beyond that.
        // (big_split == 0: the whole CTA per net, for latency-bound launches with few nets)
        const bool split = a.big_split != 0;
        const int half = split ? warp >> 1 : 0, gsz = split ? 64 : 128;
        const int htid = threadIdx.x & (gsz - 1), bar = split ? 1 + half : 0;
        const int nslots = split ? 2 : ASSIGN_WARPS;
        const int64_t n_work = a.big_end - a.big_beg;
        for (;;) {
            bar_sync(bar, gsz);
            if (htid == 0) big_item[half] = (int64_t)atomicAdd(a.ticket + 1, 1ull);
            bar_sync(bar, gsz);
            const int64_t wk = big_item[half];
            if (wk >= n_work) {
                if (a.hybrid) break;
                return;
            }
            const int4 rec = a.big_pos[a.big_beg + wk];
            const int64_t net = rec.x, n0 = (uint32_t)rec.y;
            const int nn = rec.z & 0xffff, ns = (int)((uint32_t)rec.z >> 16), q_base = rec.w;
            const NetLay lay = net_layout(nn, ns, L, LD);
            char *base = dyn + (int64_t)half * nslots * slay.bytes;
            const bool glob = lay.bytes > nslots * slay.bytes;
            if (glob) {
                // a pooled global slot, taken only once the net may start (dataflow: its
                // predecessors are done), so a slot holder never waits on another net
                if (htid == 0) {
                    if (a.wait) wait_ready(a.wait, net);
                    big_gslot[half] = gslot_acquire(a, blockIdx.x * 2 + half);
                }
                bar_sync(bar, gsz);
                base = a.gscratch + (int64_t)big_gslot[half] * a.gslot_bytes;
            }
            const NetCtx c{net_buf(base, lay), L, LD, nn};
            run_net<true>(c, w, sh, G, F, S, a, net, n0, q_base, ns, htid, gsz, bar);
            if (glob && htid == 0) gslot_release(a, big_gslot[half]);
        }
    }

    // ---------------- small nets: one warp per net ----------------
    // The ticket of the next net is taken before the current one runs, so its atomic
    // round trip overlaps the DP.
    char *mine = dyn + warp * slay.bytes;
    const int64_t n_work = a.small_end - a.small_beg;
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1ull);
    tk = __shfl_sync(FULL_MASK, tk, 0);
    for (;;) {
        if ((int64_t)tk >= n_work) return;
        const int4 rec = a.small_pos[a.small_beg + (int64_t)tk];
        unsigned long long tk_next = 0;
        if (lane == 0) tk_next = atomicAdd(a.ticket, 1ull);
        const int64_t net = rec.x, n0 = (uint32_t)rec.y;
        const int nn = rec.z & 0xffff, ns = (int)((uint32_t)rec.z >> 16), q_base = rec.w;
        const NetCtx c{net_buf(mine, slay), L, LD, nn};
        run_net<false>(c, w, sh, G, F, S, a, net, n0, q_base, ns, lane, 32);
        __syncwarp();
        tk = __shfl_sync(FULL_MASK, tk_next, 0);
    }
}

// Batch mode kernel (la_assign_batch): every CTA first takes the batch's big nets (a half-CTA or
// the whole CTA per net, wide-node DP as in k_assign), then each warp takes host-packed JOBS of
// up to four nets that fit its arena, one 8-lane group per net (group path above).  Shared
// memory: four warp arenas of a.warp_arena bytes; a big net uses its half's (or the CTA's)
// arenas, with the wide-node scratch of its warps carved from the region's end.
template <int MINB>
__global__ void __launch_bounds__(ASSIGN_WARPS * 32, MINB) k_assign_g(DevGrid G, DevForest F, DevScratch S,
                                                                      AssignLaunch a) {
    __shared__ Shared sh;
    __shared__ int64_t big_item[2];
    __shared__ int gslot_of[2];
    extern __shared__ __align__(16) char dyn[];
    stage_tab(sh.T, G.tab);
    if (threadIdx.x < 2 * MAXL) sh.lay_of[threadIdx.x / MAXL][threadIdx.x % MAXL] = 0;   // unused slots: layer 0
    __syncthreads();
    if (threadIdx.x < MAXL) {
        const int l = threadIdx.x;
        sh.dir[l] = G.dir[l];
        sh.routable[l] = G.routable[l];
        sh.lidx[l] = (uint8_t)G.lidx[l];
        if (l < G.L) sh.lay_of[G.dir[l]][G.lidx[l]] = (uint8_t)l;
    }
    if (threadIdx.x == 0) {
        sh.ndir[0] = G.LH;
        sh.ndir[1] = G.LV;
        uint32_t m0 = 0, m1 = 0;
        for (int l = 0; l < G.L; ++l)
            if (G.routable[l]) (G.dir[l] == 0 ? m0 : m1) |= 1u << l;
        sh.legal[0] = m0;
        sh.legal[1] = m1;
    }
    __syncthreads();
    const int L = G.L, LD = a.LD, WA = a.warp_arena;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // ---------------- big nets: a team (half-CTA or CTA) per net, level-parallel groups ----------------
    if (a.big_end > a.big_beg) {
        const bool split = a.big_split != 0;
        const int half = split ? warp >> 1 : 0, gsz = split ? 64 : 128, nw = gsz >> 5;
        const int htid = threadIdx.x & (gsz - 1), bar = split ? 1 + half : 0;
        char *region = dyn + (int64_t)half * 2 * WA;
        const int cap = nw * WA;
        const int64_t n_work = a.big_end - a.big_beg;
        for (;;) {
            bar_sync(bar, gsz);
            if (htid == 0) big_item[half] = (int64_t)atomicAdd(a.ticket + 1, 1ull);
            bar_sync(bar, gsz);
            const int64_t wk = big_item[half];
            if (wk >= n_work) break;
            const int4 rec = a.big_pos[a.big_beg + wk];
            const int64_t net = rec.x, n0 = (uint32_t)rec.y;
            const int nn = rec.z & 0xffff, ns = (int)((uint32_t)rec.z >> 16), q_base = rec.w;
            char *base = region;
            const bool glob = group_layout(nn, ns, L, LD, gsz >> 5).bytes > cap;
            if (glob) {
                if (htid == 0) gslot_of[half] = gslot_acquire(a, blockIdx.x * 2 + half);
                bar_sync(bar, gsz);
                base = a.gscratch + (int64_t)gslot_of[half] * a.gslot_bytes;
            }
            run_net_team(base, sh, G, F, S, a, net, n0, nn, ns, q_base, htid, gsz, bar);
            if (glob && htid == 0) gslot_release(a, gslot_of[half]);
        }
    }

    // ---------------- jobs: up to four nets per warp, one 8-lane group per net ----------------
    char *arena = dyn + (int64_t)warp * WA;
    const int g = lane >> 3, gl = lane & 7;
    const int64_t n_work = a.job_end - a.job_beg;
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1ull);
    tk = __shfl_sync(FULL_MASK, tk, 0);
    for (;;) {
        if ((int64_t)tk >= n_work) return;
        const int4 job = a.jobs[a.job_beg + (int64_t)tk];   // {first small index, count, off1 | off2 << 16, off3}
        unsigned long long tk_next = 0;
        if (lane == 0) tk_next = atomicAdd(a.ticket, 1ull);
        {
            const bool have = g < job.y;
            const int off = g == 0 ? 0 : g == 1 ? (job.z & 0xffff) : g == 2 ? ((uint32_t)job.z >> 16) : job.w;
            const int4 rec = have ? a.small_pos[(int64_t)job.x + g] : make_int4(0, 0, 0, 0);
            const int64_t net = rec.x, n0 = (uint32_t)rec.y;
            const int nn = rec.z & 0xffff, ns = (int)((uint32_t)rec.z >> 16), q_base = rec.w;
            run_net_group(arena + off, sh, G, F, S, a, net, n0, nn, ns, q_base, gl);
        }
        __syncwarp();
        tk = __shfl_sync(FULL_MASK, tk_next, 0);
    }
}

}  // namespace

size_t assign_group_net_bytes(int nodes, int sinks, int L, int LD) {
    return (size_t)group_layout(nodes, sinks, L, LD).bytes;
}

size_t assign_team_net_bytes(int nodes, int sinks, int L, int LD) {   // a big net run by a whole CTA (16 groups)
    return (size_t)group_layout(nodes, sinks, L, LD, 16).bytes;
}

size_t assign_warp_arena_bytes(int L, int LD) {
    (void)L;
    (void)LD;
    return (size_t)G_WARP_ARENA;
}

size_t assign_smem_bytes(int L, int LD, int NS, int NP) {
    return (size_t)ASSIGN_WARPS * (net_layout(NS, NP, L, LD).bytes + scr_bytes(L, LD));
}

size_t assign_net_bytes(int nodes, int sinks, int L, int LD) { return (size_t)net_layout(nodes, sinks, L, LD).bytes; }

int assign_nets_per_cta() { return ASSIGN_WARPS; }

size_t assign_cta_net_bytes(int L, int LD, int NS, int NP) {   // shared memory of one big net (half-CTA)
    return (size_t)2 * net_layout(NS, NP, L, LD).bytes;
}

template <int MINB>
static cudaError_t resident(size_t smem, int *per_sm) {
    cudaError_t e = cudaFuncSetAttribute(k_assign<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_assign<MINB>, ASSIGN_WARPS * 32, smem);
}

cudaError_t assign_resident_ctas(int L, int LD, int NS, int NP, int *per_sm_lat, int *per_sm_thr, int *n_sm) {
    const size_t smem = assign_smem_bytes(L, LD, NS, NP);
    cudaError_t e = resident<ASSIGN_CTAS_LAT>(smem, per_sm_lat);
    if (e != cudaSuccess) return e;
    e = resident<ASSIGN_CTAS_THR>(smem, per_sm_thr);
    if (e != cudaSuccess) return e;
    int dev = 0;
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    return cudaDeviceGetAttribute(n_sm, cudaDevAttrMultiProcessorCount, dev);
}

template <int MINB>
static cudaError_t launch(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a, int grid,
                          size_t smem, cudaStream_t s) {
    if (a.wait) {
        // dataflow mode: every CTA must be co-resident (nets wait on each other)
        void *args[] = {(void *)&G, (void *)&F, (void *)&S, (void *)&a};
        return cudaLaunchCooperativeKernel((const void *)k_assign<MINB>, dim3(grid), dim3(ASSIGN_WARPS * 32), args, smem, s);
    }
    k_assign<MINB><<<(unsigned)grid, ASSIGN_WARPS * 32, smem, s>>>(G, F, S, a);
    return cudaGetLastError();
}

template <int MINB>
static cudaError_t resident_g(size_t smem, int *per_sm) {
    cudaError_t e = cudaFuncSetAttribute(k_assign_g<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_assign_g<MINB>, ASSIGN_WARPS * 32, smem);
}

cudaError_t assign_g_resident_ctas(int L, int LD, int *per_sm_lat, int *per_sm_thr) {
    const size_t smem = (size_t)ASSIGN_WARPS * assign_warp_arena_bytes(L, LD);
    cudaError_t e = resident_g<G_CTAS_LAT>(smem, per_sm_lat);
    if (e != cudaSuccess) return e;
    return resident_g<G_CTAS_THR>(smem, per_sm_thr);
}

cudaError_t launch_assign_g(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a, int grid,
                            bool throughput, cudaStream_t s) {
    if ((a.job_end <= a.job_beg && a.big_end <= a.big_beg) || grid <= 0) return cudaSuccess;
    const size_t smem = (size_t)ASSIGN_WARPS * a.warp_arena;
    if (throughput) k_assign_g<G_CTAS_THR><<<(unsigned)grid, ASSIGN_WARPS * 32, smem, s>>>(G, F, S, a);
    else k_assign_g<G_CTAS_LAT><<<(unsigned)grid, ASSIGN_WARPS * 32, smem, s>>>(G, F, S, a);
    return cudaGetLastError();
}

cudaError_t launch_assign(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a, int grid,
                          bool throughput, cudaStream_t s) {
    if ((a.small_end <= a.small_beg && a.big_end <= a.big_beg) || grid <= 0) return cudaSuccess;
    const size_t smem = assign_smem_bytes(G.L, a.LD, a.NS, a.NP);
    return throughput ? launch<ASSIGN_CTAS_THR>(G, F, S, a, grid, smem, s) : launch<ASSIGN_CTAS_LAT>(G, F, S, a, grid, smem, s);
}

}  // namespace gapla
