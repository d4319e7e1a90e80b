/*
 * oracle/la_oracle.cpp -- plain, slow, sequential fp64 CPU oracle for GAP-LA's
 * layer-assignment hot path (arXiv 2507.13375, "PAPER.md" below).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2507_13375_b200/) never links, imports or executes anything here, and
 * this file shares no code, header, table or constant generator with it.
 *
 * What it computes (with the readings R1..R40 of
 * §8(c) c.4 restated in DESIGN.md "Readings"):
 *   O1 LA directed tree              PAPER.md §III-B l.264-281 (Fig. 6)
 *   O2 pin / edge weights Eq.(4)(5)  §III-C l.307-320
 *   O3 upstream-R estimate ur        §III-D l.452
 *   O4 Eq.(3) marginal tables, VR    §II-E l.178-182, Alg. 2 inputs l.339-340
 *   O5/O6 bottom-up DP (Alg. 3)      l.355-411, text l.440-463
 *   O7 backtrack (Alg. 4)            l.418-435
 *   O8 demand commit                 Alg. 2 input D l.343, §III-A l.224-226
 *   O9 Elmore / downstream cap       §II-C l.146, §III-D l.443-444 (Fig. 8)
 * plus the sequential conflict-free batch recurrence.
 *
 * Nets are processed one at a time in (order_key, index) order, each committed
 * before the next (any conflict-free batching gives the same
 * result).  fp64, round-to-nearest, built with -ffp-contract=off so every
 * expression is evaluated exactly as written (§8(c) c.6).
 *
 * Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".  Quality
 * metrics (WNS/TNS/power score, Eq. (1)) are out of scope: parity unpinned.
 */
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <omp.h>

extern "C" {

struct OGrid {
    int32_t X, Y, L;
    const uint8_t *dir;        // [L] 0 = H, 1 = V
    const uint8_t *routable;   // [L]
    const double *r, *c;       // [L]
    const double *vr;          // [L-1]
    const double *ofw;         // [L]
    double s_pos, s_zero;
    const int32_t *wire_cap;   // API layout
    const int32_t *via_cap;    // [(L-1)][Y][X]
    const int32_t *wire_dem0;  // NULL = 0
    const int32_t *via_dem0;   // NULL = 0
    double W_D, W_CAP, W_CONG, W_VIA;
    double r_avg;              // NaN = mean of routable r
    double logit_k, logit_b, w_floor;
    int32_t delta_lo, delta_hi;
};

struct ONets {
    int64_t n_nets;
    const int64_t *pin_ptr;
    const int32_t *pin_x, *pin_y;
    const uint8_t *pin_layer;
    const double *pin_cap, *pin_slack;
    const int64_t *seg_ptr;
    const int32_t *seg_xy;
    const double *r_drv;       // NULL = 0
    const int64_t *order_key;  // NULL = index
    double wns;
};

struct OOut {
    int64_t max_wires, max_vias;  // capacity of wires / vias
    int64_t max_nets_to_run;      // <= 0: all nets; else only the first K in priority order
    double *net_cost;             // [n_nets] f[root][p_drv]   (NaN if not run)
    int64_t *wire_ptr;            // [n_nets+1]
    int32_t *wires;               // [.][5] x1 y1 x2 y2 layer, x1<=x2, y1<=y2, sorted per net
    int64_t *via_ptr;             // [n_nets+1]
    int32_t *vias;                // [.][4] x y b t (t > b), sorted per net
    int32_t *wire_dem;            // API layout, final demand
    int32_t *via_dem;
    double *sink_delay;           // [n_pins], driver slots 0
    double *net_cap;              // [n_nets]
    double *net_rc;               // [n_nets]
    int32_t *batch_of;            // [n_nets] conflict-free batch (sequential recurrence)
    int32_t *n_nodes;             // [n_nets]
    double elapsed_s;             // DP + backtrack + commit + Elmore of the nets run
    int64_t nets_run;
    char err[256];
    // SURVEY §8(f) NEXT #1 (paper-style batches, PAPER §III-A l.224-226, reading R31): when
    // non-NULL, snap_batch[net] is the net's batch; batches run in ascending id, every net of a
    // batch reads the demand at the start of its batch, and the batch's commits are applied
    // after all its nets (integer adds: their order does not matter).  NULL: sequential.
    const int32_t *snap_batch;
    // mode 2: > 1 = the nets of each conflict-free batch on this many host
    // threads (exact by c.2); 0 / 1 = mode 1, sequential.  Ignored with snap_batch.
    int32_t threads;
};

}  // extern "C"

namespace {

const double INF = std::numeric_limits<double>::infinity();
enum { DIR_E = 0, DIR_W = 1, DIR_N = 2, DIR_S = 3 };

struct Ctx {
    const OGrid *g;
    const ONets *nets;
    int X, Y, L;
    std::vector<int64_t> wire_off;   // per layer offset in the API wire array
    std::vector<int32_t> wdem, vdem; // current demand
    std::vector<double> VR;          // [L][L]
    std::vector<double> Mpos, Mzero; // Eq. (3) marginal tables over [delta_lo, delta_hi]
    double r_avg;
    char *err;
};

// ---------------------------------------------------------------- O4 tables --
// VR[a][b] = sum_{k=min(a,b)}^{max(a,b)-1} vr[k], ascending k (Alg. 2 input
// "R of via on each layer vr").
// M_s[delta] = exp(s*(delta+1)) - exp(s*delta): marginal cost of one more unit
// of demand under Eq. (3) of = ofw(l) * e^{s(d-c)} (reading R18).
void build_tables(Ctx &C) {
    const OGrid *g = C.g;
    int L = C.L;
    C.VR.assign((size_t)L * L, 0.0);
    for (int a = 0; a < L; a++)
        for (int b = 0; b < L; b++) {
            int lo = std::min(a, b), hi = std::max(a, b);
            double s = 0.0;
            for (int k = lo; k < hi; k++) s = s + g->vr[k];
            C.VR[(size_t)a * L + b] = s;
        }
    int n = g->delta_hi - g->delta_lo + 1;
    C.Mpos.resize(n);
    C.Mzero.resize(n);
    for (int i = 0; i < n; i++) {
        double d = (double)(g->delta_lo + i);
        C.Mpos[i] = std::exp(g->s_pos * (d + 1.0)) - std::exp(g->s_pos * d);
        C.Mzero[i] = std::exp(g->s_zero * (d + 1.0)) - std::exp(g->s_zero * d);
    }
    if (std::isnan(g->r_avg)) {
        double s = 0.0;
        int cnt = 0;
        for (int l = 0; l < L; l++)
            if (g->routable[l]) { s = s + g->r[l]; cnt++; }
        C.r_avg = s / (double)cnt;
    } else {
        C.r_avg = g->r_avg;
    }
}

// marginal Eq. (3) cost of one more unit on an element with capacity c, demand d
double marginal(const Ctx &C, int32_t cap, int32_t dem) {
    int64_t delta = (int64_t)dem - (int64_t)cap;
    if (delta < C.g->delta_lo) delta = C.g->delta_lo;
    if (delta > C.g->delta_hi) delta = C.g->delta_hi;
    const std::vector<double> &M = (cap == 0) ? C.Mzero : C.Mpos;   // s = 1.5 if c = 0 else 0.5
    return M[(size_t)(delta - C.g->delta_lo)];
}

int64_t wire_index(const Ctx &C, int l, int x, int y) {   // unit edge with lower endpoint (x, y)
    if (C.g->dir[l] == 0) return C.wire_off[l] + (int64_t)y * (C.X - 1) + x;
    return C.wire_off[l] + (int64_t)y * C.X + x;
}
int64_t via_index(const Ctx &C, int k, int x, int y) { return ((int64_t)k * C.Y + y) * C.X + x; }

// ViaCong (Alg. 3 l.377; reading R11/R36): cost of one via cut between layer k
// and k+1 at GCell (x, y):  kappa = W_VIA + (W_CONG * ofw[k]) * M_{s(cv)}[dv - cv]
double kappa(const Ctx &C, int x, int y, int k) {
    int64_t i = via_index(C, k, x, y);
    return C.g->W_VIA + (C.g->W_CONG * C.g->ofw[k]) * marginal(C, C.g->via_cap[i], C.vdem[i]);
}

// ------------------------------------------------------------------ O1 tree --
struct Tree {
    std::vector<int> x, y, par, len, edir, height;   // edir: direction parent -> node
    std::vector<std::vector<int>> kids;                 // child order E, W, N, S
    std::vector<std::vector<int64_t>> pins;             // global pin ids, input order
    std::vector<int> pre;                               // preorder (root first)
    std::vector<int64_t> edges;                         // sorted unit-edge keys of the route
};

struct NetView {
    int64_t p0, p1;   // pin range
    int64_t s0, s1;   // segment range
};

bool fail(Ctx &C, const char *msg, int64_t net) {
    std::snprintf(C.err, 256, "net %lld: %s", (long long)net, msg);
    return false;
}

// Edge key of the unit edge with lower endpoint (x, y); t = 0 horizontal, 1 vertical.
inline int64_t ekey(const Ctx &C, int x, int y, int t) { return ((int64_t)y * C.X + x) * 2 + t; }

bool has(const std::vector<int64_t> &E, int64_t k) { return std::binary_search(E.begin(), E.end(), k); }

bool has_dir(const Ctx &C, const std::vector<int64_t> &E, int x, int y, int d) {
    switch (d) {
        case DIR_E: return x + 1 < C.X && has(E, ekey(C, x, y, 0));
        case DIR_W: return x > 0 && has(E, ekey(C, x - 1, y, 0));
        case DIR_N: return y + 1 < C.Y && has(E, ekey(C, x, y, 1));
        default:    return y > 0 && has(E, ekey(C, x, y - 1, 1));
    }
}
const int DX[4] = {1, -1, 0, 0}, DY[4] = {0, 0, 1, -1};
const int OPP[4] = {DIR_W, DIR_E, DIR_S, DIR_N};

// O1: union of unit edges -> tree check -> LA nodes (pins, degree != 2, bends)
// -> root = driver GCell -> children in E, W, N, S order (PAPER §III-B l.278-281:
// "we introduce additional nodes to ensure all inter-node connections are
// strictly straight").
bool build_tree(Ctx &C, int64_t net, const NetView &nv, Tree &T) {
    const ONets *N = C.nets;
    T = Tree();
    std::vector<int64_t> &E = T.edges;
    for (int64_t s = nv.s0; s < nv.s1; s++) {
        int x1 = N->seg_xy[4 * s], y1 = N->seg_xy[4 * s + 1], x2 = N->seg_xy[4 * s + 2], y2 = N->seg_xy[4 * s + 3];
        if (x1 < 0 || x2 < 0 || y1 < 0 || y2 < 0 || x1 >= C.X || x2 >= C.X || y1 >= C.Y || y2 >= C.Y)
            return fail(C, "segment outside the grid", net);
        if (x1 != x2 && y1 != y2) return fail(C, "segment not axis-aligned", net);
        if (y1 == y2) for (int x = std::min(x1, x2); x < std::max(x1, x2); x++) E.push_back(ekey(C, x, y1, 0));
        else          for (int y = std::min(y1, y2); y < std::max(y1, y2); y++) E.push_back(ekey(C, x1, y, 1));
    }
    std::sort(E.begin(), E.end());
    E.erase(std::unique(E.begin(), E.end()), E.end());
    int dx0 = N->pin_x[nv.p0], dy0 = N->pin_y[nv.p0];
    // vertex set of the route
    std::vector<int64_t> V;
    for (int64_t k : E) {
        int64_t g = k / 2;
        int x = (int)(g % C.X), y = (int)(g / C.X);
        V.push_back(g);
        V.push_back((k & 1) ? (int64_t)(y + 1) * C.X + x : (int64_t)y * C.X + x + 1);
    }
    if (E.empty()) V.push_back((int64_t)dy0 * C.X + dx0);
    std::sort(V.begin(), V.end());
    V.erase(std::unique(V.begin(), V.end()), V.end());
    for (int64_t p = nv.p0; p < nv.p1; p++) {
        int64_t g = (int64_t)N->pin_y[p] * C.X + N->pin_x[p];
        if (N->pin_x[p] < 0 || N->pin_y[p] < 0 || N->pin_x[p] >= C.X || N->pin_y[p] >= C.Y)
            return fail(C, "pin outside the grid", net);
        if (!std::binary_search(V.begin(), V.end(), g)) return fail(C, "pin GCell not on the route", net);
    }
    if (V.size() != E.size() + 1) return fail(C, "route is not a tree (cycle or disconnected)", net);
    // connectivity: BFS from the driver GCell over the unit edges
    {
        std::vector<char> seen(V.size(), 0);
        std::vector<int64_t> q{(int64_t)dy0 * C.X + dx0};
        seen[std::lower_bound(V.begin(), V.end(), q[0]) - V.begin()] = 1;
        size_t nseen = 1;
        for (size_t h = 0; h < q.size(); h++) {
            int x = (int)(q[h] % C.X), y = (int)(q[h] / C.X);
            for (int d = 0; d < 4; d++)
                if (has_dir(C, E, x, y, d)) {
                    int64_t g2 = (int64_t)(y + DY[d]) * C.X + (x + DX[d]);
                    size_t i = std::lower_bound(V.begin(), V.end(), g2) - V.begin();
                    if (!seen[i]) { seen[i] = 1; nseen++; q.push_back(g2); }
                }
        }
        if (nseen != V.size()) return fail(C, "route is not a tree (cycle or disconnected)", net);
    }
    // pin GCells (sorted) for the node test
    std::vector<int64_t> PG;
    for (int64_t p = nv.p0; p < nv.p1; p++) PG.push_back((int64_t)N->pin_y[p] * C.X + N->pin_x[p]);
    std::sort(PG.begin(), PG.end());
    auto is_node = [&](int x, int y) {
        if (std::binary_search(PG.begin(), PG.end(), (int64_t)y * C.X + x)) return true;
        bool e = has_dir(C, E, x, y, DIR_E), w = has_dir(C, E, x, y, DIR_W);
        bool n = has_dir(C, E, x, y, DIR_N), s = has_dir(C, E, x, y, DIR_S);
        int deg = e + w + n + s;
        if (deg != 2) return true;
        return !((e && w) || (n && s));   // degree 2 with perpendicular edges = bend
    };
    auto add_node = [&](int x, int y, int par, int len, int edir) {
        T.x.push_back(x); T.y.push_back(y); T.par.push_back(par); T.len.push_back(len);
        T.edir.push_back(edir); T.height.push_back(0);
        T.kids.emplace_back(); T.pins.emplace_back();
        return (int)T.x.size() - 1;
    };
    add_node(dx0, dy0, -1, 0, -1);
    std::vector<int> stack{0};
    while (!stack.empty()) {
        int n = stack.back();
        stack.pop_back();
        T.pre.push_back(n);
        int kids[4], nk = 0;
        for (int d = 0; d < 4; d++) {
            if (T.par[n] >= 0 && d == OPP[T.edir[n]]) continue;
            if (!has_dir(C, E, T.x[n], T.y[n], d)) continue;
            int cx = T.x[n] + DX[d], cy = T.y[n] + DY[d], len = 1;
            while (!is_node(cx, cy)) { cx += DX[d]; cy += DY[d]; len++; }
            int k = add_node(cx, cy, n, len, d);
            T.kids[n].push_back(k);
            kids[nk++] = k;
        }
        for (int i = nk - 1; i >= 0; i--) stack.push_back(kids[i]);   // E first in preorder
    }
    // attach pins (input order) to the node at their GCell
    for (int64_t p = nv.p0; p < nv.p1; p++) {
        int node = -1;
        for (size_t n = 0; n < T.x.size(); n++)
            if (T.x[n] == N->pin_x[p] && T.y[n] == N->pin_y[p]) { node = (int)n; break; }
        T.pins[node].push_back(p);
    }
    // height(leaf) = 0, height(n) = 1 + max over children (reading R7)
    for (auto it = T.pre.rbegin(); it != T.pre.rend(); ++it) {
        int n = *it, h = 0;
        for (int k : T.kids[n]) h = std::max(h, T.height[k] + 1);
        T.height[n] = h;
    }
    return true;
}

// ---------------------------------------------------------------- O2 Eq.(4) --
// Pin weight: logistic of slack/WNS with k = 10, b = 0.3 (
// printed form garbled, reading R1: 1 / (1 + e^{-k(x - b)})).  WNS >= 0: w_floor (R2).
double pin_weight(const OGrid *g, double slack, double wns) {
    if (!(wns < 0.0)) return g->w_floor;
    double x = slack / wns;
    return 1.0 / (1.0 + std::exp(-g->logit_k * (x - g->logit_b)));
}

// ------------------------------------------------------------ per-net state --
struct NetState {
    std::vector<double> wd;        // W_D * w_n (Eq. 5) per node
    std::vector<double> ur;        // O3
    std::vector<double> f, dlc;    // [node][L]
    std::vector<double> gp;        // [node][L] G' of the chosen span (Alg. 3 l.404 key; exposed for the pins)
    std::vector<int> cb, ct;       // choice (b, t) per [node][L]
    std::vector<int> entry;        // [node][L][4]
    std::vector<int> lay, sb, st;  // backtracked entry layer, span
};

inline int edge_dir_type(int edir) { return (edir == DIR_E || edir == DIR_W) ? 0 : 1; }

bool legal(const Ctx &C, int j, int dtype) { return C.g->routable[j] && C.g->dir[j] == dtype; }

// S: congestion sum over node s's parent-edge run on layer j, in ascending
// coordinate: ((m1 + m2) + ...) + m_len  (Alg. 3 "wccost", reading R16/R23).
double run_cong(const Ctx &C, const Tree &T, int s, int j) {
    int x = T.x[s], y = T.y[s], len = T.len[s];
    int a;   // lowest coordinate of the run's unit edges
    switch (T.edir[s]) {
        case DIR_E: a = x - len; break;
        case DIR_W: a = x; break;
        case DIR_N: a = y - len; break;
        default:    a = y; break;
    }
    double S = 0.0;
    for (int i = 0; i < len; i++) {
        int64_t idx = (edge_dir_type(T.edir[s]) == 0) ? wire_index(C, j, a + i, y) : wire_index(C, j, x, a + i);
        S = S + marginal(C, C.g->wire_cap[idx], C.wdem[idx]);
    }
    return S;
}

// O5 per-son terms (Alg. 3 l.386-393 "cost <- f + dcost + ccost + wccost",
// "cost' <- cost + w^d ur (dlc + wcap)"; readings R16, R17):
//   A = ((f[s][j] + wd_s*(Rw*(0.5*Cw + D))) + W_CAP*Cw) + (W_CONG*ofw[j])*S
//   B = wd_s*(Cw + D),  cost = A + B*VR[l][j],  cost' = cost + B*ur_n,  capb = Cw + D
struct SonTerms { double A, B, capb; bool ok; };
SonTerms son_terms(const Ctx &C, const Tree &T, const NetState &st, int s, int j) {
    SonTerms o{INF, 0.0, 0.0, false};
    if (!legal(C, j, edge_dir_type(T.edir[s]))) return o;
    double fs = st.f[(size_t)s * C.L + j];
    if (!(fs < INF)) return o;
    const OGrid *g = C.g;
    double Rw = g->r[j] * T.len[s];
    double Cw = g->c[j] * T.len[s];
    double D = st.dlc[(size_t)s * C.L + j];
    double S = run_cong(C, T, s, j);
    o.A = ((fs + st.wd[s] * (Rw * (0.5 * Cw + D))) + g->W_CAP * Cw) + (g->W_CONG * g->ofw[j]) * S;
    o.B = st.wd[s] * (Cw + D);
    o.capb = Cw + D;
    o.ok = true;
    return o;
}

// O6: Alg. 3 getSubtreeCandidate for one node n, all entry layers l.
void node_dp(const Ctx &C, const ONets *N, int64_t drv, const Tree &T, NetState &st, int n) {
    const OGrid *g = C.g;
    const int L = C.L;
    const bool root = (T.par[n] < 0);
    const int p_drv = N->pin_layer[drv];
    int nl = L, nh = -1;
    for (int64_t q : T.pins[n]) { nl = std::min(nl, (int)N->pin_layer[q]); nh = std::max(nh, (int)N->pin_layer[q]); }
    const bool has_pins = !T.pins[n].empty();
    const std::vector<int> &sons = T.kids[n];
    // kappa(k) at this node's GCell (vias never change inside this node's DP)
    std::vector<double> kap(L > 1 ? L - 1 : 1);
    for (int k = 0; k + 1 < L; k++) kap[k] = kappa(C, T.x[n], T.y[n], k);
    // per-son terms per layer j (do not depend on the entry layer l)
    std::vector<SonTerms> terms(sons.size() * L);
    for (size_t i = 0; i < sons.size(); i++)
        for (int j = 0; j < L; j++) terms[i * L + j] = son_terms(C, T, st, sons[i], j);

    for (int l = 0; l < L; l++) {
        size_t nlidx = (size_t)n * L + l;
        st.f[nlidx] = INF;
        st.dlc[nlidx] = 0.0;
        st.cb[nlidx] = st.ct[nlidx] = -1;
        // entry layers: root -> only the driver pin layer (R13); else the legal
        // layers of n's parent edge (R15)
        if (root ? (l != p_drv) : !legal(C, l, edge_dir_type(T.edir[n]))) continue;
        // pin terms, Alg. 3 l.4-7: d = pin_cap * vr(pin_l -> l); f += d * w; dlc += pin_cap
        double F0 = 0.0, C0 = 0.0;
        for (int64_t q : T.pins[n]) {
            if (q == drv) continue;
            double wq = root ? g->W_D * pin_weight(g, N->pin_slack[q], N->wns) : st.wd[n];
            F0 = F0 + wq * (N->pin_cap[q] * C.VR[(size_t)N->pin_layer[q] * L + l]);
            C0 = C0 + N->pin_cap[q];
        }
        // span bounds, Alg. 3 l.9-16 guards (R14: pin-free -> b0 = t0 = l)
        int b0 = has_pins ? std::min(l, nl) : l;
        int t0 = has_pins ? std::max(l, nh) : l;
        bool have = false;
        double bGp = 0, bG = 0, bK = 0;
        int bb = -1, bt = -1;
        int bj[4] = {-1, -1, -1, -1};
        for (int b = 0; b <= b0; b++) {
            for (int t = t0; t <= L - 1; t++) {
                double V = 0.0;   // vcong, one term per via cut (R9, R10)
                for (int k = b; k < t; k++) V = V + kap[k];
                double G = V, Gp = V, K = 0.0;
                int js[4] = {-1, -1, -1, -1};
                bool ok = true;
                for (size_t i = 0; i < sons.size(); i++) {
                    int jb = -1;
                    double cpb = 0, cb = 0, capb = 0;
                    for (int j = b; j <= t; j++) {
                        const SonTerms &o = terms[i * L + j];
                        if (!o.ok) continue;
                        double cost = o.A + o.B * C.VR[(size_t)l * L + j];
                        double cp = cost + o.B * st.ur[n];
                        if (!std::isfinite(cp)) continue;
                        if (jb < 0 || cp < cpb) { jb = j; cpb = cp; cb = cost; capb = o.capb; }   // ties: lowest j
                    }
                    if (jb < 0) { ok = false; break; }   // infeasible span (R12)
                    G = G + cb;
                    Gp = Gp + cpb;
                    K = K + capb;
                    js[i] = jb;
                }
                if (!ok) continue;
                // choice = argmin (G', t-b, b) lexicographic (Alg. 3 l.404; R21)
                bool better = !have || Gp < bGp || (Gp == bGp && (t - b < bt - bb || (t - b == bt - bb && b < bb)));
                if (better) {
                    have = true; bGp = Gp; bG = G; bK = K; bb = b; bt = t;
                    for (int i = 0; i < 4; i++) bj[i] = js[i];
                }
            }
        }
        if (!have) continue;
        st.gp[nlidx] = bGp;
        st.f[nlidx] = F0 + bG;          // Alg. 3 l.405
        st.dlc[nlidx] = C0 + bK;
        st.cb[nlidx] = bb;
        st.ct[nlidx] = bt;
        for (int i = 0; i < 4; i++) st.entry[nlidx * 4 + i] = bj[i];
    }
}


// O2 weights and O3 upstream resistance of one net (PAPER §III-C l.316-318, §III-D l.452).
//   wd_n = W_D * max of w_q over sinks q in subtree(n) (Eq. 5, reading R3), 0 if none (R39)
//   ur(root) = r_drv; ur(n) = ur(parent) + r_avg * len_n, len_n = n's own parent-edge length (R6)
void net_weights_ur(const Ctx &C, const ONets *nets, int64_t net, int64_t drv, const Tree &T, NetState &st) {
    const OGrid *g = C.g;
    const size_t nn = T.x.size();
    st.wd.assign(nn, 0.0);
    st.ur.assign(nn, 0.0);
    std::vector<double> w(nn, 0.0);
    for (auto it = T.pre.rbegin(); it != T.pre.rend(); ++it) {
        int n = *it;
        double m = 0.0;
        for (int64_t q : T.pins[n]) if (q != drv) m = std::max(m, pin_weight(g, nets->pin_slack[q], nets->wns));
        for (int k : T.kids[n]) m = std::max(m, w[k]);
        w[n] = m;
    }
    for (size_t n = 0; n < nn; n++) st.wd[n] = g->W_D * w[n];
    for (int n : T.pre)
        st.ur[n] = (T.par[n] < 0) ? (nets->r_drv ? nets->r_drv[net] : 0.0) : st.ur[T.par[n]] + C.r_avg * T.len[n];
}

// O6 over one net (children before parents): allocates and fills st.f/dlc/gp/cb/ct/entry.
void net_dp(const Ctx &C, const ONets *nets, int64_t drv, const Tree &T, NetState &st) {
    const size_t nn = T.x.size();
    const int L = C.L;
    st.f.assign(nn * L, INF);
    st.dlc.assign(nn * L, 0.0);
    st.gp.assign(nn * L, INF);
    st.cb.assign(nn * L, -1);
    st.ct.assign(nn * L, -1);
    st.entry.assign(nn * L * 4, -1);
    for (auto it = T.pre.rbegin(); it != T.pre.rend(); ++it) node_dp(C, nets, drv, T, st, *it);
}

// Elmore O9 canonical fast form, on the backtracked solution.
void elmore(const Ctx &C, const ONets *N, int64_t drv, const Tree &T, const NetState &st,
            double *sink_delay, double *net_cap, double *net_rc) {
    const OGrid *g = C.g;
    const int L = C.L;
    size_t nn = T.x.size();
    std::vector<double> Cd(nn), rc(nn), Tn(nn);
    // bottom-up: Cdown(n) = C0 + ((Cw1 + Cdown(s1)) + ...);  rc(n) = F0u + ((c1 + c2) + ...)
    for (auto it = T.pre.rbegin(); it != T.pre.rend(); ++it) {
        int n = *it;
        int ln = st.lay[n];
        double C0 = 0.0, F0u = 0.0;
        for (int64_t q : T.pins[n]) {
            if (q == drv) continue;
            C0 = C0 + N->pin_cap[q];
            F0u = F0u + N->pin_cap[q] * C.VR[(size_t)N->pin_layer[q] * L + ln];
        }
        double K = 0.0, R = 0.0;
        for (int s : T.kids[n]) {
            int ls = st.lay[s];
            double Cw = g->c[ls] * T.len[s], Rw = g->r[ls] * T.len[s];
            K = K + (Cw + Cd[s]);
            R = R + ((rc[s] + Rw * (0.5 * Cw + Cd[s])) + (Cw + Cd[s]) * C.VR[(size_t)ln * L + ls]);
        }
        Cd[n] = C0 + K;
        rc[n] = F0u + R;
    }
    *net_cap = Cd[T.pre[0]];
    *net_rc = rc[T.pre[0]];
    // top-down delay through via stacks and pi-model wires
    std::vector<double> Tk(L);
    for (int n : T.pre) {
        int ln = st.lay[n], b = st.sb[n], t = st.st[n];
        Tk.assign(L, 0.0);
        Tk[ln] = (T.par[n] < 0) ? 0.0 : Tn[n];
        auto Cge = [&](int j) {   // branches attached at layers >= j: sinks, then sons
            double acc = 0.0;
            for (int64_t q : T.pins[n]) if (q != drv && N->pin_layer[q] >= j) acc = acc + N->pin_cap[q];
            for (int s : T.kids[n]) if (st.lay[s] >= j) acc = acc + (g->c[st.lay[s]] * T.len[s] + Cd[s]);
            return acc;
        };
        auto Cle = [&](int j) {
            double acc = 0.0;
            for (int64_t q : T.pins[n]) if (q != drv && N->pin_layer[q] <= j) acc = acc + N->pin_cap[q];
            for (int s : T.kids[n]) if (st.lay[s] <= j) acc = acc + (g->c[st.lay[s]] * T.len[s] + Cd[s]);
            return acc;
        };
        for (int k = ln; k < t; k++) Tk[k + 1] = Tk[k] + g->vr[k] * Cge(k + 1);
        for (int k = ln; k > b; k--) Tk[k - 1] = Tk[k] + g->vr[k - 1] * Cle(k - 1);
        for (int64_t q : T.pins[n]) sink_delay[q] = (q == drv) ? 0.0 : Tk[N->pin_layer[q]];
        for (int s : T.kids[n]) {
            int ls = st.lay[s];
            double Cw = g->c[ls] * T.len[s], Rw = g->r[ls] * T.len[s];
            Tn[s] = Tk[ls] + Rw * (0.5 * Cw + Cd[s]);
        }
    }
}

}  // namespace

extern "C" {

double oracle_pin_weight(const OGrid *g, double slack, double wns) { return pin_weight(g, slack, wns); }

int oracle_tables(const OGrid *g, double *VR, double *Mpos, double *Mzero, double *r_avg) {
    Ctx C;
    C.g = g; C.L = g->L; C.X = g->X; C.Y = g->Y;
    build_tables(C);
    if (VR) std::memcpy(VR, C.VR.data(), sizeof(double) * C.VR.size());
    if (Mpos) std::memcpy(Mpos, C.Mpos.data(), sizeof(double) * C.Mpos.size());
    if (Mzero) std::memcpy(Mzero, C.Mzero.data(), sizeof(double) * C.Mzero.size());
    if (r_avg) *r_avg = C.r_avg;
    return 0;
}

// Tree of one net: out[n] = {x, y, parent, len, edir, height, npins}, nodes in preorder ids.
int oracle_tree(const OGrid *g, const ONets *nets, int64_t net, int32_t *out, int32_t max_nodes,
                int32_t *n_out, char *err) {
    Ctx C;
    C.g = g; C.nets = nets; C.X = g->X; C.Y = g->Y; C.L = g->L;
    char buf[256] = {0};
    C.err = buf;
    Tree T;
    NetView nv{nets->pin_ptr[net], nets->pin_ptr[net + 1], nets->seg_ptr[net], nets->seg_ptr[net + 1]};
    if (nv.p1 <= nv.p0) { if (err) std::snprintf(err, 256, "net %lld: no pins", (long long)net); return -1; }
    if (!build_tree(C, net, nv, T)) { if (err) std::memcpy(err, buf, 256); return -1; }
    *n_out = (int32_t)T.x.size();
    for (size_t n = 0; n < T.x.size() && (int32_t)n < max_nodes; n++) {
        int32_t *o = out + 7 * n;
        o[0] = T.x[n]; o[1] = T.y[n]; o[2] = T.par[n]; o[3] = T.len[n]; o[4] = T.edir[n];
        o[5] = T.height[n]; o[6] = (int32_t)T.pins[n].size();
    }
    return 0;
}

// Internals of O2/O3/O6 for ONE net on the grid's initial demand (exposed for the look-ahead pins,
// SURVEY §8(c) c.5 O3 and (iii)/(iv); the arithmetic is oracle_run's own, shared functions).
// Nodes in preorder ids (as oracle_tree).  Per node: ur, wd; per (node, l): f, dlc, G' of the
// chosen span, choice (b, t) (-1 if infeasible) and the sons' entry layers [4].
int oracle_net_dp(const OGrid *g, const ONets *nets, int64_t net, int32_t max_nodes, int32_t *n_out, double *ur,
                  double *wd, double *f, double *dlc, double *gp, int32_t *cb, int32_t *ct, int32_t *entry, char *err) {
    Ctx C;
    C.g = g; C.nets = nets; C.X = g->X; C.Y = g->Y; C.L = g->L;
    char buf[256] = {0};
    C.err = buf;
    const int L = C.L;
    C.wire_off.resize(L + 1);
    C.wire_off[0] = 0;
    for (int l = 0; l < L; l++)
        C.wire_off[l + 1] = C.wire_off[l] + (g->dir[l] == 0 ? (int64_t)(C.X - 1) * C.Y : (int64_t)C.X * (C.Y - 1));
    int64_t nw = C.wire_off[L], nvia = (int64_t)(L - 1) * C.X * C.Y;
    C.wdem.assign(nw, 0);
    C.vdem.assign(nvia, 0);
    if (g->wire_dem0) std::memcpy(C.wdem.data(), g->wire_dem0, 4 * nw);
    if (g->via_dem0) std::memcpy(C.vdem.data(), g->via_dem0, 4 * nvia);
    build_tables(C);
    Tree T;
    NetState st;
    NetView nv{nets->pin_ptr[net], nets->pin_ptr[net + 1], nets->seg_ptr[net], nets->seg_ptr[net + 1]};
    if (nv.p1 <= nv.p0) { if (err) std::snprintf(err, 256, "net %lld: no pins", (long long)net); return -1; }
    if (!build_tree(C, net, nv, T)) { if (err) std::memcpy(err, buf, 256); return -1; }
    const int64_t drv = nv.p0;
    const int nn = (int)T.x.size();
    *n_out = nn;
    if (nn > max_nodes) { if (err) std::snprintf(err, 256, "net %lld: %d nodes > max_nodes", (long long)net, nn); return -2; }
    net_weights_ur(C, nets, net, drv, T, st);
    net_dp(C, nets, drv, T, st);
    for (int n = 0; n < nn; n++) {
        ur[n] = st.ur[n];
        wd[n] = st.wd[n];
        for (int l = 0; l < L; l++) {
            size_t i = (size_t)n * L + l;
            f[i] = st.f[i]; dlc[i] = st.dlc[i]; gp[i] = st.gp[i]; cb[i] = st.cb[i]; ct[i] = st.ct[i];
            for (int k = 0; k < 4; k++) entry[i * 4 + k] = st.entry[i * 4 + k];
        }
    }
    return 0;
}

}  // extern "C"

namespace {

// Per-net outputs of one net (filled by solve_net; copied into OOut by the caller).
struct NetResult {
    double cost, ncap, nrc, seconds;
    std::vector<std::array<int32_t, 5>> wires;
    std::vector<std::array<int32_t, 4>> vias;
};

// O2/O3 + O6 + O7 + O8 + O9 for one net whose tree T is built: DP on the current demand, backtrack,
// commit (into C's demand, or appended to pend_w / pend_v in snapshot mode), Elmore.
void solve_net(Ctx &C, const ONets *nets, int64_t net, const Tree &T, NetState &st, bool want_sol,
               std::vector<int64_t> *pend_w, std::vector<int64_t> *pend_v, double *sink_delay, NetResult &R) {
    const int L = C.L;
    const int64_t drv = nets->pin_ptr[net];
    const size_t nn = T.x.size();
    net_weights_ur(C, nets, net, drv, T, st);
    auto t0 = std::chrono::steady_clock::now();
    // O6 bottom-up (children before parents)
    net_dp(C, nets, drv, T, st);
    // O7 backtrack (Alg. 4): root layer = driver pin layer (R13)
    st.lay.assign(nn, -1); st.sb.assign(nn, -1); st.st.assign(nn, -1);
    int root = T.pre[0];
    st.lay[root] = nets->pin_layer[drv];
    R.cost = st.f[(size_t)root * L + st.lay[root]];
    for (int n : T.pre) {
        size_t idx = (size_t)n * L + st.lay[n];
        st.sb[n] = st.cb[idx];
        st.st[n] = st.ct[idx];
        for (size_t i = 0; i < T.kids[n].size(); i++) st.lay[T.kids[n][i]] = st.entry[idx * 4 + i];
    }
    // O8 commit: +1 per unit edge on the chosen layer, +1 per via cut
    for (int n : T.pre) {
        if (T.par[n] >= 0) {
            int j = st.lay[n], x = T.x[n], y = T.y[n], len = T.len[n];
            for (int i = 0; i < len; i++) {
                int64_t idx;
                switch (T.edir[n]) {
                    case DIR_E: idx = wire_index(C, j, x - len + i, y); break;
                    case DIR_W: idx = wire_index(C, j, x + i, y); break;
                    case DIR_N: idx = wire_index(C, j, x, y - len + i); break;
                    default:    idx = wire_index(C, j, x, y + i); break;
                }
                if (pend_w) pend_w->push_back(idx);
                else C.wdem[idx] += 1;
            }
        }
        for (int k = st.sb[n]; k < st.st[n]; k++) {
            if (pend_v) pend_v->push_back(via_index(C, k, T.x[n], T.y[n]));
            else C.vdem[via_index(C, k, T.x[n], T.y[n])] += 1;
        }
    }
    // O9 Elmore
    elmore(C, nets, drv, T, st, sink_delay, &R.ncap, &R.nrc);
    R.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    R.wires.clear();
    R.vias.clear();
    if (want_sol) {
        for (int n : T.pre) {
            if (T.par[n] < 0) continue;
            int p = T.par[n];
            R.wires.push_back({std::min(T.x[n], T.x[p]), std::min(T.y[n], T.y[p]), std::max(T.x[n], T.x[p]),
                               std::max(T.y[n], T.y[p]), st.lay[n]});
        }
        std::sort(R.wires.begin(), R.wires.end());
        for (int n : T.pre)
            if (st.st[n] > st.sb[n]) R.vias.push_back({T.x[n], T.y[n], st.sb[n], st.st[n]});
        std::sort(R.vias.begin(), R.vias.end());
    }
}

// Tree of net `net` after the pin checks (no pins, pin layer >= L, route errors).
bool checked_tree(Ctx &C, const ONets *nets, int64_t net, Tree &T, char *err) {
    NetView nv{nets->pin_ptr[net], nets->pin_ptr[net + 1], nets->seg_ptr[net], nets->seg_ptr[net + 1]};
    if (nv.p1 <= nv.p0) { std::snprintf(err, 256, "net %lld: no pins", (long long)net); return false; }
    for (int64_t p = nv.p0; p < nv.p1; p++)
        if (nets->pin_layer[p] >= C.L) { std::snprintf(err, 256, "net %lld: pin layer >= L", (long long)net); return false; }
    char buf[256] = {0};
    char *keep = C.err;
    C.err = buf;
    bool ok = build_tree(C, net, nv, T);
    C.err = keep;
    if (!ok) std::memcpy(err, buf, 256);
    return ok;
}

// Per-direction average unit R / C of the pre-assignment parasitics (PAPER §III-B l.283-285:
// "For horizontal (vertical) wire connections, we calculate resistance (capacitance) using the
// average per-unit-length resistance (capacitance) of all horizontal (vertical) wires";
// reading R44: the plain mean over the routable layers of that direction, summed in ascending l).
double dir_mean(const OGrid *g, const double *v, int d) {
    double s = 0.0;
    int cnt = 0;
    for (int l = 0; l < g->L; l++)
        if (g->routable[l] && g->dir[l] == d) { s = s + v[l]; cnt++; }
    return cnt ? s / (double)cnt : 0.0;
}

// Pre-assignment timing of ONE net on its 2D LA tree with the pi-model (PAPER §III-B l.283-286,
// Alg. 1 inputs r_avg / c_avg l.240-241; reading R44), written as the
// definition of the Elmore delay:
//   edge into node n (n != root): R_n = r_dir(n) * len_n, C_n = c_dir(n) * len_n (dir: E/W = H);
//   pi-model node capacitance Cnode(u) = sum of u's sink pin caps (input order; the driver pin
//     has none) + C_u / 2 (u != root) + sum over u's sons s of C_s / 2 (child order);
//   Elmore delay of node v = sum over the edges n on the path root -> v of
//     R_n * (sum of Cnode(u) over the nodes u of subtree(n)), subtree membership tested by
//     walking u's ancestors (no recursion);
//   sink delay = the delay of its node; net load cap = sum of Cnode(u) over all nodes.
void pre_timing_net(const ONets *N, int64_t drv, const Tree &T, const double rd[2], const double cd[2],
                    double *sink_delay, double *net_cap) {
    const int nn = (int)T.x.size();
    std::vector<double> Rn(nn, 0.0), Cn(nn, 0.0), Cnode(nn, 0.0), down(nn, 0.0), D(nn, 0.0);
    for (int n = 0; n < nn; n++)
        if (T.par[n] >= 0) {
            const int t = edge_dir_type(T.edir[n]);
            Rn[n] = rd[t] * (double)T.len[n];
            Cn[n] = cd[t] * (double)T.len[n];
        }
    for (int u = 0; u < nn; u++) {
        double c = 0.0;
        for (int64_t q : T.pins[u]) if (q != drv) c = c + N->pin_cap[q];
        if (T.par[u] >= 0) c = c + 0.5 * Cn[u];
        for (int s : T.kids[u]) c = c + 0.5 * Cn[s];
        Cnode[u] = c;
    }
    double tot = 0.0;
    for (int u = 0; u < nn; u++) tot = tot + Cnode[u];
    for (int a = 0; a < nn; a++) {             // down(a) = sum of Cnode over subtree(a), by membership
        double s = 0.0;
        for (int u = 0; u < nn; u++) {
            int w = u;
            while (w >= 0 && w != a) w = T.par[w];
            if (w == a) s = s + Cnode[u];
        }
        down[a] = s;
    }
    for (int v = 0; v < nn; v++) {             // D(v) = sum over the path root -> v of R_n * down(n)
        double d = 0.0;
        for (int w = v; T.par[w] >= 0; w = T.par[w]) d = d + Rn[w] * down[w];
        D[v] = d;
    }
    for (int n = 0; n < nn; n++)
        for (int64_t q : T.pins[n]) sink_delay[q] = (q == drv) ? 0.0 : D[n];
    *net_cap = tot;
}

// footprint(j) = unit 2D edges of its route U GCells of its LA nodes; element spaces disjoint
// (SURVEY §8(c) c.2).
void footprint(const Ctx &C, const Tree &T, std::vector<int64_t> &fp) {
    fp.clear();
    for (int64_t k : T.edges) fp.push_back(k);   // unit edges: 2*(y*X+x)+t
    for (size_t n = 0; n < T.x.size(); n++) fp.push_back((int64_t)2 * C.X * C.Y + (int64_t)T.y[n] * C.X + T.x[n]);
}

}  // namespace

extern "C" {

// Pre-assignment pi-model timing of every net (pre_timing_net above).  r_h / r_v / c_h / c_v:
// per-direction unit R (kOhm) / C (fF); NaN = the mean over that direction's routable layers
// (dir_mean).  Outputs sink_delay[n_pins] (driver slots 0, ps) and net_cap[n_nets] (fF).
int oracle_pre_timing(const OGrid *g, const ONets *nets, double r_h, double r_v, double c_h, double c_v,
                      double *sink_delay, double *net_cap, char *err) {
    Ctx C;
    C.g = g; C.nets = nets; C.X = g->X; C.Y = g->Y; C.L = g->L;
    char buf[256] = {0};
    C.err = buf;
    const double rd[2] = {std::isnan(r_h) ? dir_mean(g, g->r, 0) : r_h, std::isnan(r_v) ? dir_mean(g, g->r, 1) : r_v};
    const double cd[2] = {std::isnan(c_h) ? dir_mean(g, g->c, 0) : c_h, std::isnan(c_v) ? dir_mean(g, g->c, 1) : c_v};
    for (int64_t net = 0; net < nets->n_nets; net++) {
        Tree T;
        if (!checked_tree(C, nets, net, T, err)) return -1;
        pre_timing_net(nets, nets->pin_ptr[net], T, rd, cd, sink_delay, net_cap + net);
    }
    return 0;
}

int oracle_run(const OGrid *g, const ONets *nets, OOut *out) {
    Ctx C;
    C.g = g; C.nets = nets; C.X = g->X; C.Y = g->Y; C.L = g->L;
    C.err = out->err;
    out->err[0] = 0;
    const int L = C.L;
    if (L < 2 || C.X <= 0 || C.Y <= 0) { std::snprintf(out->err, 256, "bad grid"); return -1; }
    C.wire_off.resize(L + 1);
    C.wire_off[0] = 0;
    for (int l = 0; l < L; l++)
        C.wire_off[l + 1] = C.wire_off[l] + (g->dir[l] == 0 ? (int64_t)(C.X - 1) * C.Y : (int64_t)C.X * (C.Y - 1));
    int64_t nw = C.wire_off[L], nvia = (int64_t)(L - 1) * C.X * C.Y;
    C.wdem.assign(nw, 0);
    C.vdem.assign(nvia, 0);
    if (g->wire_dem0) std::memcpy(C.wdem.data(), g->wire_dem0, 4 * nw);
    if (g->via_dem0) std::memcpy(C.vdem.data(), g->via_dem0, 4 * nvia);
    build_tables(C);

    const int64_t NN = nets->n_nets;
    // priority order: (order_key, index)
    std::vector<int64_t> order(NN);
    for (int64_t i = 0; i < NN; i++) order[i] = i;
    if (nets->order_key)
        std::stable_sort(order.begin(), order.end(),
                         [&](int64_t a, int64_t b) { return nets->order_key[a] < nets->order_key[b]; });
    const int32_t *snap = out->snap_batch;
    if (snap)   // batches in ascending id; inside a batch the order is immaterial (snapshot reads)
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return snap[a] < snap[b]; });
    std::vector<int64_t> pend_w, pend_v;   // snapshot mode: commits deferred to the end of the batch
    auto flush = [&]() {
        for (int64_t i : pend_w) C.wdem[i] += 1;
        for (int64_t i : pend_v) C.vdem[i] += 1;
        pend_w.clear();
        pend_v.clear();
    };
    int64_t nrun = (out->max_nets_to_run > 0 && out->max_nets_to_run < NN) ? out->max_nets_to_run : NN;
    const bool want_sol = out->wire_ptr || out->via_ptr;

    std::vector<std::vector<std::array<int32_t, 5>>> wires_of(out->wire_ptr ? NN : 0);
    std::vector<std::vector<std::array<int32_t, 4>>> vias_of(out->via_ptr ? NN : 0);
    if (out->net_cost) for (int64_t i = 0; i < NN; i++) out->net_cost[i] = std::numeric_limits<double>::quiet_NaN();
    if (out->sink_delay) for (int64_t p = 0; p < nets->pin_ptr[NN]; p++) out->sink_delay[p] = 0.0;
    std::vector<double> dummy;   // sink-delay sink when the caller passes none
    double *sd = out->sink_delay;
    if (!sd) { dummy.assign(nets->pin_ptr[NN], 0.0); sd = dummy.data(); }
    auto store = [&](int64_t net, NetResult &R) {
        if (out->net_cost) out->net_cost[net] = R.cost;
        if (out->net_cap) out->net_cap[net] = R.ncap;
        if (out->net_rc) out->net_rc[net] = R.nrc;
        if (out->wire_ptr) wires_of[net].swap(R.wires);
        if (out->via_ptr) vias_of[net].swap(R.vias);
    };

    double elapsed = 0.0;
    const int threads = out->threads > 1 ? out->threads : 1;
    if (threads == 1 || snap) {
        // ---- mode 1: sequential, one net at a time in priority order, commit after each (c.2) ----
        // batch recurrence: footprint = unit edges U node GCells; element spaces disjoint
        std::vector<int32_t> last;
        if (out->batch_of) last.assign((size_t)3 * C.X * C.Y, -1);
        Tree T;
        NetState st;
        NetResult R;
        std::vector<int64_t> fp;
        for (int64_t oi = 0; oi < nrun; oi++) {
            int64_t net = order[oi];
            if (snap && oi > 0 && snap[net] != snap[order[oi - 1]]) flush();
            if (!checked_tree(C, nets, net, T, out->err)) return -1;
            if (out->n_nodes) out->n_nodes[net] = (int32_t)T.x.size();
            solve_net(C, nets, net, T, st, want_sol, snap ? &pend_w : nullptr, snap ? &pend_v : nullptr, sd, R);
            elapsed += R.seconds;
            store(net, R);
            if (out->batch_of) {
                footprint(C, T, fp);
                int32_t b = 0;
                for (int64_t e : fp) b = std::max(b, last[e] + 1);
                for (int64_t e : fp) last[e] = b;
                out->batch_of[net] = b;
            }
        }
        flush();
    } else {
        // ---- mode 2: the same nets, batch by batch; the nets of one
        // conflict-free batch run concurrently on `threads` host threads.  Exact by c.2: nets of a
        // batch have disjoint footprints, so each reads and commits only state no other net of
        // the batch touches, and every net sees the commits of all earlier conflicting nets. ----
        std::vector<int32_t> bat(nrun);
        std::vector<int32_t> nodes_of(nrun);
        std::vector<int64_t> fp_ptr(nrun + 1, 0);
        std::vector<std::vector<int64_t>> fp_chunk(threads);
        std::vector<int64_t> chunk_beg(threads + 1);
        for (int t = 0; t <= threads; t++) chunk_beg[t] = nrun * t / threads;
        volatile bool failed = false;
        char errbuf[256] = {0};
        // (a) trees -> footprints, in parallel (contiguous chunks of the priority order)
#pragma omp parallel num_threads(threads)
        {
            int t = omp_get_thread_num();
            Tree T;
            std::vector<int64_t> fp;
            char err[256];
            for (int64_t oi = chunk_beg[t]; oi < chunk_beg[t + 1] && !failed; oi++) {
                if (!checked_tree(C, nets, order[oi], T, err)) {
#pragma omp critical
                    { if (!failed) { failed = true; std::memcpy(errbuf, err, 256); } }
                    break;
                }
                footprint(C, T, fp);
                nodes_of[oi] = (int32_t)T.x.size();
                fp_ptr[oi + 1] = (int64_t)fp.size();
                fp_chunk[t].insert(fp_chunk[t].end(), fp.begin(), fp.end());
            }
        }
        if (failed) { std::memcpy(out->err, errbuf, 256); return -1; }
        // (b) the sequential batch recurrence over the footprints, in priority order
        {
            std::vector<int32_t> last((size_t)3 * C.X * C.Y, -1);
            int64_t k = 0;
            for (int t = 0; t < threads; t++) {
                const std::vector<int64_t> &F = fp_chunk[t];
                int64_t pos = 0;
                for (int64_t oi = chunk_beg[t]; oi < chunk_beg[t + 1]; oi++, k++) {
                    int64_t cnt = fp_ptr[oi + 1];
                    int32_t b = 0;
                    for (int64_t i = 0; i < cnt; i++) b = std::max(b, last[F[pos + i]] + 1);
                    for (int64_t i = 0; i < cnt; i++) last[F[pos + i]] = b;
                    pos += cnt;
                    bat[oi] = b;
                }
                std::vector<int64_t>().swap(fp_chunk[t]);
            }
        }
        for (int64_t oi = 0; oi < nrun; oi++) {
            if (out->batch_of) out->batch_of[order[oi]] = bat[oi];
            if (out->n_nodes) out->n_nodes[order[oi]] = nodes_of[oi];
        }
        // (c) batches in order; inside a batch, nets in parallel
        int32_t nb = 0;
        for (int64_t oi = 0; oi < nrun; oi++) nb = std::max(nb, bat[oi] + 1);
        std::vector<int64_t> bptr(nb + 1, 0), bnets(nrun);
        for (int64_t oi = 0; oi < nrun; oi++) bptr[bat[oi] + 1]++;
        for (int32_t b = 0; b < nb; b++) bptr[b + 1] += bptr[b];
        {
            std::vector<int64_t> fill(bptr.begin(), bptr.end() - 1);
            for (int64_t oi = 0; oi < nrun; oi++) bnets[fill[bat[oi]]++] = order[oi];
        }
        auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(threads)
        {
            Tree T;
            NetState st;
            NetResult R;
            char err[256];
            for (int32_t b = 0; b < nb; b++) {
#pragma omp for schedule(dynamic, 64)
                for (int64_t i = bptr[b]; i < bptr[b + 1]; i++) {
                    int64_t net = bnets[i];
                    if (!checked_tree(C, nets, net, T, err)) continue;   // cannot fail: checked in (a)
                    solve_net(C, nets, net, T, st, want_sol, nullptr, nullptr, sd, R);
                    store(net, R);
                }   // implicit barrier: batch b is committed before b + 1 starts
            }
        }
        elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    out->elapsed_s = elapsed;
    out->nets_run = nrun;
    if (out->wire_ptr) {
        int64_t k = 0;
        out->wire_ptr[0] = 0;
        for (int64_t i = 0; i < NN; i++) {
            for (auto &w : wires_of[i]) {
                if (k >= out->max_wires) { std::snprintf(out->err, 256, "wire buffer too small"); return -2; }
                std::memcpy(out->wires + 5 * k, w.data(), 20);
                k++;
            }
            out->wire_ptr[i + 1] = k;
        }
    }
    if (out->via_ptr) {
        int64_t k = 0;
        out->via_ptr[0] = 0;
        for (int64_t i = 0; i < NN; i++) {
            for (auto &v : vias_of[i]) {
                if (k >= out->max_vias) { std::snprintf(out->err, 256, "via buffer too small"); return -2; }
                std::memcpy(out->vias + 4 * k, v.data(), 16);
                k++;
            }
            out->via_ptr[i + 1] = k;
        }
    }
    if (out->wire_dem) std::memcpy(out->wire_dem, C.wdem.data(), 4 * nw);
    if (out->via_dem) std::memcpy(out->via_dem, C.vdem.data(), 4 * nvia);
    return 0;
}

}  // extern "C"
