/*
 * gen/synth.c -- seeded synthetic ISPD-2025-shaped layer-assignment inputs.
 *
 * This module is INPUT GENERATION ONLY.  It holds none of the layer-assignment
 * method's arithmetic (no cost, no DP, no Elmore, no tree building of the LA
 * directed tree).  It plays the role of the 2D global router that the paper
 * takes as given (GAP-LA consumes "a GCell grid graph with GCell edge capacity,
 * a netlist and an optimized 2D global routing solution", §II-B
 * l.132) and emits plain arrays that both the oracle (oracle/) and the CUDA
 * library (paper_2507_13375_b200/) read.  Recipe: SURVEY.md §8(d) d.2, restated
 * in DESIGN.md "Input recipe".
 *
 * Determinism: every random draw comes from a counter-based SplitMix64 stream
 * keyed by (seed, purpose, index), so the output is independent of the thread
 * count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n_nets;
    int32_t X, Y, L;
    uint64_t seed;
    int32_t pin_max;        /* largest pin count of the base mix (8 for config 1, else 63) */
    double hf_frac;         /* fraction of nets with 64..256 pins (config 4: 0.001)          */
    int32_t rdrv_mode;      /* 0: r_drv = 0 ; 1: r_drv ~ U(0.5, 2) kOhm                      */
    double wns;             /* design WNS in ps (negative)                                    */
    double p_neg;           /* probability that a sink slack is negative                      */
} synth_params;

typedef struct {
    int64_t n_nets, n_pins, n_segs;
    int64_t *pin_ptr;
    int32_t *pin_x, *pin_y;
    uint8_t *pin_layer;
    double *pin_cap, *pin_slack;
    int64_t *seg_ptr;
    int32_t *seg_xy;
    double *r_drv;
    int64_t *order_key;
    int64_t n_wire, n_via;
    int32_t *wire_cap;   /* API layout: per layer, row-major [y][x] over edges by lower endpoint */
    int32_t *via_cap;    /* [(L-1)][Y][X] */
} synth_out;

/* ---------------------------------------------------------------- RNG ---- */
static inline uint64_t splitmix64(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t mix(uint64_t a, uint64_t b) {
    uint64_t s = a ^ (b * 0xD1B54A32D192ED03ULL);
    splitmix64(&s);
    return splitmix64(&s);
}
typedef struct { uint64_t s; } rng_t;
static inline rng_t rng_make(uint64_t seed, uint64_t purpose, uint64_t idx) {
    rng_t r; r.s = mix(mix(seed, purpose), idx); return r;
}
static inline double rng_u01(rng_t *r) { return (double)(splitmix64(&r->s) >> 11) * (1.0 / 9007199254740992.0); }
static inline int64_t rng_int(rng_t *r, int64_t lo, int64_t hi) { /* inclusive */
    uint64_t span = (uint64_t)(hi - lo + 1);
    return lo + (int64_t)(splitmix64(&r->s) % span);
}

/* ------------------------------------------------------- pin count mix ---- */
/* SURVEY §8(d) d.2 base mix: P(2)=.60 P(3)=.15 P(4)=.08 P(5-8)=.10 P(9-16)=.05
 * P(17-32)=.015 P(33-63)=.005, uniform within a band; bands above pin_max are
 * dropped and the rest renormalised. */
static int draw_pins(rng_t *r, int pin_max, double hf_frac) {
    if (hf_frac > 0 && rng_u01(r) < hf_frac) return (int)rng_int(r, 64, 256);
    static const int lo[7] = {2, 3, 4, 5, 9, 17, 33};
    static const int hi[7] = {2, 3, 4, 8, 16, 32, 63};
    static const double p[7] = {0.60, 0.15, 0.08, 0.10, 0.05, 0.015, 0.005};
    double tot = 0;
    for (int i = 0; i < 7; i++) if (lo[i] <= pin_max) tot += p[i];
    double u = rng_u01(r) * tot, acc = 0;
    for (int i = 0; i < 7; i++) {
        if (lo[i] > pin_max) break;
        acc += p[i];
        if (u < acc || i == 6 || lo[i + 1] > pin_max) {
            int h = hi[i] < pin_max ? hi[i] : pin_max;
            return (int)rng_int(r, lo[i], h);
        }
    }
    return 2;
}

/* ------------------------------------------------ one net: pins + route ---- */
typedef struct {
    int np;
    int32_t *px, *py;
    uint8_t *pl;
    double *pc, *ps;
    int ns;
    int32_t *sxy;
    double rdrv;
    int cap_p, cap_s;
} net_buf;

static void nb_reserve(net_buf *b, int np, int ns) {
    if (np > b->cap_p) {
        b->cap_p = np * 2;
        b->px = realloc(b->px, sizeof(int32_t) * b->cap_p);
        b->py = realloc(b->py, sizeof(int32_t) * b->cap_p);
        b->pl = realloc(b->pl, b->cap_p);
        b->pc = realloc(b->pc, sizeof(double) * b->cap_p);
        b->ps = realloc(b->ps, sizeof(double) * b->cap_p);
    }
    if (ns > b->cap_s) {
        b->cap_s = ns * 2 + 16;
        b->sxy = realloc(b->sxy, sizeof(int32_t) * 4 * b->cap_s);
    }
}

/* Greedy Prim-style rectilinear Steiner tree (SURVEY §8(d) d.2 "2D route"):
 * repeatedly take the unconnected pin nearest (Manhattan) to the tree, walk an
 * L-path (H-first or V-first by coin flip) toward its nearest tree GCell, and
 * stop at the first GCell already on the tree. */
static void gen_net(const synth_params *P, int64_t net, net_buf *b) {
    rng_t r = rng_make(P->seed, 1, (uint64_t)net);
    int k = draw_pins(&r, P->pin_max, P->hf_frac);
    double mean = 3.0 * sqrt((double)k);
    int w = 1 + (int)llround(-mean * log(1.0 - rng_u01(&r)));
    int h = 1 + (int)llround(-mean * log(1.0 - rng_u01(&r)));
    if (w > P->X) w = P->X;
    if (h > P->Y) h = P->Y;
    int x0 = (int)rng_int(&r, 0, P->X - w), y0 = (int)rng_int(&r, 0, P->Y - h);
    nb_reserve(b, k, 2 * k + 2);
    b->np = k;
    for (int i = 0; i < k; i++) {
        b->px[i] = x0 + (int)rng_int(&r, 0, w - 1);
        b->py[i] = y0 + (int)rng_int(&r, 0, h - 1);
        b->pl[i] = rng_u01(&r) < 0.9 ? 0 : 1;
        b->pc[i] = 0.5 + 1.5 * rng_u01(&r);
        if (i == 0) b->ps[i] = 0.0;
        else if (rng_u01(&r) < P->p_neg) { double u = rng_u01(&r); b->ps[i] = P->wns * u * u; }
        else b->ps[i] = 400.0 * rng_u01(&r);
    }
    b->rdrv = P->rdrv_mode ? 0.5 + 1.5 * rng_u01(&r) : 0.0;

    /* local bitmap over the bounding box */
    size_t area = (size_t)w * (size_t)h;
    uint8_t *on = calloc(area, 1);
    int *tx = malloc(sizeof(int) * (area < 64 ? 64 : area));
    int *ty = malloc(sizeof(int) * (area < 64 ? 64 : area));
    int nt = 0;
    int *dist = malloc(sizeof(int) * k), *near = malloc(sizeof(int) * k);
#define ON(x, y) on[(size_t)((y) - y0) * w + ((x) - x0)]
    ON(b->px[0], b->py[0]) = 1; tx[nt] = b->px[0]; ty[nt] = b->py[0]; nt++;
    for (int i = 0; i < k; i++) {
        dist[i] = abs(b->px[i] - tx[0]) + abs(b->py[i] - ty[0]);
        near[i] = 0;
    }
    b->ns = 0;
    for (;;) {
        int best = -1;
        for (int i = 1; i < k; i++) {
            if (ON(b->px[i], b->py[i])) continue;
            if (best < 0 || dist[i] < dist[best]) best = i;
        }
        if (best < 0) break;
        int gx = tx[near[best]], gy = ty[near[best]];
        int hfirst = rng_u01(&r) < 0.5;
        int cx = b->px[best], cy = b->py[best];
        int added0 = nt;
        ON(cx, cy) = 1; tx[nt] = cx; ty[nt] = cy; nt++;
        int sx = cx, sy = cy, done = 0;
        for (int leg = 0; leg < 2 && !done; leg++) {
            int horiz = (leg == 0) == hfirst;
            sx = cx; sy = cy;
            while (!done) {
                if (horiz && cx == gx) break;
                if (!horiz && cy == gy) break;
                if (horiz) cx += (gx > cx) ? 1 : -1; else cy += (gy > cy) ? 1 : -1;
                if (ON(cx, cy)) done = 1;
                else { ON(cx, cy) = 1; tx[nt] = cx; ty[nt] = cy; nt++; }
            }
            if (cx != sx || cy != sy) {
                nb_reserve(b, k, b->ns + 1);
                int32_t *s = b->sxy + 4 * b->ns;
                s[0] = sx; s[1] = sy; s[2] = cx; s[3] = cy;
                b->ns++;
            }
        }
        /* update nearest-tree distances with the newly added GCells */
        for (int i = 1; i < k; i++) {
            for (int t = added0; t < nt; t++) {
                int d = abs(b->px[i] - tx[t]) + abs(b->py[i] - ty[t]);
                if (d < dist[i]) { dist[i] = d; near[i] = t; }
            }
        }
    }
#undef ON
    free(on); free(tx); free(ty); free(dist); free(near);
}

/* ----------------------------------------------------------- capacities ---- */
static int64_t wire_layer_size(const synth_params *P, int l) {
    return (l % 2 == 0) ? (int64_t)(P->X - 1) * P->Y : (int64_t)P->X * (P->Y - 1);
}

static void gen_caps(const synth_params *P, synth_out *o) {
    int L = P->L;
    int64_t off = 0;
    for (int l = 0; l < L; l++) {
        int64_t n = wire_layer_size(P, l);
        int base = (l == 0) ? 2 : (l <= 4 ? 10 : 8);
        int32_t *cap = o->wire_cap + off;
        int W = (l % 2 == 0) ? P->X - 1 : P->X;     /* row length of this layer's edge array */
        int H = (l % 2 == 0) ? P->Y : P->Y - 1;
        #pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n; e++) {
            rng_t r = rng_make(P->seed, 100 + l, (uint64_t)e);
            int v = base + (int)rng_int(&r, -2, 2);
            cap[e] = v < 0 ? 0 : v;
        }
        /* blockages: random rectangles until ~2% of this layer's edges are covered */
        rng_t r = rng_make(P->seed, 200 + l, 0);
        int64_t target = n / 50, covered = 0;
        while (covered < target && W > 0 && H > 0) {
            int bw = (int)rng_int(&r, 2, 16), bh = (int)rng_int(&r, 2, 16);
            if (bw > W) bw = W;
            if (bh > H) bh = H;
            int bx = (int)rng_int(&r, 0, W - bw), by = (int)rng_int(&r, 0, H - bh);
            for (int yy = by; yy < by + bh; yy++)
                for (int xx = bx; xx < bx + bw; xx++) cap[(int64_t)yy * W + xx] = 0;
            covered += (int64_t)bw * bh;
        }
        off += n;
    }
    int64_t nv = (int64_t)(L - 1) * P->X * P->Y;
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < nv; e++) {
        rng_t r = rng_make(P->seed, 300, (uint64_t)e);
        o->via_cap[e] = 16 + (int)rng_int(&r, -4, 4);
    }
}

/* ------------------------------------------------------------ ordering ---- */
typedef struct { double key; int64_t idx; } kv_t;
static int kv_cmp(const void *a, const void *b) {
    const kv_t *x = a, *y = b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/* ----------------------------------------------------------------- main ---- */
int synth_generate(const synth_params *P, synth_out *o) {
    memset(o, 0, sizeof(*o));
    if (P->n_nets < 0 || P->X < 2 || P->Y < 2 || P->L < 2) return -1;
    int64_t N = P->n_nets;
    o->n_nets = N;
    int nthr = 1;
#ifdef _OPENMP
    nthr = omp_get_max_threads();
#endif
    /* nets are generated in chunks per thread, then concatenated in net order */
    int64_t chunk = (N + nthr - 1) / (nthr ? nthr : 1);
    if (chunk < 1) chunk = 1;
    int nch = (int)((N + chunk - 1) / chunk);
    typedef struct { int64_t np, ns; int32_t *px, *py, *sxy; uint8_t *pl; double *pc, *ps, *rd; int64_t *pn, *sn; } part_t;
    part_t *parts = calloc(nch > 0 ? nch : 1, sizeof(part_t));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < nch; c++) {
        int64_t a = c * chunk, z = a + chunk < N ? a + chunk : N;
        part_t *pt = &parts[c];
        int64_t cap_p = (z - a) * 8 + 64, cap_s = (z - a) * 8 + 64;
        pt->px = malloc(4 * cap_p); pt->py = malloc(4 * cap_p); pt->pl = malloc(cap_p);
        pt->pc = malloc(8 * cap_p); pt->ps = malloc(8 * cap_p);
        pt->sxy = malloc(16 * cap_s);
        pt->rd = malloc(8 * (z - a)); pt->pn = malloc(8 * (z - a)); pt->sn = malloc(8 * (z - a));
        net_buf nb; memset(&nb, 0, sizeof(nb));
        for (int64_t i = a; i < z; i++) {
            gen_net(P, i, &nb);
            if (pt->np + nb.np > cap_p) {
                cap_p = (pt->np + nb.np) * 2;
                pt->px = realloc(pt->px, 4 * cap_p); pt->py = realloc(pt->py, 4 * cap_p);
                pt->pl = realloc(pt->pl, cap_p); pt->pc = realloc(pt->pc, 8 * cap_p);
                pt->ps = realloc(pt->ps, 8 * cap_p);
            }
            if (pt->ns + nb.ns > cap_s) {
                cap_s = (pt->ns + nb.ns) * 2;
                pt->sxy = realloc(pt->sxy, 16 * cap_s);
            }
            memcpy(pt->px + pt->np, nb.px, 4 * nb.np);
            memcpy(pt->py + pt->np, nb.py, 4 * nb.np);
            memcpy(pt->pl + pt->np, nb.pl, nb.np);
            memcpy(pt->pc + pt->np, nb.pc, 8 * nb.np);
            memcpy(pt->ps + pt->np, nb.ps, 8 * nb.np);
            memcpy(pt->sxy + 4 * pt->ns, nb.sxy, 16 * nb.ns);
            pt->np += nb.np; pt->ns += nb.ns;
            pt->rd[i - a] = nb.rdrv; pt->pn[i - a] = nb.np; pt->sn[i - a] = nb.ns;
        }
        free(nb.px); free(nb.py); free(nb.pl); free(nb.pc); free(nb.ps); free(nb.sxy);
    }
    int64_t NP = 0, NS = 0;
    for (int c = 0; c < nch; c++) { NP += parts[c].np; NS += parts[c].ns; }
    o->n_pins = NP; o->n_segs = NS;
    o->pin_ptr = malloc(8 * (N + 1)); o->seg_ptr = malloc(8 * (N + 1));
    o->pin_x = malloc(4 * (NP ? NP : 1)); o->pin_y = malloc(4 * (NP ? NP : 1));
    o->pin_layer = malloc(NP ? NP : 1);
    o->pin_cap = malloc(8 * (NP ? NP : 1)); o->pin_slack = malloc(8 * (NP ? NP : 1));
    o->seg_xy = malloc(16 * (NS ? NS : 1));
    o->r_drv = malloc(8 * (N ? N : 1)); o->order_key = malloc(8 * (N ? N : 1));
    int64_t pp = 0, sp = 0;
    o->pin_ptr[0] = 0; o->seg_ptr[0] = 0;
    for (int c = 0; c < nch; c++) {
        part_t *pt = &parts[c];
        int64_t a = c * chunk, z = a + chunk < N ? a + chunk : N;
        memcpy(o->pin_x + pp, pt->px, 4 * pt->np); memcpy(o->pin_y + pp, pt->py, 4 * pt->np);
        memcpy(o->pin_layer + pp, pt->pl, pt->np);
        memcpy(o->pin_cap + pp, pt->pc, 8 * pt->np); memcpy(o->pin_slack + pp, pt->ps, 8 * pt->np);
        memcpy(o->seg_xy + 4 * sp, pt->sxy, 16 * pt->ns);
        int64_t qp = pp, qs = sp;
        for (int64_t i = a; i < z; i++) {
            o->r_drv[i] = pt->rd[i - a];
            qp += pt->pn[i - a]; qs += pt->sn[i - a];
            o->pin_ptr[i + 1] = qp; o->seg_ptr[i + 1] = qs;
        }
        pp += pt->np; sp += pt->ns;
        free(pt->px); free(pt->py); free(pt->pl); free(pt->pc); free(pt->ps); free(pt->sxy);
        free(pt->rd); free(pt->pn); free(pt->sn);
    }
    free(parts);

    /* order_key = rank of net slack (min sink slack), ascending, ties by net index
     * (SURVEY §8(c) R32). */
    kv_t *kv = malloc(sizeof(kv_t) * (N ? N : 1));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        double m = 1e300;
        for (int64_t q = o->pin_ptr[i] + 1; q < o->pin_ptr[i + 1]; q++)
            if (o->pin_slack[q] < m) m = o->pin_slack[q];
        kv[i].key = m; kv[i].idx = i;
    }
    qsort(kv, (size_t)N, sizeof(kv_t), kv_cmp);
    for (int64_t r = 0; r < N; r++) o->order_key[kv[r].idx] = r;
    free(kv);

    o->n_wire = 0;
    for (int l = 0; l < P->L; l++) o->n_wire += wire_layer_size(P, l);
    o->n_via = (int64_t)(P->L - 1) * P->X * P->Y;
    o->wire_cap = malloc(4 * o->n_wire);
    o->via_cap = malloc(4 * o->n_via);
    gen_caps(P, o);
    return 0;
}

void synth_free(synth_out *o) {
    free(o->pin_ptr); free(o->pin_x); free(o->pin_y); free(o->pin_layer);
    free(o->pin_cap); free(o->pin_slack); free(o->seg_ptr); free(o->seg_xy);
    free(o->r_drv); free(o->order_key); free(o->wire_cap); free(o->via_cap);
    memset(o, 0, sizeof(*o));
}
