"""Independent checkers used to PIN the oracle (test code; never imported by the product).

Everything here is written from the paper's definitions a second time, in a
different shape from oracle/la_oracle.cpp, so that a plausible slip in the
oracle (a dropped term, a wrong sign/index, a transposed operand) shows up:

* ``build_tree``           -- O1 (PAPER §III-B l.264-281, Fig. 6) written as a
                              plain graph walk over a Python set of unit edges.
* ``assignment_cost``      -- the DP objective of ONE complete layer assignment,
                              evaluated from scratch: per-node via-cut costs over
                              the minimal covering span, per-pin via-delay terms
                              (Alg. 3 l.4-7), and per-edge delay / capacitance /
                              congestion terms (Alg. 3 l.386-391, reading R16)
                              with the true downstream capacitance.  No DP.
* ``brute_force``          -- exhaustive enumeration of every per-edge legal
                              layer.
* ``elmore_definitional``  -- O(n^2) Elmore: explicit RC graph, and for every
                              resistor the downstream capacitance by traversal
                              (PAPER §II-C l.146, §III-D l.443-444 "d34 =
                              R34 x (C4 + C5 + C6 + C7)").
"""
from __future__ import annotations

import itertools
import math

E, W, N, S = 0, 1, 2, 3
DXY = {E: (1, 0), W: (-1, 0), N: (0, 1), S: (0, -1)}
OPP = {E: W, W: E, N: S, S: N}


def unit_edges(segs):
    es = set()
    for (x1, y1, x2, y2) in segs:
        if y1 == y2:
            for x in range(min(x1, x2), max(x1, x2)):
                es.add(((x, y1), (x + 1, y1)))
        else:
            for y in range(min(y1, y2), max(y1, y2)):
                es.add(((x1, y), (x1, y + 1)))
    return es


def build_tree(pins, segs):
    """pins: list of (x, y, layer, cap, slack), pin 0 = driver.  Returns a list of
    nodes (dicts) with root at index 0 and children in E, W, N, S order."""
    es = unit_edges(segs)
    adj = {}
    for a, b in es:
        adj.setdefault(a, set()).add(b)
        adj.setdefault(b, set()).add(a)
    pin_cells = {(p[0], p[1]) for p in pins}

    def nb(g, d):
        h = (g[0] + DXY[d][0], g[1] + DXY[d][1])
        return h if h in adj.get(g, ()) else None

    def is_node(g):
        if g in pin_cells:
            return True
        ds = [d for d in (E, W, N, S) if nb(g, d) is not None]
        if len(ds) != 2:
            return True
        return set(ds) not in ({E, W}, {N, S})

    root = (pins[0][0], pins[0][1])
    nodes = [dict(x=root[0], y=root[1], parent=-1, len=0, edir=-1, kids=[], pins=[])]
    todo = [0]
    while todo:
        n = todo.pop(0)
        g = (nodes[n]["x"], nodes[n]["y"])
        for d in (E, W, N, S):
            if nodes[n]["parent"] >= 0 and d == OPP[nodes[n]["edir"]]:
                continue
            h = nb(g, d)
            if h is None:
                continue
            ln = 1
            while not is_node(h):
                h = nb(h, d)
                ln += 1
            nodes.append(dict(x=h[0], y=h[1], parent=n, len=ln, edir=d, kids=[], pins=[]))
            nodes[n]["kids"].append(len(nodes) - 1)
            todo.append(len(nodes) - 1)
    at = {(nd["x"], nd["y"]): i for i, nd in enumerate(nodes)}
    for q, p in enumerate(pins):
        nodes[at[(p[0], p[1])]]["pins"].append(q)
    return nodes


def net_pins(d, net):
    a, b = int(d.pin_ptr[net]), int(d.pin_ptr[net + 1])
    return [(int(d.pin_x[i]), int(d.pin_y[i]), int(d.pin_layer[i]), float(d.pin_cap[i]), float(d.pin_slack[i]))
            for i in range(a, b)]


def net_segs(d, net):
    a, b = int(d.seg_ptr[net]), int(d.seg_ptr[net + 1])
    return [tuple(int(v) for v in d.seg_xy[i]) for i in range(a, b)]


def wire_idx(d, l, x, y):
    off = 0
    for k in range(l):
        off += (d.X - 1) * d.Y if d.dir[k] == 0 else d.X * (d.Y - 1)
    return off + (y * (d.X - 1) + x if d.dir[l] == 0 else y * d.X + x)


def via_idx(d, k, x, y):
    return (k * d.Y + y) * d.X + x


def marginal(d, cap, dem):
    """Eq. (3) of = ofw e^{s(d-c)}: cost of one more unit = e^{s(d+1-c)} - e^{s(d-c)}
    (ofw applied by the caller), with d - c clamped to the table domain (R20)."""
    s = d.s_zero if cap == 0 else d.s_pos
    delta = min(max(dem - cap, d.delta_lo), d.delta_hi)
    return math.exp(s * (delta + 1)) - math.exp(s * delta)


def dem_arrays(d):
    wd = d.wire_dem0 if d.wire_dem0 is not None else [0] * len(d.wire_cap)
    vd = d.via_dem0 if d.via_dem0 is not None else [0] * len(d.via_cap)
    return wd, vd


def pin_w(d, slack):
    if d.wns < 0:
        return 1.0 / (1.0 + math.exp(-d.logit_k * (slack / d.wns - d.logit_b)))
    return d.w_floor


def r_avg(d):
    if not math.isnan(d.r_avg):
        return d.r_avg
    rs = [d.r[l] for l in range(d.L) if d.routable[l]]
    return sum(rs) / len(rs)


def legal_layers(d, edir):
    t = 0 if edir in (E, W) else 1
    return [j for j in range(d.L) if d.routable[j] and d.dir[j] == t]


def run_cells(nd):
    """Lower endpoints of the unit edges of a node's parent run + orientation (0 = H)."""
    x, y, ln, e = nd["x"], nd["y"], nd["len"], nd["edir"]
    if e == E:
        return [(x - ln + i, y) for i in range(ln)], 0
    if e == W:
        return [(x + i, y) for i in range(ln)], 0
    if e == N:
        return [(x, y - ln + i) for i in range(ln)], 1
    return [(x, y + i) for i in range(ln)], 1


def assignment_cost(d, net, nodes, lay, r_drv=None):
    """Cost of one complete assignment ``lay`` (layer per non-root node = its parent-edge
    layer) with minimal covering via spans, evaluated from scratch."""
    pins = net_pins(d, net)
    wd_arr, vd_arr = dem_arrays(d)
    L = d.L
    lay = list(lay)
    lay[0] = pins[0][2]                       # root entry = driver pin layer (R13)
    n = len(nodes)
    # subtree sink weights and true downstream caps
    order = []
    st = [0]
    while st:
        v = st.pop()
        order.append(v)
        st.extend(nodes[v]["kids"])
    wsub = [0.0] * n
    cdown = [0.0] * n
    for v in reversed(order):
        m = 0.0
        cd = 0.0
        for q in nodes[v]["pins"]:
            if q == 0:
                continue
            m = max(m, pin_w(d, pins[q][4]))
            cd += pins[q][3]
        for k in nodes[v]["kids"]:
            m = max(m, wsub[k])
            cd += d.c[lay[k]] * nodes[k]["len"] + cdown[k]
        wsub[v] = m
        cdown[v] = cd

    def vr_between(a, b):
        return sum(d.vr[k] for k in range(min(a, b), max(a, b)))

    total = 0.0
    for v in range(n):
        nd = nodes[v]
        ls = [lay[v]] + [lay[k] for k in nd["kids"]] + [pins[q][2] for q in nd["pins"]]
        b, t = min(ls), max(ls)
        for k in range(b, t):
            i = via_idx(d, k, nd["x"], nd["y"])
            total += d.W_VIA + d.W_CONG * d.ofw[k] * marginal(d, int(d.via_cap[i]), int(vd_arr[i]))
        for q in nd["pins"]:
            if q == 0:
                continue
            wq = d.W_D * pin_w(d, pins[q][4]) if v == 0 else d.W_D * wsub[v]
            total += wq * pins[q][3] * vr_between(pins[q][2], lay[v])
        if v == 0:
            continue
        j = lay[v]
        Rw, Cw = d.r[j] * nd["len"], d.c[j] * nd["len"]
        cells, o = run_cells(nd)
        Scong = sum(marginal(d, int(d.wire_cap[wire_idx(d, j, x, y)]), int(wd_arr[wire_idx(d, j, x, y)]))
                    for (x, y) in cells)
        wdv = d.W_D * wsub[v]
        D = cdown[v]
        total += wdv * (Rw * (0.5 * Cw + D) + (Cw + D) * vr_between(lay[nd["parent"]], j))
        total += d.W_CAP * Cw + d.W_CONG * d.ofw[j] * Scong
    return total


def brute_force(d, net, nodes):
    """Exhaustive minimum of assignment_cost over every per-edge legal layer.
    Returns (best_cost, best_layers, second_best_cost)."""
    choices = [legal_layers(d, nodes[v]["edir"]) if v > 0 else [None] for v in range(len(nodes))]
    best, second, arg = math.inf, math.inf, None
    for combo in itertools.product(*choices):
        c = assignment_cost(d, net, nodes, combo)
        if c < best:
            second, best, arg = best, c, combo
        elif c < second:
            second = c
    return best, arg, second


def solution_layers(nodes, wires):
    """Map the oracle/library canonical wire list of one net back onto tree nodes."""
    lay = [None] * len(nodes)
    for v in range(1, len(nodes)):
        nd, p = nodes[v], nodes[nodes[v]["parent"]]
        key = (min(nd["x"], p["x"]), min(nd["y"], p["y"]), max(nd["x"], p["x"]), max(nd["y"], p["y"]))
        hits = [int(w[4]) for w in wires if tuple(int(t) for t in w[:4]) == key]
        assert len(hits) == 1, (key, wires)
        lay[v] = hits[0]
    return lay


def elmore_definitional(d, pins, nodes, lay, spans):
    """O(n^2) Elmore on the explicit 3D RC tree of one net.  Returns
    (delay per pin [driver = 0], net_cap, net_rc)."""
    lay = list(lay)
    lay[0] = pins[0][2]
    cap = {}        # vertex -> lumped capacitance
    adj = {}        # vertex -> list of (neighbour, R)

    def add_v(v):
        cap.setdefault(v, 0.0)
        adj.setdefault(v, [])

    for v, nd in enumerate(nodes):
        b, t = spans[v]
        for k in range(b, t + 1):
            add_v((v, k))
        for k in range(b, t):
            adj[(v, k)].append(((v, k + 1), d.vr[k]))
            adj[(v, k + 1)].append(((v, k), d.vr[k]))
        for q in nd["pins"]:
            if q != 0:
                cap[(v, pins[q][2])] += pins[q][3]
    for v, nd in enumerate(nodes):
        if v == 0:
            continue
        j = lay[v]
        Rw, Cw = d.r[j] * nd["len"], d.c[j] * nd["len"]
        a, b = (nd["parent"], j), (v, j)
        cap[a] += Cw / 2
        cap[b] += Cw / 2
        adj[a].append((b, Rw))
        adj[b].append((a, Rw))
    src = (0, pins[0][2])
    # orient the tree from the source
    parent = {src: None}
    pr = {}
    order = [src]
    for u in order:
        for (w, R) in adj[u]:
            if w not in parent:
                parent[w] = u
                pr[w] = R
                order.append(w)
    assert len(order) == len(cap)
    children = {u: [] for u in order}
    for w in order[1:]:
        children[parent[w]].append(w)

    def downstream(w):       # total capacitance of the subtree hanging below resistor (parent[w], w)
        tot, st = 0.0, [w]
        while st:
            u = st.pop()
            tot += cap[u]
            st.extend(children[u])
        return tot

    rc_term = {w: pr[w] * downstream(w) for w in order[1:]}
    delays = [0.0] * len(pins)
    for v, nd in enumerate(nodes):
        for q in nd["pins"]:
            if q == 0:
                continue
            u, s = (v, pins[q][2]), 0.0
            while parent[u] is not None:
                s += rc_term[u]
                u = parent[u]
            delays[q] = s
    return delays, sum(cap.values()), sum(rc_term.values())


# ---------------------------------------------------------------- look-ahead (O3) and node-local DP
def upstream_r(d, net, nodes):
    """O3 written from PAPER l.452 (reading R6) as a walk down from the root: ur(root) = r_drv,
    ur(child) = ur(parent) + r_avg * (the child's own edge length).  Returns a list per node."""
    ra = r_avg(d)
    ur = [0.0] * len(nodes)
    ur[0] = float(d.r_drv[net])
    todo = [0]
    while todo:
        v = todo.pop()
        for k in nodes[v]["kids"]:
            ur[k] = ur[v] + ra * nodes[k]["len"]
            todo.append(k)
    return ur


def subtree_wd(d, net, nodes):
    """W_D x max sink weight over each node's subtree (Eq. (5), R3), 0 if none (R39)."""
    pins = net_pins(d, net)
    w = [0.0] * len(nodes)

    def rec(v):
        m = 0.0
        for q in nodes[v]["pins"]:
            if q != 0:
                m = max(m, pin_w(d, pins[q][4]))
        for k in nodes[v]["kids"]:
            m = max(m, rec(k))
        w[v] = m
        return m

    rec(0)
    return [d.W_D * x for x in w]


def _vr_asc(d, a, b):
    s = 0.0
    for k in range(min(a, b), max(a, b)):
        s = s + d.vr[k]
    return s


def node_local_enumeration(d, net, nodes, dp, omap):
    """for every node n and entry layer l with a finite oracle f,
    enumerate EVERY tuple of son layers (each son on a legal layer where its oracle f is finite),
    take the tuple's minimal covering via span [min(b0, js), max(t0, js)], and evaluate
    G' = ((V + cost'_1) + cost'_2) + ... with the O5 expression order, V summed ascending from b.
    The minimum over tuples must equal the oracle's G' (dp['gp']) bitwise (kappa >= 0 and rounded
    addition is monotone).  Where that minimum is attained by one tuple only, the oracle's son
    layers and span must be that tuple and its cover.  (iv): at the minimising tuple,
    G' - G = ur_n x sum(B_i) within rounding, and the oracle's f = F0 + G bitwise.
    ``omap[v]`` is the oracle's node id of refcheck node v.  Returns (checked, unique) counts."""
    pins = net_pins(d, net)
    wd_arr, vd_arr = dem_arrays(d)
    L = d.L
    ur = upstream_r(d, net, nodes)
    wdv = subtree_wd(d, net, nodes)
    checked = unique = 0
    for v, nd in enumerate(nodes):
        o = omap[v]
        assert dp["ur"][o] == ur[v], ("ur", v, dp["ur"][o], ur[v])
        assert dp["wd"][o] == wdv[v], ("wd", v)
        root = v == 0
        kap = []
        for k in range(L - 1):
            i = via_idx(d, k, nd["x"], nd["y"])
            kap.append(d.W_VIA + (d.W_CONG * d.ofw[k]) * marginal(d, int(d.via_cap[i]), int(vd_arr[i])))
        pl = [pins[q][2] for q in nd["pins"]]
        sons = nd["kids"]
        # per son: legal finite layers and the O5 terms (A, B, capb) from the son's oracle f / dlc
        opts = []
        for s in sons:
            sn = nodes[s]
            cells, _ = run_cells(sn)
            lst = []
            for j in legal_layers(d, sn["edir"]):
                fs = dp["f"][omap[s]][j]
                if not math.isfinite(fs):
                    continue
                Rw, Cw = d.r[j] * sn["len"], d.c[j] * sn["len"]
                D = dp["dlc"][omap[s]][j]
                S = 0.0
                for (x, y) in cells:
                    wi = wire_idx(d, j, x, y)
                    S = S + marginal(d, int(d.wire_cap[wi]), int(wd_arr[wi]))
                A = ((fs + wdv[s] * (Rw * (0.5 * Cw + D))) + d.W_CAP * Cw) + (d.W_CONG * d.ofw[j]) * S
                lst.append((j, A, wdv[s] * (Cw + D), Cw + D))
            opts.append(lst)
        entries = [pins[0][2]] if root else legal_layers(d, nd["edir"])
        for l in entries:
            if not math.isfinite(dp["f"][o][l]):
                continue
            b0 = min([l] + pl) if pl else l
            t0 = max([l] + pl) if pl else l
            best, arg, cnt = math.inf, None, 0
            for combo in itertools.product(*opts):
                js = [c[0] for c in combo]
                b, t = min([b0] + js), max([t0] + js)
                V = 0.0
                for k in range(b, t):
                    V = V + kap[k]
                Gp, G, Bs = V, V, 0.0
                for (j, A, B, _) in combo:
                    cost = A + B * _vr_asc(d, l, j)
                    G = G + cost
                    Gp = Gp + (cost + B * ur[v])
                    Bs = Bs + B
                if Gp < best:
                    best, arg, cnt = Gp, (js, b, t, G, Bs), 1
                elif Gp == best:
                    cnt += 1
            assert best == dp["gp"][o][l], ("min G'", v, l, best, dp["gp"][o][l])
            js, b, t, G, Bs = arg
            gap = best - G
            assert abs(gap - ur[v] * Bs) <= 1e-12 * max(1.0, abs(best)), ("cost' - cost", v, l, gap, ur[v] * Bs)
            checked += 1
            if cnt == 1:
                unique += 1
                assert (dp["cb"][o][l], dp["ct"][o][l]) == (b, t), ("span", v, l)
                assert [int(dp["entry"][o][l][i]) for i in range(len(sons))] == js, ("son layers", v, l)
                F0 = 0.0
                for q in nd["pins"]:
                    if q == 0:
                        continue
                    wq = d.W_D * pin_w(d, pins[q][4]) if root else wdv[v]
                    F0 = F0 + wq * (pins[q][3] * _vr_asc(d, pins[q][2], l))
                assert dp["f"][o][l] == F0 + G, ("f = F0 + G", v, l)
    return checked, unique


def oracle_node_map(nodes, otree):
    """refcheck node index -> oracle node id, matched by GCell (one LA node per GCell)."""
    at = {(int(r[0]), int(r[1])): i for i, r in enumerate(otree)}
    return [at[(nd["x"], nd["y"])] for nd in nodes]
