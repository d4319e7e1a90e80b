"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the passage it follows.  None of them re-calls the oracle's own
routine to produce an expected value: expected values are closed forms, hand
numbers (tests/golden/), brute-force enumeration (tests/refcheck.py), an
independent definitional Elmore, or invariants.
"""
import copy
import math

import numpy as np
import pytest

import refcheck as rc
from gen import synth
from helpers import fixture_design, golden, randomize_state, rebuild_demand, single_net, tiny_pool
from oracle import oracle

REL = 1e-12


def rel_close(a, b, tol):
    return abs(a - b) <= tol * max(1.0, abs(a), abs(b))


# ------------------------------------------------------------------ O4 tables
def test_eq3_marginal_tables_closed_form():
    """Eq. (3): marginal at d = c is e^s - 1; sums telescope to the state."""
    g = golden("closed_forms.json")["eq3"]
    d = synth.empty_design(4, 4, 4)
    VR, Mp, Mz, ravg = oracle.tables(d)
    z = -d.delta_lo                     # index of delta = 0
    assert Mp[z] == pytest.approx(g["marginal_at_d_eq_c_cpos"], rel=1e-15)
    assert Mz[z] == pytest.approx(g["marginal_at_d_eq_c_czero"], rel=1e-15)
    # state e^{1.5*2} - e^0 = sum of marginals for delta = 0, 1 (c = 0, d: 0 -> 2)
    assert Mz[z] + Mz[z + 1] + 1.0 == pytest.approx(g["state_c0_d2"], rel=1e-14)
    # c > 0, d = c - 4: e^{-2} = 1 - sum_{delta=-4}^{-1} M(delta)
    assert 1.0 - Mp[z - 4:z].sum() == pytest.approx(g["state_d_eq_c_minus_4_cpos"], rel=1e-12)
    assert np.all(Mp > 0) and np.all(np.diff(Mp) > 0) and np.all(Mz[z:] > Mp[z:])   # c = 0 implies d - c >= 0


def test_via_resistance_table():
    """VR[a][b] = sum of vr over the crossed cuts (Alg. 2 input vr)."""
    d = synth.empty_design(4, 4, 4)
    d.vr = np.array([0.010, 0.008, 0.006])
    VR, _, _, ravg = oracle.tables(d)
    assert VR[0][0] == 0.0 and VR[2][2] == 0.0
    assert VR[0][3] == pytest.approx(0.024, rel=1e-15) and VR[3][0] == VR[0][3]
    assert VR[1][2] == pytest.approx(0.008, rel=1e-15)
    assert ravg == pytest.approx(np.mean(d.r), rel=1e-15)


# ------------------------------------------------------------------ O2 Eq. (4)
def test_eq4_pin_weight_values():
    """Eq. (4) logistic, k = 10, b = 0.3 (reading R1) and Fig. 7 (l.305-308)."""
    g = golden("closed_forms.json")["eq4"]
    d = synth.empty_design(4, 4, 4)
    assert oracle.pin_weight(d, -500.0, -500.0) == pytest.approx(g["ratio_1"], rel=1e-15)
    assert oracle.pin_weight(d, -150.0, -500.0) == pytest.approx(g["ratio_b"], rel=1e-15)
    assert oracle.pin_weight(d, 0.0, -500.0) == pytest.approx(g["ratio_0"], rel=1e-15)
    assert oracle.pin_weight(d, -1.0, g["fig7_wns"]) == pytest.approx(g["fig7_sink_minus1"], rel=1e-14)
    assert oracle.pin_weight(d, -100.0, g["fig7_wns"]) == pytest.approx(g["fig7_sink_minus100"], rel=1e-15)
    # WNS >= 0: floor weight (reading R2)
    assert oracle.pin_weight(d, 5.0, 0.0) == d.w_floor


# ------------------------------------------------------------------ O1 tree
def test_fig6_node_counts():
    """Fig. 6: net 1 (straight 2-pin) -> 2 nodes; net 2 -> 4 route nodes + 1 bend = 5,
    with the Fig. 8 topology 3->4, 4->5, 4->6, 6->7 (l.452-453; reading R34)."""
    g = golden("closed_forms.json")["fig6"]
    d = synth.empty_design(8, 8, 4)
    n1 = dict(pins=[(0, 5, 0, 1.0, -1.0), (4, 5, 0, 1.0, -1.0)], segs=[(0, 5, 4, 5)])
    # node3 = (0,0) driver, node4 = (2,0) Steiner, node5 = (4,0) sink, node6 = (2,2) bend, node7 = (4,2) sink
    n2 = dict(pins=[(0, 0, 0, 1.0, -1.0), (4, 0, 0, 1.0, -1.0), (4, 2, 0, 1.0, -1.0)],
              segs=[(0, 0, 4, 0), (2, 0, 2, 2), (2, 2, 4, 2)])
    d = synth.with_nets(d, [n1, n2])
    t1, t2 = oracle.tree(d, 0), oracle.tree(d, 1)
    assert len(t1) == g["net1_nodes"] and len(t2) == g["net2_nodes"]
    pos = {(int(r[0]), int(r[1])): i for i, r in enumerate(t2)}
    par = {k: (int(t2[v][2])) for k, v in pos.items()}
    at = {i: k for k, i in pos.items()}
    assert par[(0, 0)] == -1
    assert at[par[(2, 0)]] == (0, 0)          # 3 -> 4
    assert at[par[(4, 0)]] == (2, 0)          # 4 -> 5
    assert at[par[(2, 2)]] == (2, 0)          # 4 -> 6 (the added bend)
    assert at[par[(4, 2)]] == (2, 2)          # 6 -> 7
    heights = {k: int(t2[v][5]) for k, v in pos.items()}
    assert heights == {(0, 0): 3, (2, 0): 2, (4, 0): 0, (2, 2): 1, (4, 2): 0}


@pytest.mark.parametrize("seed", [11, 12])
def test_tree_matches_independent_builder(seed):
    """O1 vs an independent graph-walk implementation (tests/refcheck.py) on generated nets:
    same node set, parent links, run lengths; every edge straight; sum len = unit edges."""
    d = synth.generate(n_nets=300, X=24, Y=24, L=6, seed=seed, pin_max=16)
    for net in range(d.n_nets):
        t = oracle.tree(d, net)
        ref = rc.build_tree(rc.net_pins(d, net), rc.net_segs(d, net))
        assert len(t) == len(ref)
        mine = {(int(r[0]), int(r[1])): (int(r[3]), int(r[4])) for r in t}
        theirs = {(n["x"], n["y"]): (n["len"], n["edir"]) for n in ref}
        assert mine == theirs
        assert sum(int(r[3]) for r in t) == len(rc.unit_edges(rc.net_segs(d, net)))


def test_route_errors():
    """Route validation (SURVEY §8(b) errors): cycle, pin off-route, diagonal segment."""
    d = synth.empty_design(8, 8, 4)
    bad = [dict(pins=[(0, 0, 0, 1, 0), (2, 2, 0, 1, 0)], segs=[(0, 0, 2, 0), (2, 0, 2, 2), (0, 0, 0, 2), (0, 2, 2, 2)]),
           dict(pins=[(0, 0, 0, 1, 0), (3, 3, 0, 1, 0)], segs=[(0, 0, 2, 0)]),
           dict(pins=[(0, 0, 0, 1, 0), (2, 2, 0, 1, 0)], segs=[(0, 0, 2, 2)]),
           # a cycle plus a separate run (vertices = edges + 1): driver on the cycle / on the run
           dict(pins=[(0, 0, 0, 1, 0), (2, 2, 0, 1, 0)],
                segs=[(0, 0, 2, 0), (2, 0, 2, 2), (0, 0, 0, 2), (0, 2, 2, 2), (4, 4, 5, 4)]),
           dict(pins=[(4, 4, 0, 1, 0), (5, 4, 0, 1, 0), (2, 2, 0, 1, 0)],
                segs=[(0, 0, 2, 0), (2, 0, 2, 2), (0, 0, 0, 2), (0, 2, 2, 2), (4, 4, 5, 4)])]
    msgs = ["not a tree", "not on the route", "axis-aligned", "not a tree", "not a tree"]
    for n, m in zip(bad, msgs):
        e = synth.with_nets(synth.empty_design(8, 8, 4), [n])
        with pytest.raises(oracle.OracleError, match=m):
            oracle.run(e)


# ------------------------------------------------------------------ O9 Elmore
@pytest.mark.parametrize("name", ["A", "B"])
def test_elmore_hand_fixtures(name):
    """Hand-computed Elmore on 2-3 segment nets (tests/golden/elmore_fixtures.json)."""
    G = golden("elmore_fixtures.json")
    fx = G[name]
    d = fixture_design(fx, G["tech"])
    r = oracle.run(d)
    assert r["net_cap"][0] == pytest.approx(fx["net_cap"], rel=1e-12)
    assert r["net_rc"][0] == pytest.approx(fx["net_rc"], rel=1e-12)
    if name == "A":
        assert r["sink_delay"][1] == pytest.approx(fx["delay_sink"], rel=1e-12)
        assert r["sink_delay"][1] == pytest.approx(sum(fx["terms"].values()), rel=1e-12)
    else:
        assert r["sink_delay"][1] == pytest.approx(fx["delay_A"], rel=1e-12)
        assert r["sink_delay"][2] == pytest.approx(fx["delay_B"], rel=1e-12)
    assert r["sink_delay"][0] == 0.0
    assert int((r["vias"][:, 3] - r["vias"][:, 2]).sum()) == fx["via_cuts"]
    assert int(r["wire_dem"].sum()) == fx["wirelength"]


@pytest.mark.parametrize("seed,L", [(21, 4), (22, 6)])
def test_elmore_vs_definitional(seed, L):
    """Canonical fast form vs the O(n^2) explicit-RC-graph Elmore within 1e-9 relative."""
    d = tiny_pool(seed, L, n=150, X=10, Y=10, pin_max=8)
    r = oracle.run(d)
    for net in range(d.n_nets):
        pins, nodes = rc.net_pins(d, net), rc.build_tree(rc.net_pins(d, net), rc.net_segs(d, net))
        w = r["wires"][r["wire_ptr"][net]:r["wire_ptr"][net + 1]]
        v = r["vias"][r["via_ptr"][net]:r["via_ptr"][net + 1]]
        lay = rc.solution_layers(nodes, w)
        spans = []
        vmap = {(int(a[0]), int(a[1])): (int(a[2]), int(a[3])) for a in v}
        for i, nd in enumerate(nodes):
            l = pins[0][2] if i == 0 else lay[i]
            spans.append(vmap.get((nd["x"], nd["y"]), (l, l)))
        delays, ncap, nrc = rc.elmore_definitional(d, pins, nodes, lay, spans)
        p0 = d.pin_ptr[net]
        for q in range(len(pins)):
            assert rel_close(r["sink_delay"][p0 + q], delays[q], 1e-9)
        assert rel_close(r["net_cap"][net], ncap, 1e-9)
        assert rel_close(r["net_rc"][net], nrc, 1e-9)


# ------------------------------------------------------------------ O6 DP
def _dp_cases(seed, L, rdrv_mode=0, max_nodes=6, want=60):
    pool = tiny_pool(seed, L, n=500, rdrv_mode=rdrv_mode)
    rng = np.random.default_rng(seed)
    out = []
    for net in range(pool.n_nets):
        nodes = rc.build_tree(rc.net_pins(pool, net), rc.net_segs(pool, net))
        if 2 <= len(nodes) <= max_nodes:
            out.append((randomize_state(single_net(pool, net), rng), nodes))
        if len(out) >= want:
            break
    return out


@pytest.mark.parametrize("seed,L", [(31, 4), (32, 4), (33, 6)])
def test_dp_exact_when_wd_zero(seed, L):
    """W_D = 0: the objective is separable, so Alg. 3/4 is an exact tree DP.
    Cost equals the brute-force minimum; layers equal wherever that minimum is unique."""
    for d, nodes in _dp_cases(seed, L):
        d.W_D = 0.0
        r = oracle.run(d)
        best, arg, second = rc.brute_force(d, 0, nodes)
        assert rel_close(r["net_cost"][0], best, REL), (r["net_cost"][0], best)
        if second > best * (1 + 1e-9) + 1e-12:
            assert rc.solution_layers(nodes, r["wires"])[1:] == list(arg[1:])


def test_dp_exact_on_depth1_trees():
    """Depth-1 trees (root + leaf sons), any weights, r_drv = 0: no after-effect, DP = optimum (SURVEY c.5)."""
    n_checked = 0
    for seed in (41, 42, 43):
        for d, nodes in _dp_cases(seed, 6, max_nodes=5, want=200):
            if any(nd["kids"] for nd in nodes[1:]):
                continue
            d.W_D = 100.0
            r = oracle.run(d)
            best, arg, second = rc.brute_force(d, 0, nodes)
            assert rel_close(r["net_cost"][0], best, REL)
            if second > best * (1 + 1e-9) + 1e-12:
                assert rc.solution_layers(nodes, r["wires"])[1:] == list(arg[1:])
            n_checked += 1
    assert n_checked > 50


@pytest.mark.parametrize("seed,L,rdrv", [(51, 4, 0), (52, 6, 1), (53, 4, 1)])
def test_dp_cost_reconstruction_and_lower_bound(seed, L, rdrv):
    """W_D > 0 (heuristic look-ahead): (i) re-evaluating the emitted solution from
    scratch reproduces f[root]; (ii) f[root] >= the brute-force optimum."""
    for d, nodes in _dp_cases(seed, L, rdrv_mode=rdrv):
        d.W_D = 100.0
        r = oracle.run(d)
        lay = rc.solution_layers(nodes, r["wires"])
        recon = rc.assignment_cost(d, 0, nodes, lay)
        assert rel_close(r["net_cost"][0], recon, REL), (r["net_cost"][0], recon)
        best, _, _ = rc.brute_force(d, 0, nodes)
        assert r["net_cost"][0] >= best * (1 - 1e-12)


def test_straight_two_pin_choice_by_hand():
    """Straight 2-pin net, W_D = W_CAP = 0 (SURVEY c.5 'O6 special case'): the chosen layer minimises
    V_root + W_CONG*ofw[j]*S_j + V_sink over legal j, lowest j on ties.  Hand-built case: L = 6,
    H layers 0, 2, 4; layer 0 congested, so the cheapest total is decided by via cuts vs ofw."""
    d = synth.empty_design(8, 8, 6, cap_wire=2, cap_via=16)
    d.W_D, d.W_CAP = 0.0, 0.0
    d = synth.with_nets(d, [dict(pins=[(1, 3, 0, 1.0, -5.0), (5, 3, 0, 1.0, -5.0)], segs=[(1, 3, 5, 3)])])
    d.wire_dem0 = np.zeros(d.wire_cap.shape[0], np.int32)
    # hand values: M_pos(d-c) = e^{0.5(d-c+1)} - e^{0.5(d-c)}; via kappa = 0.05 + ofw[k] * M_pos(-16)
    Mpos = lambda dl: math.exp(0.5 * (dl + 1)) - math.exp(0.5 * dl)
    kap = [0.05 + (2.0 if k < 2 else 1.0) * Mpos(-16) for k in range(5)]
    cands = {}
    for j, ofw in ((0, 2.0), (2, 1.0), (4, 1.0)):
        S = 4 * Mpos(0 - 2)
        cands[j] = 2 * sum(kap[:j]) + ofw * S
    want = min(cands, key=lambda j: (cands[j], j))
    r = oracle.run(d)
    assert int(r["wires"][0][4]) == want
    assert r["net_cost"][0] == pytest.approx(cands[want], rel=1e-12)
    # now congest layer 0 heavily: the via stack becomes worth paying
    e = synth.with_nets(synth.empty_design(8, 8, 6, cap_wire=2, cap_via=16),
                        [dict(pins=[(1, 3, 0, 1.0, -5.0), (5, 3, 0, 1.0, -5.0)], segs=[(1, 3, 5, 3)])])
    e.W_D, e.W_CAP = 0.0, 0.0
    e.wire_dem0 = np.zeros(e.wire_cap.shape[0], np.int32)
    e.wire_dem0[: (e.X - 1) * e.Y] = 12          # layer 0: d - c = 10
    r2 = oracle.run(e)
    S0 = 4 * Mpos(10)
    cands[0] = 2.0 * S0
    want2 = min(cands, key=lambda j: (cands[j], j))
    assert want2 != 0 and int(r2["wires"][0][4]) == want2


def test_unit_weight_identity_cost_equals_net_rc():
    """W_CAP = W_CONG = W_VIA = 0, W_D = 1, WNS >= 0 with w_floor = 1: f[root] == net_rc bitwise
    (SURVEY c.5 'O6 vs O9'), and for single-sink nets without spurs it is the sink's Elmore delay."""
    d = tiny_pool(61, 6, n=300, X=12, Y=12, pin_max=6)
    d.W_CAP = d.W_CONG = d.W_VIA = 0.0
    d.W_D = 1.0
    d.wns, d.w_floor = 0.0, 1.0
    r = oracle.run(d)
    assert np.array_equal(r["net_cost"], r["net_rc"])
    two = np.where(np.diff(d.pin_ptr) == 2)[0]
    for net in two:
        assert r["net_cost"][net] == pytest.approx(r["sink_delay"][d.pin_ptr[net] + 1], rel=1e-9, abs=1e-15)


# ------------------------------------------------------------------ O8 commit + projection
def test_commit_invariants_and_projection():
    """Commit: final grid == rebuild from the emitted solution; wire
    demand added == wirelength; via demand added == layer changes; projection == the 2D input."""
    d = synth.make_config(1)
    r = oracle.run(d)
    wd, vd = rebuild_demand(d, r["wires"], r["vias"])
    assert np.array_equal(wd, r["wire_dem"]) and np.array_equal(vd, r["via_dem"])
    assert int(r["wire_dem"].sum()) == d.unit_edges_total()
    assert int(r["via_dem"].sum()) == int((r["vias"][:, 3] - r["vias"][:, 2]).sum())
    for net in range(d.n_nets):
        w = r["wires"][r["wire_ptr"][net]:r["wire_ptr"][net + 1]]
        proj = rc.unit_edges([tuple(int(t) for t in x[:4]) for x in w])
        assert proj == rc.unit_edges(rc.net_segs(d, net))
        for x in w:      # wires respect layer direction
            assert d.dir[x[4]] == (0 if x[1] == x[3] else 1)
    v = r["vias"]
    assert np.all(v[:, 3] > v[:, 2])


# ------------------------------------------------------------------ batching recurrence
def test_batch_recurrence_vs_bruteforce():
    """Conflict-free layering: batch(j) = 1 + max batch over earlier-priority nets
    whose footprints (unit edges U LA-node GCells) intersect j's, 0 if none -- by brute force."""
    d = synth.make_config(1)
    r = oracle.run(d, solution=False, grids=False, timing=False)
    order = sorted(range(d.n_nets), key=lambda i: (int(d.order_key[i]), i))
    fps = {}
    for net in range(d.n_nets):
        nodes = rc.build_tree(rc.net_pins(d, net), rc.net_segs(d, net))
        fps[net] = {("e",) + e for e in rc.unit_edges(rc.net_segs(d, net))} | {("g", n["x"], n["y"]) for n in nodes}
    want = {}
    for k, j in enumerate(order):
        b = 0
        for i in order[:k]:
            if fps[i] & fps[j]:
                b = max(b, want[i] + 1)
        want[j] = b
    assert [int(r["batch_of"][j]) for j in range(d.n_nets)] == [want[j] for j in range(d.n_nets)]


def _tie_design(pins, segs, L=6):
    """Tie-heavy setting (SURVEY c.5 'Test inputs that provoke ties'): identical r, c, ofw on all
    layers, W_VIA = W_CONG = W_D = 0, so many layer choices and spans cost exactly the same."""
    d = synth.empty_design(8, 8, L)
    d.r = np.full(L, 0.005)
    d.c = np.full(L, 0.2)
    d.ofw = np.ones(L)
    d.W_VIA = d.W_CONG = d.W_D = 0.0
    return synth.with_nets(d, [dict(pins=pins, segs=segs)])


def test_tie_break_son_lowest_layer():
    """Son argmin ties go to the lowest layer j (R21; Alg. 3 l.395 'argmin' with ties unspecified).
    Root pins on layers 0 and 2 force the root span to cover [0, 2], where H layers 0 and 2 tie."""
    d = _tie_design([(0, 0, 0, 1.0, -5.0), (0, 0, 2, 1.0, -5.0), (4, 0, 0, 1.0, -5.0)], [(0, 0, 4, 0)])
    r = oracle.run(d)
    assert int(r["wires"][0][4]) == 0


def test_tie_break_span_key():
    """Span ties on G' go to the smaller t - b, then the lower b (R21).  Pins on the V layer 1 at both
    ends of an H wire: spans (0,1) and (1,2) tie on cost and size; the lower b wins -> wire on layer 0."""
    d = _tie_design([(0, 0, 1, 1.0, -5.0), (4, 0, 1, 1.0, -5.0)], [(0, 0, 4, 0)])
    r = oracle.run(d)
    assert int(r["wires"][0][4]) == 0
    assert [tuple(int(t) for t in v) for v in r["vias"]] == [(0, 0, 0, 1), (4, 0, 0, 1)]


def test_evaluator_closed_forms():
    """oracle.evaluate (NEXT #3) against Eq. (3)/(2) closed forms: an edge with d = c
    contributes ofw(l) (e^0); c = 0, d = 2 contributes ofw(l) e^3 and d = c - 4 (c > 0)
    ofw(l) e^-2 (golden values, tests/golden/closed_forms.json); Eq. (2)
    counts only the positive excess.  Wirelength, via cuts and wire C by hand."""
    g = golden("closed_forms.json")["eq3"]
    d = synth.empty_design(3, 3, 2, cap_wire=5, cap_via=4)
    sizes = d.wire_layer_sizes()              # layer 0 (H): 2*3 edges, layer 1 (V): 3*2 edges
    assert list(sizes) == [6, 6]
    wcap = d.wire_cap.copy()
    wdem = wcap.copy()                        # every edge d = c ...
    wcap[0], wdem[0] = 0, 2                   # ... but edge 0 of layer 0: c = 0, d = 2
    wdem[7] = wcap[7] - 4                     # and edge 1 of layer 1: d = c - 4
    d.wire_cap = wcap
    vcap = d.via_cap.copy()
    vdem = vcap.copy()
    vdem[4] = vcap[4] + 3                     # one via cut 3 over capacity
    d.via_cap = vcap
    wires = [(0, 0, 2, 0, 0), (1, 0, 1, 2, 1)]   # 2 unit edges on layer 0, 2 on layer 1
    vias = [(0, 0, 0, 1), (1, 2, 0, 1)]
    ev = oracle.evaluate(d, wdem, vdem, wires, vias)
    ofw0, ofw1 = float(d.ofw[0]), float(d.ofw[1])
    want_w = ofw0 * (5 + g["state_c0_d2"]) + ofw1 * (5 + g["state_d_eq_c_minus_4_cpos"])
    assert abs(ev["tof_wire"] - want_w) <= 1e-12 * want_w
    want_v = ofw0 * (8 + np.e ** 1.5)        # 8 cuts at d = c, one at d = c + 3 (c > 0: s = 0.5 -> e^1.5)
    assert abs(ev["tof_via"] - want_v) <= 1e-12 * want_v
    assert ev["legacy_wire"] == 2 and ev["legacy_via"] == 3
    assert ev["wirelength"][:2] == [2, 2] and sum(ev["wirelength"]) == 4
    assert ev["via_cuts"] == 2
    assert abs(ev["wire_cap"] - (2 * d.c[0] + 2 * d.c[1])) <= 1e-15


def test_snapshot_batches_reduce_to_known_schedules():
    """Oracle snapshot batches (NEXT #1, reading R31) pinned by the two schedules it must reduce
    to: one net per batch is sequential assignment; a batch of nets that pairwise share no
    footprint element (the conflict-free recurrence) is sequential too; and
    one batch of everything gives every net the initial demand, i.e. the solution of running
    each net alone on the initial grid."""
    d = tiny_pool(81, 6, n=120, X=8, Y=8, pin_max=5)
    seq = oracle.run(d)
    one_each = oracle.run(d, snap_batch=np.argsort(np.argsort(d.order_key, kind="stable"), kind="stable"))
    for k in ("wires", "vias", "wire_dem", "via_dem", "net_cost"):
        assert np.array_equal(one_each[k], seq[k]), k
    cf = oracle.run(d, snap_batch=seq["batch_of"])
    for k in ("wires", "vias", "wire_dem", "via_dem", "net_cost"):
        assert np.array_equal(cf[k], seq[k]), k
    allin = oracle.run(d, snap_batch=np.zeros(d.n_nets, np.int32))
    wires, vias = [], []
    for j in range(d.n_nets):
        r = oracle.run(single_net(d, j))
        wires.append(r["wires"])
        vias.append(r["vias"])
        assert r["net_cost"][0] == allin["net_cost"][j]
    assert np.array_equal(np.concatenate(wires), allin["wires"])
    assert np.array_equal(np.concatenate(vias) if vias else allin["vias"], allin["vias"])
    wd, vd = rebuild_demand(d, allin["wires"], allin["vias"])
    assert np.array_equal(wd, allin["wire_dem"]) and np.array_equal(vd, allin["via_dem"])


def test_paper_batches_by_hand():
    """Alg. 1 lines 3-10 (oracle.paper_batches) on eight hand-made nets, WNS = -100, alpha 0.7,
    th 3: criticality 8, 8, 5, 4 are critical (bands [8, 8] then [4, 8)); net slacks -98 and -80
    are semi-critical (< -70), in slack bands (-99, -96] and (-84, -75]; -60 and +10 are not,
    and go by 2D wirelength."""
    # nets: (criticality, sink slack, wirelength)
    spec = [(8, -90, 3), (8, -95, 1), (5, -50, 2), (4, -99, 5), (0, -98, 2), (1, -80, 4), (0, 10, 7), (2, -60, 1)]
    pin_ptr, slacks, seg_ptr, segs = [0], [], [0], []
    for c, s, w in spec:
        slacks += [0.0, float(s)]
        pin_ptr.append(len(slacks))
        segs.append((0, 0, w, 0))
        seg_ptr.append(len(segs))
    crit = [c for c, _, _ in spec]
    b, nb = oracle.paper_batches(pin_ptr, slacks, seg_ptr, segs, -100.0, crit, 0.7, 3, max_batch=1)
    # order: [8,8] band by slack: net1 (-95), net0 (-90); [4,8): net2 (5), net3 (4); semi: net4 (-98, band 1),
    # net5 (-80, band 5); non-critical by wirelength: net7 (1), net6 (7)
    assert nb == 8
    assert list(b) == [1, 0, 2, 3, 4, 5, 7, 6]
    b2, nb2 = oracle.paper_batches(pin_ptr, slacks, seg_ptr, segs, -100.0, crit, 0.7, 3, max_batch=100)
    assert nb2 == 5 and list(b2) == [0, 0, 1, 1, 2, 3, 4, 4]


# ------------------------------------------------------------------ O3 look-ahead
def _tree_ids(d, net=0):
    """(x, y) -> oracle node id."""
    return {(int(r[0]), int(r[1])): i for i, r in enumerate(oracle.tree(d, net))}


@pytest.mark.parametrize("r_avg", [0.003, float("nan")])
def test_ur_chain_closed_form(r_avg):
    """O3 closed form on a chain (SURVEY §8(c) c.5 'O3 ur'; PAPER l.452 'node distances and the
    average unit-length metal resistance r_avg'; reading R6): pins along one straight run give a
    chain root -> n1 -> n2 -> n3 with ur(n_k) = r_drv + r_avg * (distance from the driver), strictly
    increasing.  r_avg = NaN means the mean r of the routable layers (Alg. 1 input, l.240)."""
    d = synth.empty_design(12, 6, 6)
    d.r_avg = r_avg
    d.routable = np.array([1, 1, 1, 1, 0, 1], np.uint8)
    ra = 0.003 if r_avg == r_avg else float(np.mean(d.r[[0, 1, 2, 3, 5]]))
    d = synth.with_nets(d, [dict(pins=[(0, 2, 0, 1.0, -5.0), (2, 2, 0, 1.0, -5.0), (5, 2, 1, 1.0, -5.0),
                                       (9, 2, 0, 1.0, -5.0)], segs=[(0, 2, 9, 2)], r_drv=1.25)])
    ids = _tree_ids(d)
    ur = oracle.net_dp(d, 0)["ur"]
    got = [ur[ids[(x, 2)]] for x in (0, 2, 5, 9)]
    want = [1.25 + ra * x for x in (0, 2, 5, 9)]
    assert got[0] == 1.25                                        # ur(root) = r_drv exactly
    for g_, w_ in zip(got, want):
        assert g_ == pytest.approx(w_, rel=1e-15)
    assert all(a < b for a, b in zip(got, got[1:]))


def _fig8_design(case):
    G = golden("lookahead_fig8.json")
    t, w, n = G["tech"], G["weights"], G["net"]
    d = synth.empty_design(8, 8, t["L"])
    d.dir = np.array(t["dir"], np.uint8)
    d.routable = np.array(t["routable"], np.uint8)
    d.r, d.c, d.vr = (np.array(t[k], np.float64) for k in ("r", "c", "vr"))
    d.r_avg = t["r_avg"]
    for k in ("W_D", "W_CAP", "W_CONG", "W_VIA", "w_floor"):
        setattr(d, k, w[k])
    d = synth.with_nets(d, [dict(pins=[tuple(p) for p in n["pins"]], segs=[tuple(s) for s in n["segs"]],
                                 r_drv=G["cases"][case]["r_drv"])])
    d.wns = w["wns"]
    return d, G["cases"][case]


@pytest.mark.parametrize("case", ["r_drv_0", "r_drv_0p04"])
def test_lookahead_fig8_hand_example(case):
    """The paper's look-ahead example on the Fig. 8 tree (f'_6 = ... + w^d (d_67 +
    r^est_6 c_6)), worked by hand in tests/golden/lookahead_fig8.json: ur of every node, the two
    cost' candidates of son 7 at node 6, the full solution and the net cost.  With r_drv = 0.04 the
    look-ahead moves edge 67 from layer 0 (plain cost) to layer 2; with r_drv = 0 it does not."""
    d, want = _fig8_design(case)
    ids = _tree_ids(d)
    coord = {"3": (0, 0), "4": (2, 0), "5": (4, 0), "6": (2, 3), "7": (4, 3)}
    dp = oracle.net_dp(d, 0)
    for k, u in want["ur"].items():
        assert dp["ur"][ids[coord[k]]] == pytest.approx(u, rel=1e-12, abs=1e-15), ("ur", k)
    j = want["layers"]["67"]
    # node 6, entry 1: G' = V(b, t) + cost'(1; 7, j*) with V = 0 (W_VIA = W_CONG = 0)
    assert dp["gp"][ids[coord["6"]]][1] == pytest.approx(want["node6_cost_prime"][str(j)], rel=1e-12)
    assert min(want["node6_cost_prime"].values()) == want["node6_cost_prime"][str(j)]
    r = oracle.run(d)
    edge = {"34": (0, 0, 2, 0), "45": (2, 0, 4, 0), "46": (2, 0, 2, 3), "67": (2, 3, 4, 3)}
    lay = {tuple(int(v) for v in w[:4]): int(w[4]) for w in r["wires"]}
    assert {k: lay[e] for k, e in edge.items()} == want["layers"]
    assert sorted(tuple(int(v) for v in x) for x in r["vias"]) == sorted(tuple(x) for x in want["vias"])
    assert r["net_cost"][0] == pytest.approx(want["net_cost"], rel=1e-12)


@pytest.mark.parametrize("seed,L,r_avg", [(131, 4, float("nan")), (132, 6, 0.05), (133, 4, 0.2), (134, 6, 0.01)])
def test_node_local_enumeration(seed, L, r_avg):
    """SURVEY §8(c) c.5 (iii)/(iv) on random nets with W_D > 0 and r_drv > 0 (look-ahead live):
    for every node and entry layer, the minimum over ALL son-layer tuples (each with its minimal
    covering via span, tests/refcheck.py) equals the oracle's span-DP G' bitwise; the oracle's span
    and son layers are the unique minimiser's; cost' - cost = ur_n * sum B (iv); f = F0 + G; and
    ur / wd equal an independent top-down walk."""
    checked = unique = 0
    for d, nodes in _dp_cases(seed, L, rdrv_mode=1, max_nodes=8, want=40):
        d.W_D = 100.0
        d.r_avg = r_avg
        omap = rc.oracle_node_map(nodes, oracle.tree(d, 0))
        c, u = rc.node_local_enumeration(d, 0, nodes, oracle.net_dp(d, 0), omap)
        checked += c
        unique += u
    assert checked > 100 and unique > checked // 2


def test_lookahead_is_live_on_random_nets():
    """The pins above exercise a live term: on the same random pool, switching the look-ahead
    off (r_drv = r_avg = 0, the Table IV 'w/o ahead' ablation) changes the
    chosen layers of some nets."""
    changed = 0
    for d, nodes in _dp_cases(133, 4, rdrv_mode=1, max_nodes=8, want=150):
        d.W_D, d.r_avg = 1000.0, 0.2
        a = oracle.run(d)
        e = copy.copy(d)
        e.r_avg = 0.0
        e.r_drv = np.zeros_like(d.r_drv)
        b = oracle.run(e)
        changed += int(not np.array_equal(a["wires"], b["wires"]))
    assert changed >= 3


def test_eq3_clamp_outside_table_domain():
    """Reading R20: d - c outside [delta_lo, delta_hi] clamps to the nearest end of the table.
    Straight 2-pin net on layer 0 only (other H layers unroutable), W_D = W_CAP = W_VIA = 0:
    the cost is ofw[0] * sum of M_pos over the run's edges, by hand, with d - c = 10 > delta_hi = 2
    on the first edge and -8 < delta_lo = -3 on the second."""
    d = synth.empty_design(8, 8, 4, cap_wire=5, cap_via=16)
    d.delta_lo, d.delta_hi = -3, 2
    d.routable = np.array([1, 1, 0, 1], np.uint8)
    d.W_D = d.W_CAP = d.W_VIA = 0.0
    d = synth.with_nets(d, [dict(pins=[(1, 4, 0, 1.0, -5.0), (3, 4, 0, 1.0, -5.0)], segs=[(1, 4, 3, 4)])])
    d.wire_dem0 = np.zeros(d.wire_cap.shape[0], np.int32)
    d.wire_dem0[4 * (d.X - 1) + 1] = 15        # layer 0 edge (1,4)-(2,4): d - c = 10 -> clamp to 2
    d.wire_dem0[4 * (d.X - 1) + 2] = 0         # layer 0 edge (2,4)-(3,4): d - c = -5 -> clamp to -3
    d.wire_cap = d.wire_cap.copy()
    d.wire_cap[4 * (d.X - 1) + 2] = 8          # ... make it -8
    M = lambda dl: math.exp(0.5 * (dl + 1)) - math.exp(0.5 * dl)
    # via cuts: the pins sit on layer 0 = the wire layer, so no vias; V = 0
    want = 2.0 * (M(2) + M(-3))                # ofw[0] = 2 (generator tech, d.2)
    r = oracle.run(d)
    assert int(r["wires"][0][4]) == 0 and len(r["vias"]) == 0
    assert r["net_cost"][0] == pytest.approx(want, rel=1e-14)
    assert r["net_cost"][0] != pytest.approx(2.0 * (M(10) + M(-8)), rel=1e-6)
