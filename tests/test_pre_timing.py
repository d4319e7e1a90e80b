"""Pre-assignment pi-model timing on the 2D trees (PAPER §III-B l.283-286,
Alg. 1 inputs r_avg / c_avg l.240-241; reading R44 in DESIGN.md).

CPU part (-m "not gpu"): pins of oracle.pre_timing against hand-worked fixtures
(tests/golden/pre_timing_fixtures.json), an independent Elmore on the unit-edge graph (every
unit 2D edge its own pi section: the pi model is exact under subdivision of a uniform wire, so
the LA tree's lumped runs must give the same delays), and the net-cap closed form.
GPU part (-m gpu): la_pre_timing (k_pre_timing) against the oracle, element by element.
"""
import math

import numpy as np
import pytest

import refcheck as rc
from gen import synth
from helpers import golden
from oracle import oracle

NAN = float("nan")


def _fixture(name):
    g = golden("pre_timing_fixtures.json")
    fx = g[name]
    d = synth.empty_design(8, 8, 4)
    d = synth.with_nets(d, [dict(pins=[tuple(p) for p in fx["pins"]], segs=[tuple(s) for s in fx["segs"]])])
    return d, g["rc"], fx


@pytest.mark.parametrize("name", ["L", "T", "driver_cell"])
def test_pre_timing_hand_fixtures(name):
    """Hand-worked pi-model Elmore values (golden)."""
    d, r, fx = _fixture(name)
    delay, cap = oracle.pre_timing(d, r["r_h"], r["r_v"], r["c_h"], r["c_v"])
    assert delay.tolist() == pytest.approx(fx["delay"], rel=1e-15, abs=0)
    assert cap[0] == pytest.approx(fx["net_cap"], rel=1e-15)


def unit_graph_elmore(d, net, rd, cd):
    """Elmore on the route's unit-edge graph: each unit edge (a, b) of direction t is a pi
    section r_t, c_t (c_t / 2 at each end); cell cap = its sinks' caps + the halves of its
    incident unit edges; delay(cell) = delay(parent) + r_t * (cap of the cell's subtree)."""
    pins = rc.net_pins(d, net)
    segs = rc.net_segs(d, net)
    es = rc.unit_edges(segs)
    adj = {}
    for a, b in es:
        adj.setdefault(a, []).append(b)
        adj.setdefault(b, []).append(a)
    root = (pins[0][0], pins[0][1])
    par, order = {root: None}, [root]
    i = 0
    while i < len(order):
        g = order[i]
        i += 1
        for h in adj.get(g, []):
            if h not in par:
                par[h] = g
                order.append(h)
    t_of = lambda a, b: 0 if a[1] == b[1] else 1
    cap = {g: 0.0 for g in order}
    for q, p in enumerate(pins):
        if q > 0:
            cap[(p[0], p[1])] += p[3]
    for a, b in es:
        t = t_of(a, b)
        cap[a] += 0.5 * cd[t]
        cap[b] += 0.5 * cd[t]
    down = dict(cap)
    for g in reversed(order):
        if par[g] is not None:
            down[par[g]] += down[g]
    D = {root: 0.0}
    for g in order[1:]:
        D[g] = D[par[g]] + rd[t_of(par[g], g)] * down[g]
    delays = [0.0] + [D[(p[0], p[1])] for p in pins[1:]]
    return delays, sum(cap.values())


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_pre_timing_vs_unit_edge_graph(seed):
    """The oracle's lumped LA-tree pi model == the unit-edge pi ladder (exact under subdivision:
    n sections of (r, c) into a load C_L give n r C_L + r c n^2 / 2 = R (C / 2 + C_L))."""
    d = synth.generate(n_nets=300, X=24, Y=24, L=6, seed=seed, pin_max=12, name=f"pre_{seed}")
    rd, cd = (0.37, 0.21), (1.7, 2.9)
    delay, cap = oracle.pre_timing(d, rd[0], rd[1], cd[0], cd[1])
    for net in range(d.n_nets):
        want, wcap = unit_graph_elmore(d, net, rd, cd)
        a = int(d.pin_ptr[net])
        got = delay[a:a + len(want)]
        for x, y in zip(got.tolist(), want):
            assert math.isclose(x, y, rel_tol=1e-11, abs_tol=1e-12), (net, got, want)
        assert math.isclose(cap[net], wcap, rel_tol=1e-12), net


def test_pre_timing_net_cap_closed_form_and_default_rc():
    """net_cap = sum of sink caps + c_h * (H wirelength) + c_v * (V wirelength) straight from the
    segments; NaN unit values = the mean over the routable layers of that direction (R44)."""
    d = synth.generate(n_nets=500, X=32, Y=32, L=6, seed=11, pin_max=20, name="pre_cap")
    r = np.asarray(d.r, np.float64)
    c = np.asarray(d.c, np.float64)
    dirs, rt = np.asarray(d.dir), np.asarray(d.routable).astype(bool)
    rh, rv = r[rt & (dirs == 0)].mean(), r[rt & (dirs == 1)].mean()
    ch, cv = c[rt & (dirs == 0)].mean(), c[rt & (dirs == 1)].mean()
    delay, cap = oracle.pre_timing(d)
    delay2, cap2 = oracle.pre_timing(d, rh, rv, ch, cv)
    np.testing.assert_allclose(delay, delay2, rtol=1e-14, atol=0)
    np.testing.assert_allclose(cap, cap2, rtol=1e-14, atol=0)
    for net in range(d.n_nets):
        es = rc.unit_edges(rc.net_segs(d, net))
        wh = sum(1 for a, b in es if a[1] == b[1])
        wv = len(es) - wh
        sinks = d.pin_cap[int(d.pin_ptr[net]) + 1:int(d.pin_ptr[net + 1])].sum()
        assert math.isclose(cap[net], sinks + ch * wh + cv * wv, rel_tol=1e-12), net
    drv = d.pin_ptr[:-1]
    assert np.all(delay[drv] == 0.0) and np.all(delay >= 0.0)


# ------------------------------------------------------------------ GPU parity (la_pre_timing)
@pytest.fixture(scope="module")
def la():
    import __graft_entry__ as ge
    ge.build()
    from paper_2507_13375_b200 import la as mod
    return mod


def _gpu_pre(la, d, *rc_vals):
    A = la.LayerAssigner(d, device=0)
    A.load()
    out = la.la_pre_timing(A.ctx, int(d.pin_ptr[-1]), d.n_nets, *rc_vals)
    A.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["fixtures", "cfg1", "cfg2", "cfg4_sample", "explicit_rc"])
def test_pre_timing_gpu_parity(la, case):
    """k_pre_timing == oracle.pre_timing element by element within 1e-9 relative (the north
    star's fp64 tolerance; the two sum the same terms in different orders).  cfg4_sample holds
    64-256-pin nets (the windowed big-net path) next to the chunked small nets."""
    rcv = ()
    if case == "fixtures":
        g = golden("pre_timing_fixtures.json")
        d = synth.empty_design(8, 8, 4)
        d = synth.with_nets(d, [dict(pins=[tuple(p) for p in g[k]["pins"]], segs=[tuple(s) for s in g[k]["segs"]])
                                for k in ("L", "T", "driver_cell")])
        rcv = (g["rc"]["r_h"], g["rc"]["r_v"], g["rc"]["c_h"], g["rc"]["c_v"])
    elif case == "cfg1":
        d = synth.make_config(1)
    elif case == "cfg2":
        d = synth.make_config(2)
    elif case == "cfg4_sample":
        d = synth.generate(n_nets=40_000, X=512, Y=512, L=13, seed=104, hf_frac=0.01, rdrv_mode=1, name="pre_hf")
    else:
        d = synth.make_config(2, n_nets=20_000)
        rcv = (0.0123, 0.0456, 0.31, 0.27)
    got_d, got_c = _gpu_pre(la, d, *rcv)
    ref_d, ref_c = oracle.pre_timing(d, *rcv)
    np.testing.assert_allclose(got_d, ref_d, rtol=1e-9, atol=0.0)
    np.testing.assert_allclose(got_c, ref_c, rtol=1e-9, atol=0.0)
    assert np.all(got_d[d.pin_ptr[:-1]] == 0.0)
    if case == "fixtures":
        assert got_d.tolist() == pytest.approx(sum((g[k]["delay"] for k in ("L", "T", "driver_cell")), []), rel=1e-15)


@pytest.mark.gpu
def test_pre_timing_gpu_full_cfg3_sampled(la):
    """Config 3 at full size (1M nets) through the bench's launch: 2,000 nets sampled across
    the forest compared with the oracle run on exactly those nets."""
    d = synth.make_config(3)
    got_d, got_c = _gpu_pre(la, d)
    rng = np.random.default_rng(3)
    nets = np.sort(rng.choice(d.n_nets, 2000, replace=False))
    from helpers import single_net
    for j in nets:
        e = single_net(d, int(j))
        rd, rcap = oracle.pre_timing(e)
        a, b = int(d.pin_ptr[j]), int(d.pin_ptr[j + 1])
        np.testing.assert_allclose(got_d[a:b], rd, rtol=1e-9, atol=0.0)
        assert math.isclose(got_c[j], rcap[0], rel_tol=1e-9)


# ------------------------------------------------------------------ GPU Alg. 1 (la_paper_batches)
def _gpu_batches(la, d, crit, alpha=0.7, th=3, mb=1 << 20):
    A = la.LayerAssigner(d, device=0)
    try:
        return la.la_paper_batches(A.ctx, d, crit, alpha, th, mb)
    finally:
        A.close()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg1_50", "cfg2_1000", "cfg2_ties", "wns_pos", "all_critical", "th0_cap1"])
def test_paper_batches_gpu_equals_oracle(la, case):
    """Alg. 1 lines 3-10 on the GPU == oracle.paper_batches, batch ids bit-exact (integer work),
    including ties of slack / criticality / wirelength (index order decides), WNS >= 0 (no
    semi-critical class), every net critical, and a size cap of one net per batch."""
    d = synth.make_config(2 if "cfg2" in case or case in ("wns_pos", "all_critical", "th0_cap1") else 1)
    crit = synth.criticality(d, 1)
    alpha, th, mb = 0.7, 3, 50
    if case == "cfg2_1000":
        mb = 1000
    elif case == "cfg2_ties":
        d.pin_slack = np.round(d.pin_slack / 50.0) * 50.0       # many equal net slacks
        crit = (crit // 2) * 2
        mb = 333
    elif case == "wns_pos":
        d.wns = 10.0
        mb = 777
    elif case == "all_critical":
        crit = crit + 4
        mb = 5000
    elif case == "th0_cap1":
        d = synth.make_config(1)
        crit = synth.criticality(d, 2)
        th, mb = 0, 1
    got, nb = _gpu_batches(la, d, crit, alpha, th, mb)
    ref, nbr = oracle.paper_batches(d.pin_ptr, d.pin_slack, d.seg_ptr, d.seg_xy, d.wns, crit, alpha, th, mb)
    assert nb == nbr
    if not np.array_equal(got, ref):
        bad = np.flatnonzero(got != ref)
        raise AssertionError(f"{bad.size} nets differ, first {bad[:5].tolist()}: {got[bad[:5]]} vs {ref[bad[:5]]}")


@pytest.mark.gpu
def test_paper_batches_gpu_argument_errors(la):
    """la_paper_batches validates its arguments (include/la.h): alpha > 0, th >= 0,
    max_batch >= 1, non-negative criticality."""
    d = synth.make_config(1)
    crit = np.zeros(d.n_nets, np.int32)
    A = la.LayerAssigner(d, device=0)
    try:
        for kw in (dict(alpha=0.0), dict(mb=0), dict(th=-1)):
            args = dict(alpha=0.7, th=3, mb=100)
            args.update(kw)
            with pytest.raises(la.LaError) as ei:
                la.la_paper_batches(A.ctx, d, crit, args["alpha"], args["th"], args["mb"])
            assert ei.value.status == la.LA_EINVAL
        bad = crit.copy()
        bad[3] = -1
        with pytest.raises(la.LaError, match="criticality"):
            la.la_paper_batches(A.ctx, d, bad)
        b, nb = la.la_paper_batches(A.ctx, d, crit, max_batch=10**9)
        assert nb >= 1 and b.min() == 0 and b.max() == nb - 1
    finally:
        A.close()
