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


def _dir_rc(d, r_h, r_v, c_h, c_v):
    return (r_h, r_v), (c_h, c_v)


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
