"""GPU (CUDA, sm_100a) vs CPU oracle parity, through the C ABI.

Bar (BASELINE.json north_star): layer choices, via spans, demand grids
and batch ids bit-exact; net cost f[root], sink delays, net caps and net RC sums
within 1e-9 relative (and, by the shared expression-order contract, expected
bitwise -- checked separately so a rounding-order drift is visible on its own).
"""
import copy

import numpy as np
import pytest

import refcheck as rc
from gen import synth
from helpers import randomize_state
from oracle import oracle

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def la():
    import __graft_entry__ as ge
    ge.build()
    from paper_2507_13375_b200 import la as mod
    return mod


def run_gpu(la, d, per_batch=False, schedule=None):
    A = la.LayerAssigner(d, device=0)
    nb = A.load()
    if schedule is not None:
        A.set_schedule(schedule)
    if per_batch:
        for k in range(nb):
            A.assign_batch(k)
            A.commit_demand(k)
        out = A.eval_timing()
        out.update(A.solution())
        wd, vd = A.demand()
        out.update(wire_dem=wd, via_dem=vd, batch_of=A.batches())
    else:
        out = A.run()
    out["stats"] = A.stats()
    out["n_batches"] = nb
    A.close()
    return out


def assert_parity(got, ref, bitwise_fp=False):
    for k in ("wire_ptr", "wires", "via_ptr", "vias", "wire_dem", "via_dem", "batch_of"):
        a, b = np.asarray(got[k]), np.asarray(ref[k])
        assert a.shape == b.shape, (k, a.shape, b.shape)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)[:5]
            raise AssertionError(f"{k}: {int((a != b).sum())} mismatches, first at {bad.tolist()}")
    for k in ("net_cost", "sink_delay", "net_cap", "net_rc"):
        a, b = got[k], ref[k]
        np.testing.assert_allclose(a, b, rtol=RTOL, atol=0.0, err_msg=k)
        if bitwise_fp:
            assert np.array_equal(a, b), f"{k}: not bitwise equal ({int((a != b).sum())} values)"


@pytest.mark.parametrize("cfg", [1, 2])
def test_config_parity(la, cfg):
    d = synth.make_config(cfg)
    got = run_gpu(la, d)
    ref = oracle.run(d)
    assert_parity(got, ref)
    assert got["n_batches"] == int(ref["batch_of"].max()) + 1


def test_config3_parity_full(la):
    """Config 3 (1M nets, 1024^2, L = 10, criticality-weighted, r_drv > 0) at full size."""
    d = synth.make_config(3)
    got = run_gpu(la, d)
    ref = oracle.run(d)
    assert_parity(got, ref)


def test_config4_parity_sample(la):
    """Config 4's grid / 13 layers / high-fanout mix (64-256 pins) at 400K nets."""
    d = synth.make_config(4, n_nets=400_000)
    got = run_gpu(la, d)
    ref = oracle.run(d)
    assert got["stats"]["max_net_nodes"] > 64
    assert_parity(got, ref)


@pytest.mark.parametrize("cfg", [1, 2])
def test_bitwise_fp(la, cfg):
    """Shared expression-order contract: costs, delays, caps bitwise equal."""
    d = synth.make_config(cfg)
    assert_parity(run_gpu(la, d), oracle.run(d), bitwise_fp=True)


def test_per_batch_api_equals_assign_all(la):
    d = synth.make_config(1)
    a = run_gpu(la, d, per_batch=True)
    b = run_gpu(la, d, per_batch=False)
    for k in ("wires", "vias", "wire_dem", "via_dem", "net_cost", "sink_delay"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("cfg,n", [(2, None), (4, 150_000)])
def test_dataflow_equals_batch_schedule(la, cfg, n):
    """the one-launch dataflow schedule and the batch-by-batch schedule
    give bit-identical results (big nets, global-scratch nets and ties included)."""
    d = synth.make_config(cfg, n_nets=n)
    a = run_gpu(la, d, schedule=la.LA_SCHED_DATAFLOW)
    b = run_gpu(la, d, schedule=la.LA_SCHED_BATCH)
    for k in ("wires", "vias", "wire_dem", "via_dem", "net_cost", "sink_delay", "net_cap", "net_rc"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("sched", ["dataflow", "batch"])
def test_dense_conflicts_deep_dag(la, sched):
    """20K nets on a 24x24 grid: long conflict chains (hundreds of batches), so the
    dataflow schedule's waits and releases are exercised on every net, and the
    batch schedule launches hundreds of mostly tiny batches."""
    d = synth.generate(20_000, 24, 24, 6, seed=77, pin_max=16, rdrv_mode=1, name="dense")
    got = run_gpu(la, d, schedule=la.LA_SCHED_DATAFLOW if sched == "dataflow" else la.LA_SCHED_BATCH)
    ref = oracle.run(d)
    assert got["n_batches"] > 200
    assert_parity(got, ref, bitwise_fp=True)


def test_reset_and_rerun_identical(la):
    d = synth.make_config(1)
    A = la.LayerAssigner(d)
    A.load()
    first = A.run()
    A.reset()
    second = A.run()
    A.close()
    for k in ("wires", "vias", "wire_dem", "via_dem", "net_cost", "sink_delay", "net_rc"):
        assert np.array_equal(first[k], second[k]), k


# --------------------------------------------------------------- edge cases
def _hand(L=6, X=12, Y=12, **kw):
    d = synth.empty_design(X, Y, L)
    for k, v in kw.items():
        setattr(d, k, v)
    return d


def test_empty_design(la):
    d = synth.with_nets(_hand(), [])
    got = run_gpu(la, d)
    assert got["n_batches"] == 0 and len(got["wires"]) == 0 and got["wire_dem"].sum() == 0


def test_degenerate_nets(la):
    """Single-GCell nets (R38), pins on high layers, several pins per GCell (R29), a dangling spur (R39),
    overlapping input segments (R30), same-direction continuation at a pin node (R40), a ring-free plus."""
    nets = [
        dict(pins=[(3, 3, 0, 1.0, -50.0), (3, 3, 4, 0.7, -400.0), (3, 3, 2, 1.1, 10.0)], segs=[]),
        dict(pins=[(0, 0, 5, 1.0, -1.0), (5, 0, 3, 1.0, -450.0)], segs=[(0, 0, 5, 0)]),
        dict(pins=[(1, 5, 1, 1.0, -30.0), (4, 5, 0, 2.0, -300.0)], segs=[(1, 5, 6, 5)]),              # spur to (6,5)
        dict(pins=[(2, 8, 0, 1.0, -5.0), (7, 8, 1, 1.0, -5.0)], segs=[(2, 8, 5, 8), (4, 8, 7, 8)]),    # overlap
        dict(pins=[(1, 10, 0, 1.0, -5.0), (4, 10, 0, 1.0, -490.0), (8, 10, 2, 1.0, -100.0)], segs=[(1, 10, 8, 10)]),
        dict(pins=[(9, 3, 0, 1.0, 0.0), (9, 5, 0, 1.0, -10.0), (9, 1, 0, 1.0, -20.0), (11, 3, 0, 1.0, -30.0),
                   (7, 3, 0, 1.0, -40.0)], segs=[(9, 1, 9, 5), (7, 3, 11, 3)], r_drv=1.5),
    ]
    d = synth.with_nets(_hand(), nets)
    assert_parity(run_gpu(la, d), oracle.run(d), bitwise_fp=True)


@pytest.mark.parametrize("L", [2, 3, 4, 16])
def test_layer_counts(la, L):
    d = synth.generate(n_nets=3000, X=40, Y=40, L=L, seed=70 + L, pin_max=16, rdrv_mode=1)
    assert_parity(run_gpu(la, d), oracle.run(d))


def test_random_state_ties_and_zero_caps(la):
    """Random initial demand, many zero capacities (s_zero), tie-heavy tech (identical layers)."""
    rng = np.random.default_rng(5)
    d = synth.generate(n_nets=4000, X=48, Y=48, L=8, seed=81, pin_max=32, rdrv_mode=1)
    d = randomize_state(d, rng, wire_caps=(0, 0, 1, 2, 5), via_caps=(0, 1, 8), wire_dem=3, via_dem=3)
    e = copy.copy(d)
    e.r, e.c, e.ofw = np.full(8, 0.004), np.full(8, 0.18), np.ones(8)
    e.W_VIA = 0.0
    for dd in (d, e):
        assert_parity(run_gpu(la, dd), oracle.run(dd), bitwise_fp=True)


@pytest.mark.parametrize("wd,wns", [(0.0, -500.0), (1e4, -500.0), (100.0, 25.0)])
def test_weight_regimes(la, wd, wns):
    d = synth.generate(n_nets=5000, X=64, Y=64, L=10, seed=91, pin_max=63, rdrv_mode=1)
    d.W_D, d.wns = wd, wns
    assert_parity(run_gpu(la, d), oracle.run(d))


def test_unrouteable_direction_layers(la):
    """Some layers not routable (R15): they never carry wires, still carry vias."""
    d = synth.generate(n_nets=3000, X=40, Y=40, L=8, seed=95, pin_max=16)
    d.routable = np.array([0, 1, 1, 0, 1, 1, 0, 1], np.uint8)
    got, ref = run_gpu(la, d), oracle.run(d)
    assert_parity(got, ref)
    assert set(np.unique(got["wires"][:, 4])).isdisjoint({0, 3, 6})


# --------------------------------------------------------------- ABI errors on the device path
def test_call_order_errors(la):
    d = synth.make_config(1, n_nets=200)
    A = la.LayerAssigner(d)
    nb = A.load()
    assert nb >= 2
    with pytest.raises(la.LaError) as e:
        la.la_assign_batch(A.ctx, 1)
    assert e.value.status == la.LA_ESTATE
    with pytest.raises(la.LaError) as e:
        la.la_assign_batch(A.ctx, nb)
    assert e.value.status == la.LA_ERANGE
    with pytest.raises(la.LaError) as e:
        la.la_commit_demand(A.ctx, 0)
    assert e.value.status == la.LA_ESTATE
    with pytest.raises(la.LaError) as e:
        A.eval_timing()
    assert e.value.status == la.LA_ESTATE
    with pytest.raises(la.LaError) as e:
        A.load()
    assert e.value.status == la.LA_ESTATE
    A.assign_all()
    A.eval_timing()
    A.close()


@pytest.mark.parametrize("net,msg", [
    (dict(pins=[(0, 0, 0, 1, 0), (2, 2, 0, 1, 0)], segs=[(0, 0, 2, 0), (2, 0, 2, 2), (0, 0, 0, 2), (0, 2, 2, 2)]),
     "not a tree"),
    # a cycle plus a separate run: vertices = edges + 1, so the DFS itself must find the cycle
    # (driver on the square) or the unreached component (driver on the separate run)
    (dict(pins=[(0, 0, 0, 1, 0), (2, 2, 0, 1, 0)],
          segs=[(0, 0, 2, 0), (2, 0, 2, 2), (0, 0, 0, 2), (0, 2, 2, 2), (4, 4, 5, 4)]), "not a tree"),
    (dict(pins=[(4, 4, 0, 1, 0), (5, 4, 0, 1, 0), (2, 2, 0, 1, 0)],
          segs=[(0, 0, 2, 0), (2, 0, 2, 2), (0, 0, 0, 2), (0, 2, 2, 2), (4, 4, 5, 4)]), "not a tree"),
    (dict(pins=[(0, 0, 0, 1, 0), (3, 3, 0, 1, 0)], segs=[(0, 0, 2, 0)]), "not on the route"),
    (dict(pins=[(0, 0, 0, 1, 0), (2, 2, 0, 1, 0)], segs=[(0, 0, 2, 2)]), "axis-aligned"),
    (dict(pins=[(0, 0, 0, 1, 0), (2, 0, 9, 1, 0)], segs=[(0, 0, 2, 0)]), "layer"),
    (dict(pins=[(0, 0, 0, 1, 0), (2, 0, 0, 1, 0)], segs=[(0, 0, 40, 0)]), "outside"),
])
def test_route_errors(la, net, msg):
    d = synth.with_nets(_hand(), [dict(pins=[(5, 5, 0, 1, 0), (6, 5, 0, 1, 0)], segs=[(5, 5, 6, 5)]), net])
    A = la.LayerAssigner(d)
    with pytest.raises(la.LaError, match=msg) as e:
        A.load()
    assert e.value.status == la.LA_EINVAL and "net 1" in str(e.value)
    A.close()


# --------------------------------------------------------------- properties at full scale
@pytest.mark.slow
def test_config5_full_scale_properties(la):
    """Config 5 (12M nets, 4096^2, L = 13) in the bench's launch configuration: projection, demand ==
    rebuild from the solution, wirelength and via-count invariants, conflict-free batches, and the
    definitional O(n^2) Elmore on a sample of nets recomputed one by one from the GPU solution."""
    d = synth.make_config(5)
    got = run_gpu(la, d)
    st = got["stats"]
    assert int(got["wire_dem"].sum()) == st["wirelength"] == d.unit_edges_total()
    assert int(got["via_dem"].sum()) == int((got["vias"][:, 3] - got["vias"][:, 2]).sum())
    rng = np.random.default_rng(0)
    for net in rng.choice(d.n_nets, 300, replace=False):
        pins, segs = rc.net_pins(d, net), rc.net_segs(d, net)
        nodes = rc.build_tree(pins, segs)
        w = got["wires"][got["wire_ptr"][net]:got["wire_ptr"][net + 1]]
        v = got["vias"][got["via_ptr"][net]:got["via_ptr"][net + 1]]
        assert rc.unit_edges([tuple(int(t) for t in x[:4]) for x in w]) == rc.unit_edges(segs)
        lay = rc.solution_layers(nodes, w)
        vmap = {(int(a[0]), int(a[1])): (int(a[2]), int(a[3])) for a in v}
        spans = [vmap.get((nd["x"], nd["y"]), (pins[0][2] if i == 0 else lay[i],) * 2) for i, nd in enumerate(nodes)]
        delays, ncap, nrc = rc.elmore_definitional(d, pins, nodes, lay, spans)
        p0 = int(d.pin_ptr[net])
        np.testing.assert_allclose(got["sink_delay"][p0:p0 + len(pins)], delays, rtol=1e-9, atol=1e-15)
        np.testing.assert_allclose([got["net_cap"][net], got["net_rc"][net]], [ncap, nrc], rtol=1e-9)


@pytest.mark.parametrize("cfg,n", [(1, None), (2, None)])
def test_evaluator_parity(la, cfg, n):
    """la_eval_overflow (NEXT #3) vs oracle.evaluate on the oracle's own solution and demand:
    integers (Eq. (2) totals, wirelength per layer, via cuts) exact; the Eq. (3) totals and
    wire C within 1e-12 of the correctly rounded sums (the library bins elements exactly and
    sums count * ofw * e^{s(d-c)} per layer: a few roundings per bin, DESIGN §5 k_eval)."""
    d = synth.make_config(cfg, n_nets=n)
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.assign_all()
    ev = A.eval_overflow()
    assert A.eval_overflow() == ev          # second call: cached initial-state sums
    A.close()
    ref = oracle.run(d)
    ex = oracle.evaluate(d, ref["wire_dem"], ref["via_dem"], ref["wires"], ref["vias"])
    assert ev["out_of_domain"] == 0
    for k in ("legacy_wire", "legacy_via", "via_cuts"):
        assert ev[k] == ex[k], k
    assert ev["wirelength"] == ex["wirelength"]
    for k in ("tof_wire", "tof_via", "wire_cap"):
        assert abs(ev[k] - ex[k]) <= 1e-12 * abs(ex[k]), (k, ev[k], ex[k])


def test_evaluator_clamped_domain(la):
    """la_eval_overflow when d - c leaves the table domain [δ_lo, δ_hi] (R20): the per-layer
    wirelength and via cuts can then no longer come from the plane histograms' Σ(d - c) (clamped
    bins), so the library counts them from the nodes; they must still equal the oracle's, and
    repeated calls (the initial-state sums are cached) must agree."""
    d = synth.make_config(1)
    d.delta_lo, d.delta_hi = -3, 1
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.assign_all()
    ev = A.eval_overflow()
    ev2 = A.eval_overflow()
    A.close()
    ref = oracle.run(d)
    ex = oracle.evaluate(d, ref["wire_dem"], ref["via_dem"], ref["wires"], ref["vias"])
    assert ev["out_of_domain"] > 0
    for k in ("legacy_wire", "legacy_via", "via_cuts"):
        assert ev[k] == ex[k] == ev2[k], k
    assert ev["wirelength"] == ex["wirelength"] == ev2["wirelength"]


@pytest.mark.parametrize("variant", ["no_lookahead", "no_timing", "heavy_timing"])
def test_ablation_variants(la, variant):
    """the 'w/o ahead' ablation (Table IV: ur = 0, i.e.
    r_avg = 0 and r_drv = 0, so cost' = cost) and the W_D sweep ends are input switches of the
    same hot path: parity with the oracle under each."""
    d = synth.generate(n_nets=20_000, X=96, Y=96, L=10, seed=97, pin_max=63, rdrv_mode=1)
    if variant == "no_lookahead":
        d.r_avg = 0.0
        d.r_drv = np.zeros_like(d.r_drv)
    elif variant == "no_timing":
        d.W_D = 0.0
    else:
        d.W_D = 1e4
    assert_parity(run_gpu(la, d), oracle.run(d), bitwise_fp=True)


@pytest.mark.parametrize("kind", ["random20", "all_in_one", "conflict_free", "size_cap"])
def test_snapshot_batches_parity(la, kind):
    """Paper-style snapshot batches (NEXT #1, la_set_snapshot_batches): GPU == oracle snapshot
    mode, bit for bit, for arbitrary partitions -- including one batch of everything (every
    net reads the initial demand) and the conflict-free batches (== sequential)."""
    d = synth.make_config(2, n_nets=30_000)
    rng = np.random.default_rng(5)
    rank = np.argsort(np.argsort(d.order_key, kind="stable"), kind="stable")
    if kind == "random20":
        sb = rng.integers(0, 20, d.n_nets).astype(np.int32)
    elif kind == "all_in_one":
        sb = np.zeros(d.n_nets, np.int32)
    elif kind == "conflict_free":
        sb = oracle.run(d, solution=False, grids=False, timing=False)["batch_of"]
    else:
        sb = (rank // 4096).astype(np.int32)            # priority order cut into batches of 4096
    A = la.LayerAssigner(d, device=0)
    nb = A.load(snapshot_batches=sb)
    assert nb == int(sb.max()) + 1
    got = A.run()
    A.close()
    ref = oracle.run(d, snap_batch=sb)
    ref["batch_of"] = sb
    assert_parity(got, ref, bitwise_fp=True)
    if kind == "conflict_free":
        seq = oracle.run(d)
        assert np.array_equal(seq["wires"], ref["wires"]) and np.array_equal(seq["wire_dem"], ref["wire_dem"])


@pytest.mark.parametrize("world,cfg,n", [(2, 2, None), (3, 4, 60_000), (4, 2, 40_000), (8, 3, 60_000)])
def test_sharded_path_host_transport(la, world, cfg, n):
    """The multi-GPU data path on one GPU: `world` contexts, one per
    rank, each assigns only its shard of every batch (la_shard_range over the batch's big and
    small nets), the packed decisions and net costs of all ranks are summed on the host (the
    NCCL all-reduce's job) and handed back, every rank commits the whole batch (k_commit).
    Every replica must end bit-identical to the others and to the oracle."""
    d = synth.make_config(cfg, n_nets=n)
    ranks = [la.LayerAssigner(d, device=0, rank=r, world=world) for r in range(world)]
    nbs = {A.load() for A in ranks}
    assert len(nbs) == 1
    nb = nbs.pop()
    for k in range(nb):
        for A in ranks:
            A.assign_batch(k)
        parts = [la.la_get_decisions(A.ctx, k) for A in ranks]
        dec = np.sum([p[0] for p in parts], axis=0, dtype=np.uint64).astype(np.uint32)
        cost = np.sum([p[1] for p in parts], axis=0)
        owned = np.sum([(p[0] >> 24) & 1 for p in parts], axis=0)
        assert np.all(owned == 1), "every node of the batch decided by exactly one rank"
        for A in ranks:
            la.la_put_decisions(A.ctx, k, dec, cost)
            A.commit_demand(k)
    # la_eval_timing is sharded too: each rank evaluates the nets it assigned (others 0); the
    # caller's element-wise sum is the all-gather (one nonzero contributor per value)
    timing = [A.eval_timing() for A in ranks]
    for k in ("sink_delay", "net_cap", "net_rc"):
        nz = np.sum([t[k] != 0 for t in timing], axis=0)
        assert np.all(nz <= 1), f"{k}: a value evaluated by two ranks"
    summed = {k: np.sum([t[k] for t in timing], axis=0) for k in ("sink_delay", "net_cap", "net_rc")}
    outs = []
    for A in ranks:
        out = dict(summed)
        out.update(A.solution())
        wd, vd = A.demand()
        out.update(wire_dem=wd, via_dem=vd, batch_of=A.batches())
        outs.append(out)
        A.close()
    ref = oracle.run(d)
    for out in outs:
        assert_parity(out, ref, bitwise_fp=True)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,sched", [(2, None, "batch"), (1, None, "auto"), (3, 150_000, "batch")])
def test_nccl_reconcile_one_gpu(la, cfg, n, sched):
    """The NCCL branch of la_commit_demand and la_eval_timing on one GPU: a world-1 context with an
    ncclUniqueId packs its decisions, all-reduces them (and the net costs, then the timing outputs)
    through a real NCCL communicator and unpacks them; the result must equal the oracle bit for bit
    and the reconcile must have run (profile)."""
    d = synth.make_config(cfg, n_nets=n)
    A = la.LayerAssigner(d, device=0, rank=0, world=1, nccl_id=la.la_nccl_unique_id())
    A.load()
    if sched == "batch":
        A.set_schedule(la.LA_SCHED_BATCH)
    A.profiling(True)
    A.profile(reset=True)
    got = A.run()
    prof = A.profile(reset=True)
    A.close()
    assert prof["reconcile_ms"] > 0.0
    assert_parity(got, oracle.run(d), bitwise_fp=True)


def test_new_call_order_errors(la):
    """Call-order errors of the widened API: snapshot batches after la_load_nets, the host
    transport on a single-rank context, the dataflow schedule with snapshot batches."""
    d = synth.make_config(1)
    A = la.LayerAssigner(d, device=0)
    A.load()
    with pytest.raises(la.LaError) as ei:
        la.la_set_snapshot_batches(A.ctx, np.zeros(d.n_nets, np.int32))
    assert ei.value.status == la.LA_ESTATE
    A.assign_batch(0)
    with pytest.raises(la.LaError) as ei:
        la.la_get_decisions(A.ctx, 0)
    assert ei.value.status == la.LA_ESTATE
    A.close()
    B = la.LayerAssigner(d, device=0)
    B.load(snapshot_batches=np.zeros(d.n_nets, np.int32))
    with pytest.raises(la.LaError) as ei:
        B.set_schedule(la.LA_SCHED_DATAFLOW)
    assert ei.value.status == la.LA_EINVAL
    B.close()


@pytest.mark.parametrize("kind", ["permutation", "reversed", "ties", "sparse", "negative"])
def test_priority_key_shapes(la, kind):
    """Alg. 2's net order is (order_key, index) ascending (reading R43 / DESIGN §3).  la_load_nets
    takes it by direct placement (a permutation of a key range), a stable parallel counting sort
    (small key range, ties by index: 'ties' uses 150k nets so several threads split the count),
    or a comparison sort (sparse or huge ranges); every shape must give the oracle's order, batches
    and solution bit for bit."""
    n = 150_000 if kind == "ties" else 30_000
    d = synth.make_config(2, n_nets=n)
    rng = np.random.default_rng(11)
    if kind == "reversed":
        d.order_key = (d.n_nets - 1 - d.order_key).astype(np.int64) + 7
    elif kind == "ties":
        d.order_key = rng.integers(0, 300, d.n_nets).astype(np.int64)
    elif kind == "sparse":
        d.order_key = (d.order_key * 1_000_003 + rng.integers(0, 2, d.n_nets)).astype(np.int64) - (1 << 62)
    elif kind == "negative":
        d.order_key = rng.integers(-(1 << 62), 1 << 62, d.n_nets).astype(np.int64)
        d.order_key[:4] = [np.iinfo(np.int64).min, np.iinfo(np.int64).max, 0, 0]
    assert_parity(run_gpu(la, d), oracle.run(d), bitwise_fp=True)


@pytest.mark.parametrize("variant", ["0", "1"])
@pytest.mark.parametrize("cfg", [1, 2])
def test_assign_variants_bitwise(la, cfg, variant, monkeypatch):
    """k_assign is built at two register budgets (6 CTAs/SM for latency-bound launches, 7 for
    throughput-bound ones, chosen per launch); forcing either one on every launch must give the
    oracle's solution bit for bit."""
    monkeypatch.setenv("GAPLA_ASSIGN_VARIANT", variant)
    d = synth.make_config(cfg)
    assert_parity(run_gpu(la, d), oracle.run(d), bitwise_fp=True)


# --------------------------------------------------------------- full-size parity (hashes)
@pytest.mark.slow
@pytest.mark.parametrize("cfg", [4, 5])
def test_config_full_size_oracle_hashes(la, cfg):
    """Configs 4 and 5 at full size in the bench's launch configuration (LayerAssigner.run =
    la_assign_all + la_eval_timing, default schedule and variants) against the SHA-256 hashes of
    the oracle's outputs (tests/golden/oracle_hashes_cfg{4,5}.json, written by
    tools/oracle_golden.py from oracle/ only).  Every array bit for bit:
    solution, both demand grids, batch ids, and the bit patterns of f_root, sink delays, net
    caps and net RC sums.  A mismatch names the first differing 1/64 slice of each array."""
    from helpers import compare_hashes, golden, output_hashes
    want = golden(f"oracle_hashes_cfg{cfg}.json")
    d = synth.make_config(cfg)
    assert d.n_nets == want["n_nets"] and d.n_pins == want["n_pins"]
    got = run_gpu(la, d)
    assert got["n_batches"] == want["n_batches"]
    bad = compare_hashes(output_hashes(got), want["hashes"])
    assert not bad, "; ".join(bad)
