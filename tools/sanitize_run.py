"""Small hot-path runs for compute-sanitizer (memcheck / racecheck / synccheck), SURVEY §4 T5.

Each scenario runs the library through the C ABI on a design small enough for the sanitizer's
instrumentation, and checks the result against the CPU oracle (so a run that "passes" the
sanitizer but computes garbage is still caught).  Scenarios cover both schedules, both
register variants of k_assign, the big-net (half-CTA / whole-CTA / global-slot) paths, the
snapshot-batch mode and the host-transport multi-rank path.

    python tools/sanitize_run.py [scenario ...]      (default: all)
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from gen import synth  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2507_13375_b200 import la  # noqa: E402

KEYS = ("wires", "vias", "wire_dem", "via_dem", "net_cost", "sink_delay", "net_cap", "net_rc")


def check(got, ref, what):
    for k in KEYS:
        if not np.array_equal(np.asarray(got[k]), np.asarray(ref[k])):
            raise SystemExit(f"{what}: {k} differs from the oracle")
    print(f"{what}: ok ({len(got['wires'])} wires)", flush=True)


def run(d, schedule=None, snap=None):
    A = la.LayerAssigner(d, device=0)
    A.load(snapshot_batches=snap)
    if schedule is not None:
        A.set_schedule(schedule)
    out = A.run()
    A.close()
    return out


def sc_cfg1_batch():
    d = synth.make_config(1)
    check(run(d, la.LA_SCHED_BATCH), oracle.run(d), "cfg1 batch")


def sc_cfg1_flow():
    d = synth.make_config(1)
    check(run(d, la.LA_SCHED_DATAFLOW), oracle.run(d), "cfg1 dataflow")


def sc_cfg2_small():
    d = synth.make_config(2, n_nets=6000)
    check(run(d, la.LA_SCHED_BATCH), oracle.run(d), "cfg2[6000] batch")


def sc_bignets():
    # config 4's high-fanout mix (64-256 pins): big nets on half-CTAs / whole CTAs / global slots
    d = synth.make_config(4, n_nets=4000)
    check(run(d, la.LA_SCHED_BATCH), oracle.run(d), "cfg4[4000] batch (big nets)")
    check(run(d, la.LA_SCHED_DATAFLOW), oracle.run(d), "cfg4[4000] dataflow (big nets)")


def sc_snapshot():
    d = synth.make_config(1)
    sb = np.random.default_rng(3).integers(0, 8, d.n_nets).astype(np.int32)
    check(run(d, snap=sb), oracle.run(d, snap_batch=sb), "cfg1 snapshot batches")


def sc_host_transport():
    d = synth.make_config(1)
    world = 2
    ranks = [la.LayerAssigner(d, device=0, rank=r, world=world) for r in range(world)]
    nb = [A.load() for A in ranks][0]
    for k in range(nb):
        for A in ranks:
            A.assign_batch(k)
        parts = [la.la_get_decisions(A.ctx, k) for A in ranks]
        dec = np.sum([p[0] for p in parts], axis=0, dtype=np.uint64).astype(np.uint32)
        cost = np.sum([p[1] for p in parts], axis=0)
        for A in ranks:
            la.la_put_decisions(A.ctx, k, dec, cost)
            A.commit_demand(k)
    ref = oracle.run(d)
    timing = [A.eval_timing() for A in ranks]          # each rank evaluates its own nets; the sum is the all-gather
    summed = {k: np.sum([t[k] for t in timing], axis=0) for k in ("sink_delay", "net_cap", "net_rc")}
    for A in ranks:
        out = dict(summed)
        out.update(A.solution())
        wd, vd = A.demand()
        out.update(wire_dem=wd, via_dem=vd)
        check(out, ref, f"cfg1 host transport rank {A.grid_desc.rank}")
        A.close()


def sc_nccl_one_gpu():
    d = synth.make_config(2, n_nets=6000)
    A = la.LayerAssigner(d, device=0, rank=0, world=1, nccl_id=la.la_nccl_unique_id())
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    out = A.run()
    A.close()
    check(out, oracle.run(d), "cfg2[6000] NCCL reconcile, world 1")


def sc_group_paths():
    # k_assign_g: the group path with every job size and the team path (half-CTA and whole-CTA
    # teams, group/team split at small and large node counts)
    d = synth.make_config(3, n_nets=5000)
    ref = oracle.run(d)
    for env in ({"GAPLA_GROUP_NMAX": "4"}, {"GAPLA_GROUP_NMAX": "64"}, {"GAPLA_BIG_SPLIT": "0"}, {"GAPLA_BIG_SPLIT": "1"}):
        os.environ.update(env)
        check(run(d, la.LA_SCHED_BATCH), ref, f"cfg3[5000] batch {env}")
        for k in env:
            del os.environ[k]


def sc_next2():
    """NEXT #2 on the GPU: k_pre_timing (chunks of small nets and a windowed bigger net) and the
    Alg. 1 kernels, against the oracle; plus k_elmore's local / global node-value paths (bignets)."""
    d = synth.generate(n_nets=3000, X=96, Y=96, L=10, seed=9, hf_frac=0.01, rdrv_mode=1, name="san_next2")
    A = la.LayerAssigner(d, device=0)
    A.load()
    got_d, got_c = la.la_pre_timing(A.ctx, int(d.pin_ptr[-1]), d.n_nets)
    crit = synth.criticality(d, 1)
    b, nb = la.la_paper_batches(A.ctx, d, crit, 0.7, 3, 97)
    A.close()
    ref_d, ref_c = oracle.pre_timing(d)
    if not (np.allclose(got_d, ref_d, rtol=1e-9, atol=0) and np.allclose(got_c, ref_c, rtol=1e-9, atol=0)):
        raise SystemExit("pre_timing differs from the oracle")
    rb, rnb = oracle.paper_batches(d.pin_ptr, d.pin_slack, d.seg_ptr, d.seg_xy, d.wns, crit, 0.7, 3, 97)
    if nb != rnb or not np.array_equal(b, rb):
        raise SystemExit("paper_batches differs from the oracle")
    print(f"next2: ok ({d.n_nets} nets, {nb} Alg. 1 batches)", flush=True)


SCENARIOS = {k[3:]: v for k, v in globals().items() if k.startswith("sc_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(SCENARIOS)
    for n in names:
        SCENARIOS[n]()
