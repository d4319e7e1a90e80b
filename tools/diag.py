"""Diagnostic timing of k_assign schedules (not part of the bench contract).

    python tools/diag.py --config 3 [--schedule flow|batch] [--reps 3]
Prints per-mode ms per assign_all (device events via the library profiler).
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n-nets", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

from gen import synth
from paper_2507_13375_b200 import la

d = synth.make_config(args.config, n_nets=args.n_nets)
A = la.LayerAssigner(d, device=0)
nb = A.load()
st = A.stats()
print(f"cfg{args.config}: nets {d.n_nets} nodes {st['n_nodes']} batches {nb} env "
      f"{ {k: v for k, v in os.environ.items() if k.startswith('GAPLA_')} }", flush=True)
for name, sched in (("flow", la.LA_SCHED_DATAFLOW), ("batch", la.LA_SCHED_BATCH)) if args.reps > 0 else ():
    A.set_schedule(sched)
    ts = []
    for r in range(args.reps + 1):
        A.reset()
        A.sync()
        A.profiling(True)
        A.profile(reset=True)
        A.assign_all()
        A.sync()
        p = A.profile(reset=True)
        A.profiling(False)
        if r:
            ts.append(p["assign_ms"] + p["commit_ms"])
    if ts:
        print(f"  {name:6s} assign ms: {min(ts):8.2f} (min of {args.reps})  launches {p['assign_launches']}", flush=True)
A.close()

if os.environ.get("DIAG_TRACE"):
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    for name, sched in (("flow", la.LA_SCHED_DATAFLOW), ("batch", la.LA_SCHED_BATCH)):
        A.set_schedule(sched)
        A.reset()
        la.la_set_tracing(A.ctx, True)
        A.assign_all()
        A.sync()
        la.la_set_tracing(A.ctx, False)
        t = la.la_get_trace(A.ctx, d.n_nets)
        st = A.stats()
        t0 = t[:, 0].min()
        wait = (t[:, 1] - t[:, 0]) / 1e3
        gath = (t[:, 2] - t[:, 1]) / 1e3
        comp = (t[:, 3] - t[:, 2]) / 1e3
        tot = (t[:, 3] - t[:, 0]) / 1e3
        span = (t[:, 3].max() - t0) / 1e3
        print(f"  trace {name}: span {span:.0f} us; per net us: wait p50 {np.median(wait):.1f} mean {wait.mean():.1f} "
              f"max {wait.max():.0f} | gather p50 {np.median(gath):.1f} mean {gath.mean():.1f} max {gath.max():.0f} | "
              f"dp+commit p50 {np.median(comp):.1f} mean {comp.mean():.1f} p99 {np.percentile(comp, 99):.0f} max {comp.max():.0f}",
              flush=True)
        sol = A.solution()
        nw = np.diff(sol["wire_ptr"])
        for lo, hi in ((0, 2), (2, 4), (4, 8), (8, 16), (16, 40), (40, 10000)):
            m = (nw >= lo) & (nw < hi)
            if m.any():
                print(f"    wires [{lo},{hi}): {m.sum():8d} nets  dp+commit mean {comp[m].mean():8.1f} us  "
                      f"gather {gath[m].mean():6.1f}  total {tot[m].mean():8.1f}", flush=True)
        pass
    A.close()

if os.environ.get("DIAG_BATCHMAX"):
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    A.reset()
    la.la_set_tracing(A.ctx, True)
    A.assign_all()
    A.sync()
    t = la.la_get_trace(A.ctx, d.n_nets)
    bo = A.batches()
    sol = A.solution()
    nw = np.diff(sol["wire_ptr"])
    lat = (t[:, 3] - t[:, 0]) / 1e3
    nbat = int(bo.max()) + 1
    rows = []
    for b in range(nbat):
        m = np.nonzero(bo == b)[0]
        k = m[np.argmax(lat[m])]
        bspan = (t[m, 3].max() - t[m, 0].min()) / 1e3
        rows.append((b, len(m), bspan, lat[k], nw[k]))
    rows = np.array(rows)
    print(f"  batches {nbat}: sum of batch spans {rows[:, 2].sum():.0f} us, sum of max net latency {rows[:, 3].sum():.0f} us")
    print(f"  max-latency net wires: p10 {np.percentile(rows[:, 4], 10):.0f} p50 {np.median(rows[:, 4]):.0f} "
          f"p90 {np.percentile(rows[:, 4], 90):.0f}; max latency p50 {np.median(rows[:, 3]):.0f} us")
    for r in rows[::10]:
        print(f"    batch {int(r[0]):4d} nets {int(r[1]):6d} span {r[2]:7.0f} us  slowest {r[3]:6.0f} us ({int(r[4])} wires)")
    A.close()

if os.environ.get("DIAG_PERNET"):
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    A.reset()
    la.la_set_tracing(A.ctx, True)
    A.assign_all()
    A.sync()
    t = la.la_get_trace(A.ctx, d.n_nets)
    sol = A.solution()
    nw = np.diff(sol["wire_ptr"])
    nv = np.diff(sol["via_ptr"])
    g = (t[:, 2] - t[:, 1]) / 1e3
    dp = (t[:, 3] - t[:, 2]) / 1e3
    for lo, hi in ((1, 2), (2, 3), (3, 4), (4, 6), (6, 9), (9, 13), (13, 20), (20, 30), (30, 50), (50, 80), (80, 120),
                   (120, 100000)):
        m = (nw >= lo) & (nw < hi)
        if not m.any():
            continue
        print(f"    wires [{lo:3d},{hi:3d}): {m.sum():7d} nets gather p50 {np.median(g[m]):7.1f} us  dp+commit p50 "
              f"{np.median(dp[m]):7.1f} p90 {np.percentile(dp[m], 90):7.1f} max {dp[m].max():7.1f} us", flush=True)
    A.close()

if os.environ.get("DIAG_NCU"):
    import torch
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH if os.environ["DIAG_NCU"] == "batch" else la.LA_SCHED_DATAFLOW)
    A.reset()
    A.assign_all()
    A.sync()
    A.reset()
    A.sync()
    torch.cuda.profiler.start()
    A.assign_all()
    A.sync()
    torch.cuda.profiler.stop()
    A.close()

if os.environ.get("DIAG_TAIL"):
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    A.reset()
    la.la_set_tracing(A.ctx, True)
    A.assign_all()
    A.sync()
    t = la.la_get_trace(A.ctx, d.n_nets)
    bo = A.batches()
    nbat = int(bo.max()) + 1
    span = tail = 0.0
    gaps = 0.0
    prev_end = None
    for b in range(nbat):
        m = bo == b
        s0, e = t[m, 0].min(), t[m, 3].max()
        e90 = np.percentile(t[m, 3], 90)
        span += (e - s0) / 1e3
        tail += (e - e90) / 1e3
        if prev_end is not None:
            gaps += (s0 - prev_end) / 1e3
        prev_end = e
    print(f"  batches {nbat}: sum of spans {span:.0f} us, of which after the 90th-percentile finish {tail:.0f} us; "
          f"gaps between batches {gaps:.0f} us", flush=True)
    A.close()

if os.environ.get("DIAG_PHASES"):
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    A.reset()
    la.la_set_tracing(A.ctx, True)
    A.assign_all()
    A.sync()
    t = la.la_get_trace(A.ctx, d.n_nets).astype(np.float64)
    sol = A.solution()
    nw = np.diff(sol["wire_ptr"])
    ph = {"gather": t[:, 1] - t[:, 0], "leaves": t[:, 2] - t[:, 1], "nodes": t[:, 4] - t[:, 2],
          "backtrack+commit": t[:, 3] - t[:, 4]}
    tot = t[:, 3] - t[:, 0]
    print("  mean us per net: " + "  ".join(f"{k} {v.mean() / 1e3:.2f}" for k, v in ph.items()) +
          f"  total {tot.mean() / 1e3:.2f}", flush=True)
    for lo, hi in ((0, 2), (2, 4), (4, 8), (8, 16), (16, 10000)):
        m = (nw >= lo) & (nw < hi)
        print(f"    wires [{lo},{hi}) {m.mean():.3f}: " + "  ".join(f"{k} {v[m].mean() / 1e3:.2f}" for k, v in ph.items()),
              flush=True)
    A.close()

if os.environ.get("DIAG_NODEKIND"):
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    A.reset()
    la.la_set_tracing(A.ctx, True)
    A.assign_all()
    A.sync()
    t = la.la_get_trace(A.ctx, d.n_nets).astype(np.float64)
    sol = A.solution()
    nw = np.diff(sol["wire_ptr"])
    tot = t[:, 3] - t[:, 0]
    print(f"  mean us per net: total {tot.mean() / 1e3:.2f}  one-son nodes {t[:, 1].mean() / 1e3:.2f}  "
          f"other internal nodes {t[:, 4].mean() / 1e3:.2f}", flush=True)
    for lo, hi in ((0, 2), (2, 4), (4, 8), (8, 16), (16, 10000)):
        m = (nw >= lo) & (nw < hi)
        print(f"    wires [{lo},{hi}): total {tot[m].mean() / 1e3:.2f} one-son {t[m, 1].mean() / 1e3:.2f} "
              f"other {t[m, 4].mean() / 1e3:.2f}", flush=True)
    A.close()

if os.environ.get("DIAG_TEAM"):
    # team-path nets (k_assign_g big nets): per size band, take -> gather end -> level loop end -> commit end
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    A.reset()
    la.la_set_tracing(A.ctx, True)
    A.assign_all()
    A.sync()
    t = la.la_get_trace(A.ctx, d.n_nets)
    sol = A.solution()
    nw = np.diff(sol["wire_ptr"])
    team = t[:, 1] > t[:, 2]            # team nets stamp [1] after the level loop; group nets [1] = [0]
    g = (t[:, 2] - t[:, 0]) / 1e3
    lv = (t[:, 1] - t[:, 2]) / 1e3
    tl = (t[:, 3] - t[:, 1]) / 1e3
    print(f"  team nets: {int(team.sum())} of {d.n_nets}")
    for lo, hi in ((1, 13), (13, 20), (20, 30), (30, 50), (50, 80), (80, 120), (120, 200), (200, 100000)):
        m = team & (nw >= lo) & (nw < hi)
        if m.any():
            print(f"    wires [{lo:3d},{hi:3d}): {m.sum():6d} nets gather p50 {np.median(g[m]):7.1f} us  levels p50 "
                  f"{np.median(lv[m]):7.1f} p90 {np.percentile(lv[m], 90):7.1f}  backtrack+commit p50 {np.median(tl[m]):6.1f} us",
                  flush=True)
    A.close()

if os.environ.get("DIAG_TIMELINE"):
    # per batch: when team nets and group nets are taken / finish, relative to the batch's first take
    import numpy as np
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(la.LA_SCHED_BATCH)
    A.reset()
    la.la_set_tracing(A.ctx, True)
    A.assign_all()
    A.sync()
    t = la.la_get_trace(A.ctx, d.n_nets)
    bo = A.batches()
    team = t[:, 1] > t[:, 2]
    nb = int(bo.max()) + 1
    print(f"  {'batch':>5} {'nets':>7} {'team':>6} {'span':>7} | team take p50/max  end max | group take max  end p99 max  (us)")
    for b in list(range(0, nb, max(1, nb // 16))):
        m = bo == b
        t0 = t[m, 0].min()
        tm, gm = m & team, m & ~team
        def q(x, p): return (np.percentile(x, p) - t0) / 1e3 if len(x) else float("nan")
        print(f"  {b:5d} {int(m.sum()):7d} {int(tm.sum()):6d} {(t[m, 3].max() - t0) / 1e3:7.0f} | "
              f"{q(t[tm, 0], 50):7.0f} {q(t[tm, 0], 100):7.0f} {q(t[tm, 3], 100):7.0f} | "
              f"{q(t[gm, 0], 100):7.0f} {q(t[gm, 3], 99):7.0f} {q(t[gm, 3], 100):7.0f}", flush=True)
    A.close()
