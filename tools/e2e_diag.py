"""Phase times of the e2e path (la_init_grid, la_load_nets phases, assign, Elmore, solution).

    GAPLA_VERBOSE=1 python tools/e2e_diag.py --config 5
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
args = ap.parse_args()
from gen import synth
from paper_2507_13375_b200 import la

t = time.perf_counter()
d = synth.make_config(args.config)
print(f"generate {time.perf_counter() - t:.2f} s", flush=True)
for rep in range(2):
    T = {}
    t = time.perf_counter()
    A = la.LayerAssigner(d, device=0)
    A.sync()
    T["init_grid"] = time.perf_counter() - t
    t = time.perf_counter()
    A.load()
    T["load_nets"] = time.perf_counter() - t
    t = time.perf_counter()
    A.assign_all()
    A.sync()
    T["assign_all"] = time.perf_counter() - t
    t = time.perf_counter()
    A.eval_timing()
    T["eval_timing"] = time.perf_counter() - t
    t = time.perf_counter()
    A.solution()
    T["solution"] = time.perf_counter() - t
    A.close()
    print(f"rep {rep}: " + "  ".join(f"{k} {v:.3f}s" for k, v in T.items()) + f"  total {sum(T.values()):.2f}s",
          flush=True)
