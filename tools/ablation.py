"""Look-ahead ablation and weight sweep (PAPER Table IV "w/o ahead"
l.633-637, Fig. 11 l.672-684), on the GPU hot path.

    python tools/ablation.py [--config 3] [--n-nets N]

For each variant of the same synthetic design (full method; ur = 0 "w/o ahead"; W_D and
W_CAP sweeps) it runs la_assign_all + la_eval_timing + la_eval_overflow and prints one JSON
line with proxies of the paper's metrics that need no STA (OpenROAD is out of scope):
criticality-weighted sink delay sum sum_q w_q d_q and the largest delay among the 20%
most critical sinks (timing), total net capacitance (power, R27), Eq. (3) total overflow
(congestion), via cuts and the k_assign time.
"""
import argparse
import copy
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n-nets", type=int, default=None)
args = ap.parse_args()
from gen import synth
from paper_2507_13375_b200 import la

base = synth.make_config(args.config, n_nets=args.n_nets)
# pin criticality weights (Eq. (4), reading R1) of every sink, driver slots 0
x = base.pin_slack / base.wns
w = 1.0 / (1.0 + np.exp(-base.logit_k * (x - base.logit_b)))
is_drv = np.zeros(base.n_pins, bool)
is_drv[base.pin_ptr[:-1]] = True
w[is_drv] = 0.0
crit = (~is_drv) & (base.pin_slack <= np.quantile(base.pin_slack[~is_drv], 0.2))
net_of_pin = np.repeat(np.arange(base.n_nets), np.diff(base.pin_ptr))


def variant(name, **kw):
    d = copy.copy(base)
    for k, v in kw.items():
        setattr(d, k, v)
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.profiling(True)
    A.profile(reset=True)
    A.assign_all()
    p = A.profile(reset=True)
    A.profiling(False)
    t = A.eval_timing()
    ev = A.eval_overflow()
    A.close()
    sd = t["sink_delay"]
    # with the driver resistance the net delay gains r_drv * C_total at every sink: the term the
    # look-ahead (cost' = cost + B ur) anticipates
    sdd = sd + base.r_drv[net_of_pin] * t["net_cap"][net_of_pin]
    print(json.dumps({"variant": name, "workload": d.name, "k_assign_ms": p["assign_ms"],
                      "weighted_delay_ps": float(np.dot(w, sd)), "weighted_delay_with_driver_ps": float(np.dot(w, sdd)),
                      "max_critical_delay_ps": float(sd[crit].max()),
                      "max_critical_delay_with_driver_ps": float(sdd[crit].max()),
                      "total_net_cap_fF": float(t["net_cap"].sum()), "tof_wire": ev["tof_wire"],
                      "legacy_overflow": ev["legacy_wire"], "via_cuts": ev["via_cuts"]}), flush=True)


variant("full")
variant("w/o ahead (ur = 0)", r_avg=0.0, r_drv=np.zeros_like(base.r_drv))
for wd in (0.0, 10.0, 1000.0):
    variant(f"W_D = {wd:g}", W_D=wd)
for wc in (0.0, 2.0):
    variant(f"W_CAP = {wc:g}", W_CAP=wc)
