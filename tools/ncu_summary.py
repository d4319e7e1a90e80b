"""Summarise an ncu launch list (CSV) of one bench step into profiles/ (DESIGN §8).

    python tools/ncu_summary.py gpurun_out/launches_cfg5.csv cfg5_12M_4096x4096_L13 profiles/r01_...json

Reads per-launch gpu__time_duration.sum and (when present) dram__bytes_read.sum /
dram__bytes_write.sum, groups by kernel, and writes per-kernel launch counts, total and
mean device time, each kernel's share of the summed kernel time, and dram bytes per
launch.  Also writes profiles/ncu_k_assign_summary.json, which bench.py reads for the
roofline "traffic" field when its workload matches.
"""
import csv
import json
import os
import sys
from collections import defaultdict

src, workload, out = sys.argv[1], sys.argv[2], sys.argv[3]
full = sys.argv[4] if len(sys.argv) > 4 else None     # optional ncu --set full report of one k_assign launch
rows = []
with open(src) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    rows.append(r)
per = defaultdict(lambda: defaultdict(float))
launches = defaultdict(set)
for r in rows:
    k = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]   # k_assign<6> / <7>: one kernel
    launches[k].add(r["ID"])
    unit = r.get("Metric Unit", "")
    v = float(r["Metric Value"].replace(",", ""))
    name = r["Metric Name"]
    if name == "gpu__time_duration.sum":
        v = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        per[k]["ms"] += v
    elif name.startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[k]["dram_bytes"] += v * scale
total_ms = sum(p["ms"] for p in per.values())
summ = {"source": os.path.basename(src), "workload": workload, "kernels": {}}
for k, p in sorted(per.items(), key=lambda kv: -kv[1]["ms"]):
    n = len(launches[k])
    summ["kernels"][k] = {"launches": n, "ms_total": p["ms"], "ms_mean": p["ms"] / n, "share": p["ms"] / total_ms,
                          "dram_bytes_total": p.get("dram_bytes"),
                          "dram_bytes_per_launch": (p["dram_bytes"] / n) if "dram_bytes" in p else None}
with open(out, "w") as f:
    json.dump(summ, f, indent=1)
ka = summ["kernels"].get("k_assign_g") or summ["kernels"].get("k_assign")
if ka and ka["dram_bytes_per_launch"] is not None:
    j = {"workload": workload, "file": os.path.basename(out),
         "dram_bytes_per_launch": ka["dram_bytes_per_launch"], "launches": ka["launches"],
         "note": "ncu serialised cold-cache launches of one bench step; mean over the step's launches"}
    if full:
        import subprocess
        raw = subprocess.run(["ncu", "-i", full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        h, v = rr[0], rr[2]
        get = lambda m: float(v[h.index(m)]) / 100.0 if m in h else None
        j["fp64_pipe_active_frac"] = get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        j["issue_active_frac"] = get("smsp__issue_active.avg.pct_of_peak_sustained_active")
        j["fp64_source"] = os.path.basename(full) + " (ncu --set full, one mid-step launch)"
    with open(os.path.join(os.path.dirname(out), "ncu_k_assign_summary.json"), "w") as f:
        json.dump(j, f, indent=1)
print(json.dumps(summ, indent=1))
