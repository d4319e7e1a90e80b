"""Per-CUDA-line instruction / stall-sample breakdown of an ncu report (cuda,sass source view).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
hdr = None
fname = "?"
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 10 or r[0] == "":
        continue
    try:
        ie = float(r[hdr.index("Instructions Executed")])
        te = float(r[hdr.index("Thread Instructions Executed")])
        sm = float(r[hdr.index("# Samples")])
    except ValueError:
        continue
    k = (fname, int(r[0]))
    a = agg.setdefault(k, [0.0, 0.0, 0.0, r[1][:100]])
    a[0] += ie; a[1] += te; a[2] += sm
ti = sum(a[0] for a in agg.values()) or 1
ts = sum(a[2] for a in agg.values()) or 1
print(f"total warp-inst {ti:.0f}  samples {ts:.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{100*a[0]/ti:5.1f}% inst {100*a[2]/ts:5.1f}% smp thr/inst {a[1]/max(a[0],1):5.1f} {k[0]}:{k[1]:<5} {a[3]}")
