"""Instruction / sample share per code region of k_assign(_g) from an ncu report (cuda,sass view).
usage: python tools/ncu_regions.py report.ncu-rep"""
import csv, re, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
src = open("paper_2507_13375_b200/csrc/la_assign.cu").read().splitlines()
# regions = enclosing top-level function of each line of la_assign.cu
func_at = {}
cur = "?"
for i, line in enumerate(src, 1):
    m = re.match(r"^(?:template <[^>]*>\s*)?(?:__\w+__\s+)*(?:static\s+)?(?:inline\s+)?[\w:<>\*& ]+?\b(\w+)\(", line)
    if m and not line.startswith(" ") and not line.startswith("//") and "(" in line and not line.rstrip().endswith(";"):
        cur = m.group(1)
    func_at[i] = cur
rows = list(csv.reader(out.splitlines()))
hdr, fname, agg = None, "?", {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) < 10 or r[0] == "":
        continue
    try:
        ie = float(r[hdr.index("Instructions Executed")]); te = float(r[hdr.index("Thread Instructions Executed")])
        sm = float(r[hdr.index("# Samples")])
    except ValueError:
        continue
    k = func_at.get(int(r[0]), "?") if fname == "la_assign.cu" else fname
    a = agg.setdefault(k, [0.0, 0.0, 0.0]); a[0] += ie; a[1] += te; a[2] += sm
ti = sum(a[0] for a in agg.values()) or 1; ts = sum(a[2] for a in agg.values()) or 1
print(f"total warp-inst {ti:.0f}  samples {ts:.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} inst {100*a[0]/ti:5.1f}%  samples {100*a[2]/ts:5.1f}%  thr/inst {a[1]/max(a[0],1):5.1f}")
