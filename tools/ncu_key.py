"""Key metrics of the (single) kernel in an ncu report. usage: python tools/ncu_key.py report.ncu-rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, v = r[0], r[2]
for w in ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__grid_size", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"] + \
         [x for x in h if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio")]:
    if w in h:
        val = v[h.index(w)]
        try:
            if w.startswith("smsp__average_warps_issue_stalled_") and float(val) < 0.2:
                continue
        except ValueError:
            pass
        print(f"{w.replace('smsp__average_warps_issue_stalled_', 'stall_').replace('_per_issue_active.ratio', '')}: {val}")
