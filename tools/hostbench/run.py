"""Time the host tree builder of la_load_nets on this machine (no GPU): python tools/hostbench/run.py --config 5"""
import argparse, ctypes, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--n-nets", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
import numpy as np
from paper_2507_13375_b200 import build as B
so = os.path.join(ROOT, "tools", "hostbench", "libbuildbench.so")
src = os.path.join(ROOT, "tools", "hostbench", "build_bench.cpp")
deps = [src, os.path.join(ROOT, "paper_2507_13375_b200", "csrc", "la_host.cpp"), os.path.join(ROOT, "paper_2507_13375_b200", "csrc", "la_internal.h")]
if not os.path.exists(so) or any(os.path.getmtime(d) > os.path.getmtime(so) for d in deps):
    nccl = B.nccl_dir()
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-pthread", "-g",
                           "-I/usr/local/cuda/include", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
                           src, "-o", so, "-L/usr/local/cuda/lib64", "-lcudart", "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2"])
ctypes.CDLL(B.SO, mode=ctypes.RTLD_GLOBAL)   # the launch_* symbols la_host.cpp references
lib = ctypes.CDLL(so)
from gen import synth
from paper_2507_13375_b200 import la
t = time.perf_counter()
d = synth.make_config(args.config, n_nets=args.n_nets) if args.n_nets else synth.make_config(args.config)
print(f"generate {time.perf_counter() - t:.1f} s, {d.n_nets} nets", flush=True)
keep = []
nd = la.net_desc_of(d, keep)
dirv = np.ascontiguousarray(d.dir, np.uint8); rout = np.ascontiguousarray(d.routable, np.uint8)
f = lib.gapla_bench_build
f.restype = ctypes.c_double
out = (ctypes.c_int64 * 4)()
ravg = d.r_avg
if ravg != ravg:
    acc, cnt = 0.0, 0
    for l in range(d.L):
        if d.routable[l]:
            acc += float(d.r[l]); cnt += 1
    ravg = acc / cnt
for r in range(args.reps):
    s = f(ctypes.byref(nd), d.X, d.Y, d.L, dirv.ctypes.data_as(ctypes.c_void_p), rout.ctypes.data_as(ctypes.c_void_p),
          ctypes.c_double(ravg), ctypes.c_double(d.W_D), ctypes.c_double(d.logit_k),
          ctypes.c_double(d.logit_b), ctypes.c_double(d.w_floor), args.threads, out)
    print(f"rep {r}: build {s*1000:.1f} ms  nodes {out[0]} sinks {out[1]} fp {out[2]} hash {out[3] & 0xffffffffffffffff:016x}", flush=True)
