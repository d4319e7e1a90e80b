"""Build the GAP-LA B200 library (libgapla.so) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
SO = os.path.join(LIBDIR, "libgapla.so")
SOURCES = ["la_host.cpp", "la_kernels.cu", "la_assign.cu", "la_batch.cu", "la_order.cu", "la_tree.cu", "la_solution.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers (nvidia/nccl from the torch wheel) not found")


def build(force: bool = False, verbose: bool = False, extra: list | None = None, out: str | None = None) -> str:
    """extra / out: tuning variants (extra nvcc flags, an alternate library name in lib/, loaded with GAPLA_SO)."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "la_internal.h"), os.path.join(CSRC, "la_device.cuh"),
                   os.path.join(ROOT, "include", "la.h")]
    so = os.path.join(LIBDIR, out) if out else SO
    if not force and os.path.exists(so) and all(os.path.getmtime(so) >= os.path.getmtime(d) for d in deps):
        return so
    os.makedirs(LIBDIR, exist_ok=True)
    nccl = nccl_dir()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
           "-Xcompiler", "-fPIC,-O2,-ffp-contract=off,-pthread", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
           *(extra or []), "-shared", "-o", so, *srcs,
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nccl, "lib")]
    subprocess.check_call(cmd)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
