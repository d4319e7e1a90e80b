"""C-ABI library: loads, exports every symbol include/la.h declares, host-side validation
(no compute calls; runs without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

from gen import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def la():
    import __graft_entry__ as ge
    ge.build()
    from paper_2507_13375_b200 import la as mod
    return mod


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "la.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(la_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(la):
    syms = declared_symbols()
    assert "la_init_grid" in syms and "la_assign_batch" in syms and len(syms) >= 15
    lib = ctypes.CDLL(la.SO_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(la.EXPORTS) == set(syms)


def test_library_built_for_sm100a(la):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", la.SO_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _desc(la, d, **over):
    A = la.LayerAssigner.__new__(la.LayerAssigner)
    A._keep = []
    # build the descriptor exactly as LayerAssigner does, without creating a context
    g = la.la_grid_desc()
    keep = A._keep

    def arr(a, dt):
        x = np.ascontiguousarray(a, dtype=dt)
        keep.append(x)
        return x

    vals = dict(X=d.X, Y=d.Y, L=d.L, r=d.r, c=d.c, vr=d.vr, ofw=d.ofw, W_D=d.W_D, delta_lo=d.delta_lo,
                delta_hi=d.delta_hi, routable=d.routable, wire_cap=d.wire_cap, world=1, rank=0)
    vals.update(over)
    g.X, g.Y, g.L = vals["X"], vals["Y"], vals["L"]
    g.dir = arr(d.dir, np.uint8).ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    g.routable = arr(vals["routable"], np.uint8).ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    for k in ("r", "c", "vr", "ofw"):
        setattr(g, k, arr(vals[k], np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    g.wire_cap = arr(vals["wire_cap"], np.int32).ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    g.via_cap = arr(d.via_cap, np.int32).ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    g.s_pos, g.s_zero = 0.5, 1.5
    g.W_D, g.W_CAP, g.W_CONG, g.W_VIA = vals["W_D"], 0.2, 1.0, 0.05
    g.r_avg, g.logit_k, g.logit_b, g.w_floor = float("nan"), 10.0, 0.3, 0.05
    g.delta_lo, g.delta_hi = vals["delta_lo"], vals["delta_hi"]
    g.world, g.rank = vals["world"], vals["rank"]
    return g, keep


@pytest.mark.parametrize("over,msg", [
    (dict(L=1), "L must be"),
    (dict(L=17), "L must be"),
    (dict(X=1), "X, Y"),
    (dict(X=40000, Y=40000), "grid too large"),
    (dict(r=-np.ones(6)), "negative"),
    (dict(W_D=-1.0), "negative"),
    (dict(delta_lo=5, delta_hi=4), "delta_lo"),
    (dict(routable=np.array([1, 0, 1, 0, 1, 0])), "routable"),
    (dict(world=0, rank=0), "rank"),
    (dict(world=2, rank=3), "rank"),
])
def test_init_grid_validation(la, over, msg):
    """Descriptor errors are LA_EINVAL before any device work (include/la.h la_init_grid)."""
    d = synth.empty_design(8, 8, 6)
    g, keep = _desc(la, d, **over)
    with pytest.raises(la.LaError, match=msg) as ei:
        la.la_init_grid(g)
    assert ei.value.status == la.LA_EINVAL


def test_negative_capacity_rejected(la):
    d = synth.empty_design(8, 8, 6)
    cap = d.wire_cap.copy()
    cap[3] = -1
    g, keep = _desc(la, d, wire_cap=cap)
    with pytest.raises(la.LaError, match="negative wire capacity"):
        la.la_init_grid(g)


def test_null_arguments(la):
    with pytest.raises(la.LaError) as ei:
        la._check(la._lib.la_load_nets(None, None, None))
    assert ei.value.status == la.LA_EINVAL
    with pytest.raises(la.LaError):
        la._check(la._lib.la_assign_batch(None, 0))


@pytest.mark.parametrize("n,world", [(0, 1), (1, 2), (7, 3), (100, 8), (5, 8)])
def test_shard_range_partitions(la, n, world):
    """la_shard_range: contiguous, disjoint, covering, balanced within 1."""
    spans = [la.la_shard_range(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, e) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_paper_batches_needs_a_context(la):
    """la_paper_batches runs on a context's GPU (include/la.h): without one it reports
    LA_EINVAL before touching its inputs (no device needed for this check).  The argument
    checks and the GPU == oracle parity are tests/test_pre_timing.py (-m gpu)."""
    d = synth.make_config(1)
    crit = np.zeros(d.n_nets, np.int32)
    with pytest.raises(la.LaError, match="context") as ei:
        la.la_paper_batches(None, d, crit)
    assert ei.value.status == la.LA_EINVAL
