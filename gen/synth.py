"""Seeded synthetic ISPD-2025-shaped designs (input generation only).

This module holds NONE of the layer-assignment method's arithmetic.  It is the
stand-in for the 2D global router and benchmark files the paper consumes
(§II-B l.132: "a GCell grid graph with GCell edge capacity, a netlist
and an optimized 2D global routing solution") and is the one module that both
the oracle (``oracle/``) and the CUDA library read their inputs from.

Recipe: SURVEY.md §8(d) d.2, restated in DESIGN.md "Input recipe".  The heavy
lifting (per-net pins and greedy Prim-style Steiner routes, capacities) is in
``gen/synth.c`` for speed at 12M nets; this file adds the per-layer technology
and weight constants and packages everything as numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


class _Params(ctypes.Structure):
    _fields_ = [("n_nets", ctypes.c_int64), ("X", ctypes.c_int32), ("Y", ctypes.c_int32),
                ("L", ctypes.c_int32), ("seed", ctypes.c_uint64), ("pin_max", ctypes.c_int32),
                ("hf_frac", ctypes.c_double), ("rdrv_mode", ctypes.c_int32), ("wns", ctypes.c_double),
                ("p_neg", ctypes.c_double)]


class _Out(ctypes.Structure):
    _fields_ = [("n_nets", ctypes.c_int64), ("n_pins", ctypes.c_int64), ("n_segs", ctypes.c_int64),
                ("pin_ptr", ctypes.POINTER(ctypes.c_int64)),
                ("pin_x", ctypes.POINTER(ctypes.c_int32)), ("pin_y", ctypes.POINTER(ctypes.c_int32)),
                ("pin_layer", ctypes.POINTER(ctypes.c_uint8)),
                ("pin_cap", ctypes.POINTER(ctypes.c_double)), ("pin_slack", ctypes.POINTER(ctypes.c_double)),
                ("seg_ptr", ctypes.POINTER(ctypes.c_int64)), ("seg_xy", ctypes.POINTER(ctypes.c_int32)),
                ("r_drv", ctypes.POINTER(ctypes.c_double)), ("order_key", ctypes.POINTER(ctypes.c_int64)),
                ("n_wire", ctypes.c_int64), ("n_via", ctypes.c_int64),
                ("wire_cap", ctypes.POINTER(ctypes.c_int32)), ("via_cap", ctypes.POINTER(ctypes.c_int32))]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.synth_generate.argtypes = [ctypes.POINTER(_Params), ctypes.POINTER(_Out)]
        _lib.synth_generate.restype = ctypes.c_int
        _lib.synth_free.argtypes = [ctypes.POINTER(_Out)]
    return _lib


def _np(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


@dataclass
class Design:
    """One layer-assignment instance: grid + technology + weights + nets + 2D routes.

    Grid arrays use the API layout of include/la.h: wire capacity per layer l
    (layer 0 first), edges keyed by their lower endpoint, row-major [y][x];
    H layers have (X-1)*Y edges, V layers X*(Y-1).  Via-cut capacity is
    [(L-1)][Y][X].  Units: kOhm, fF, ps (kOhm*fF = ps), GCell pitch = 1.
    """
    name: str
    X: int
    Y: int
    L: int
    dir: np.ndarray          # [L] u8, 0 = H, 1 = V
    routable: np.ndarray     # [L] u8
    r: np.ndarray            # [L] kOhm per GCell
    c: np.ndarray            # [L] fF per GCell
    vr: np.ndarray           # [L-1] kOhm per via cut
    ofw: np.ndarray          # [L] Eq. (3) overflow weight
    wire_cap: np.ndarray     # int32
    via_cap: np.ndarray      # int32
    wire_dem0: np.ndarray | None = None
    via_dem0: np.ndarray | None = None
    s_pos: float = 0.5
    s_zero: float = 1.5
    W_D: float = 100.0
    W_CAP: float = 0.2
    W_CONG: float = 1.0
    W_VIA: float = 0.05
    r_avg: float = float("nan")
    logit_k: float = 10.0
    logit_b: float = 0.3
    w_floor: float = 0.05
    delta_lo: int = -1024
    delta_hi: int = 256
    # nets
    pin_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    pin_x: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    pin_y: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    pin_layer: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    pin_cap: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    pin_slack: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    seg_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    seg_xy: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.int32))
    r_drv: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    order_key: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    wns: float = -500.0

    @property
    def n_nets(self) -> int:
        return int(self.pin_ptr.shape[0] - 1)

    @property
    def n_pins(self) -> int:
        return int(self.pin_ptr[-1])

    def wire_layer_sizes(self):
        return [(self.X - 1) * self.Y if self.dir[l] == 0 else self.X * (self.Y - 1) for l in range(self.L)]

    def unit_edges_total(self) -> int:
        s = self.seg_xy.astype(np.int64)
        return int((np.abs(s[:, 2] - s[:, 0]) + np.abs(s[:, 3] - s[:, 1])).sum())


def layer_tech(L: int):
    """Per-layer technology of SURVEY §8(d) d.2 (lower layers: larger R and C,
    PAPER.md §I l.53; GCell-edge R < 0.01 kOhm, §III-D l.439)."""
    l = np.arange(L, dtype=np.float64)
    r = 0.008 * 0.7 ** l
    c = 0.20 * 0.95 ** l
    vr = 0.010 * 0.85 ** np.arange(L - 1, dtype=np.float64)
    ofw = np.where(np.arange(L) < 2, 2.0, 1.0)
    d = (np.arange(L) % 2).astype(np.uint8)       # layer 0 = H, alternating (R35)
    routable = np.ones(L, np.uint8)
    return d, routable, r, c, vr, ofw


# BASELINE.json configs.
CONFIGS = {
    1: dict(name="cfg1_tiny_1k_32x32_L6", n_nets=1000, X=32, Y=32, L=6, seed=101, pin_max=8, hf_frac=0.0, rdrv_mode=0),
    2: dict(name="cfg2_100k_256x256_L10", n_nets=100_000, X=256, Y=256, L=10, seed=102, pin_max=63, hf_frac=0.0, rdrv_mode=0),
    3: dict(name="cfg3_1M_1024x1024_L10", n_nets=1_000_000, X=1024, Y=1024, L=10, seed=103, pin_max=63, hf_frac=0.0, rdrv_mode=1),
    4: dict(name="cfg4_4M_2048x2048_L13_hf", n_nets=4_000_000, X=2048, Y=2048, L=13, seed=104, pin_max=63, hf_frac=0.001, rdrv_mode=1),
    5: dict(name="cfg5_12M_4096x4096_L13", n_nets=12_000_000, X=4096, Y=4096, L=13, seed=105, pin_max=63, hf_frac=0.0, rdrv_mode=1),
}


def generate(n_nets: int, X: int, Y: int, L: int, seed: int, pin_max: int = 63, hf_frac: float = 0.0,
             rdrv_mode: int = 0, wns: float = -500.0, p_neg: float = 0.2, name: str = "custom") -> Design:
    lib = _load()
    p = _Params(n_nets, X, Y, L, seed, pin_max, hf_frac, rdrv_mode, wns, p_neg)
    o = _Out()
    rc = lib.synth_generate(ctypes.byref(p), ctypes.byref(o))
    if rc != 0:
        raise ValueError("synth_generate failed")
    try:
        N, NP, NS = o.n_nets, o.n_pins, o.n_segs
        dsg_dir, routable, r, c, vr, ofw = layer_tech(L)
        d = Design(
            name=name, X=X, Y=Y, L=L, dir=dsg_dir, routable=routable, r=r, c=c, vr=vr, ofw=ofw,
            wire_cap=_np(o.wire_cap, o.n_wire, np.int32), via_cap=_np(o.via_cap, o.n_via, np.int32),
            pin_ptr=_np(o.pin_ptr, N + 1, np.int64), pin_x=_np(o.pin_x, NP, np.int32),
            pin_y=_np(o.pin_y, NP, np.int32), pin_layer=_np(o.pin_layer, NP, np.uint8),
            pin_cap=_np(o.pin_cap, NP, np.float64), pin_slack=_np(o.pin_slack, NP, np.float64),
            seg_ptr=_np(o.seg_ptr, N + 1, np.int64),
            seg_xy=_np(o.seg_xy, 4 * NS, np.int32).reshape(NS, 4),
            r_drv=_np(o.r_drv, N, np.float64), order_key=_np(o.order_key, N, np.int64), wns=wns)
    finally:
        lib.synth_free(ctypes.byref(o))
    return d


def make_config(k: int, n_nets: int | None = None) -> Design:
    """Config k of BASELINE.json (1-based).  ``n_nets`` overrides the net count
    (same grid / layers / seed) for bounded samples."""
    cfg = dict(CONFIGS[k])
    if n_nets is not None:
        cfg["n_nets"] = int(n_nets)
        cfg["name"] = cfg["name"] + f"_n{n_nets}"
    return generate(**cfg)


def empty_design(X: int, Y: int, L: int, cap_wire: int = 10, cap_via: int = 16, name: str = "hand") -> Design:
    """A grid with uniform capacities and no nets; tests add nets by hand."""
    dsg_dir, routable, r, c, vr, ofw = layer_tech(L)
    n_wire = sum((X - 1) * Y if dsg_dir[l] == 0 else X * (Y - 1) for l in range(L))
    return Design(name=name, X=X, Y=Y, L=L, dir=dsg_dir, routable=routable, r=r, c=c, vr=vr, ofw=ofw,
                  wire_cap=np.full(n_wire, cap_wire, np.int32),
                  via_cap=np.full((L - 1) * X * Y, cap_via, np.int32))


def with_nets(d: Design, nets) -> Design:
    """Attach hand-made nets.  ``nets`` is a list of dicts with keys
    pins=[(x, y, layer, cap, slack), ...] (pin 0 = driver), segs=[(x1,y1,x2,y2), ...],
    optional r_drv (default 0) and order_key (default: list position)."""
    pp, ss = [0], [0]
    px, py, pl, pc, ps, sxy, rd, ok = [], [], [], [], [], [], [], []
    for i, n in enumerate(nets):
        for (x, y, l, cap, sl) in n["pins"]:
            px.append(x); py.append(y); pl.append(l); pc.append(cap); ps.append(sl)
        for s in n["segs"]:
            sxy.append(list(s))
        pp.append(len(px)); ss.append(len(sxy))
        rd.append(n.get("r_drv", 0.0)); ok.append(n.get("order_key", i))
    d.pin_ptr = np.array(pp, np.int64)
    d.pin_x = np.array(px, np.int32); d.pin_y = np.array(py, np.int32)
    d.pin_layer = np.array(pl, np.uint8); d.pin_cap = np.array(pc, np.float64)
    d.pin_slack = np.array(ps, np.float64)
    d.seg_ptr = np.array(ss, np.int64)
    d.seg_xy = np.array(sxy, np.int32).reshape(-1, 4)
    d.r_drv = np.array(rd, np.float64); d.order_key = np.array(ok, np.int64)
    return d


def criticality(d: Design, seed: int = 7) -> np.ndarray:
    """Synthetic net criticality (number of critical paths through a net), the STA
    output Alg. 1 line 2 would give: nets whose worst sink slack is below 0.7 WNS get a count
    that grows as the slack approaches WNS (a few up to ~12), the rest 0-1.  Input
    generation only (no method arithmetic)."""
    rng = np.random.default_rng(seed)
    n = d.n_nets
    slack = np.full(n, np.inf)
    sinks = np.ones(d.n_pins, bool)
    sinks[d.pin_ptr[:-1]] = False
    idx = np.repeat(np.arange(n), np.diff(d.pin_ptr))
    np.minimum.at(slack, idx[sinks], d.pin_slack[sinks])
    ratio = np.where(np.isfinite(slack), slack / d.wns, 0.0)
    base = np.where(ratio > 0.7, 12.0 * (ratio - 0.7) / 0.3, 0.0)
    return np.floor(base * rng.uniform(0.5, 1.5, n) + rng.uniform(0, 1.5, n)).astype(np.int32)
