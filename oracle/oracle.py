"""ctypes front end of the fp64 CPU oracle (oracle/la_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2507_13375_b200/) never imports this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "la_oracle.cpp")

P = ctypes.POINTER
c_i32, c_i64, c_u8, c_f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint8, ctypes.c_double


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-fopenmp", "-shared", "-fPIC",
                               "-o", _SO, _SRC])
    return _SO


class OGrid(ctypes.Structure):
    _fields_ = [("X", c_i32), ("Y", c_i32), ("L", c_i32),
                ("dir", P(c_u8)), ("routable", P(c_u8)), ("r", P(c_f64)), ("c", P(c_f64)),
                ("vr", P(c_f64)), ("ofw", P(c_f64)), ("s_pos", c_f64), ("s_zero", c_f64),
                ("wire_cap", P(c_i32)), ("via_cap", P(c_i32)), ("wire_dem0", P(c_i32)), ("via_dem0", P(c_i32)),
                ("W_D", c_f64), ("W_CAP", c_f64), ("W_CONG", c_f64), ("W_VIA", c_f64), ("r_avg", c_f64),
                ("logit_k", c_f64), ("logit_b", c_f64), ("w_floor", c_f64),
                ("delta_lo", c_i32), ("delta_hi", c_i32)]


class ONets(ctypes.Structure):
    _fields_ = [("n_nets", c_i64), ("pin_ptr", P(c_i64)), ("pin_x", P(c_i32)), ("pin_y", P(c_i32)),
                ("pin_layer", P(c_u8)), ("pin_cap", P(c_f64)), ("pin_slack", P(c_f64)),
                ("seg_ptr", P(c_i64)), ("seg_xy", P(c_i32)), ("r_drv", P(c_f64)), ("order_key", P(c_i64)),
                ("wns", c_f64)]


class OOut(ctypes.Structure):
    _fields_ = [("max_wires", c_i64), ("max_vias", c_i64), ("max_nets_to_run", c_i64),
                ("net_cost", P(c_f64)), ("wire_ptr", P(c_i64)), ("wires", P(c_i32)),
                ("via_ptr", P(c_i64)), ("vias", P(c_i32)), ("wire_dem", P(c_i32)), ("via_dem", P(c_i32)),
                ("sink_delay", P(c_f64)), ("net_cap", P(c_f64)), ("net_rc", P(c_f64)),
                ("batch_of", P(c_i32)), ("n_nodes", P(c_i32)), ("elapsed_s", c_f64), ("nets_run", c_i64),
                ("err", ctypes.c_char * 256), ("snap_batch", P(c_i32)), ("threads", c_i32)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_run.argtypes = [P(OGrid), P(ONets), P(OOut)]
        _lib.oracle_run.restype = ctypes.c_int
        _lib.oracle_tables.argtypes = [P(OGrid), P(c_f64), P(c_f64), P(c_f64), P(c_f64)]
        _lib.oracle_pin_weight.argtypes = [P(OGrid), c_f64, c_f64]
        _lib.oracle_pin_weight.restype = c_f64
        _lib.oracle_tree.argtypes = [P(OGrid), P(ONets), c_i64, P(c_i32), c_i32, P(c_i32), ctypes.c_char_p]
        _lib.oracle_tree.restype = ctypes.c_int
        _lib.oracle_net_dp.argtypes = [P(OGrid), P(ONets), c_i64, c_i32, P(c_i32), P(c_f64), P(c_f64), P(c_f64),
                                       P(c_f64), P(c_f64), P(c_i32), P(c_i32), P(c_i32), ctypes.c_char_p]
        _lib.oracle_net_dp.restype = ctypes.c_int
        _lib.oracle_pre_timing.argtypes = [P(OGrid), P(ONets), c_f64, c_f64, c_f64, c_f64, P(c_f64), P(c_f64),
                                           ctypes.c_char_p]
        _lib.oracle_pre_timing.restype = ctypes.c_int
    return _lib


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(P(ctype))


class OracleError(RuntimeError):
    pass


def _grid(d, keep):
    arrs = dict(dir=np.ascontiguousarray(d.dir, np.uint8), routable=np.ascontiguousarray(d.routable, np.uint8),
                r=np.ascontiguousarray(d.r, np.float64), c=np.ascontiguousarray(d.c, np.float64),
                vr=np.ascontiguousarray(d.vr, np.float64), ofw=np.ascontiguousarray(d.ofw, np.float64),
                wire_cap=np.ascontiguousarray(d.wire_cap, np.int32), via_cap=np.ascontiguousarray(d.via_cap, np.int32),
                wire_dem0=None if d.wire_dem0 is None else np.ascontiguousarray(d.wire_dem0, np.int32),
                via_dem0=None if d.via_dem0 is None else np.ascontiguousarray(d.via_dem0, np.int32))
    keep.append(arrs)
    g = OGrid(d.X, d.Y, d.L, _ptr(arrs["dir"], c_u8), _ptr(arrs["routable"], c_u8), _ptr(arrs["r"], c_f64),
              _ptr(arrs["c"], c_f64), _ptr(arrs["vr"], c_f64), _ptr(arrs["ofw"], c_f64), d.s_pos, d.s_zero,
              _ptr(arrs["wire_cap"], c_i32), _ptr(arrs["via_cap"], c_i32), _ptr(arrs["wire_dem0"], c_i32),
              _ptr(arrs["via_dem0"], c_i32), d.W_D, d.W_CAP, d.W_CONG, d.W_VIA, d.r_avg, d.logit_k, d.logit_b,
              d.w_floor, d.delta_lo, d.delta_hi)
    return g


def _nets(d, keep):
    arrs = dict(pin_ptr=np.ascontiguousarray(d.pin_ptr, np.int64), pin_x=np.ascontiguousarray(d.pin_x, np.int32),
                pin_y=np.ascontiguousarray(d.pin_y, np.int32), pin_layer=np.ascontiguousarray(d.pin_layer, np.uint8),
                pin_cap=np.ascontiguousarray(d.pin_cap, np.float64),
                pin_slack=np.ascontiguousarray(d.pin_slack, np.float64),
                seg_ptr=np.ascontiguousarray(d.seg_ptr, np.int64),
                seg_xy=np.ascontiguousarray(d.seg_xy.reshape(-1), np.int32),
                r_drv=np.ascontiguousarray(d.r_drv, np.float64), order_key=np.ascontiguousarray(d.order_key, np.int64))
    keep.append(arrs)
    return ONets(d.n_nets, _ptr(arrs["pin_ptr"], c_i64), _ptr(arrs["pin_x"], c_i32), _ptr(arrs["pin_y"], c_i32),
                 _ptr(arrs["pin_layer"], c_u8), _ptr(arrs["pin_cap"], c_f64), _ptr(arrs["pin_slack"], c_f64),
                 _ptr(arrs["seg_ptr"], c_i64), _ptr(arrs["seg_xy"], c_i32), _ptr(arrs["r_drv"], c_f64),
                 _ptr(arrs["order_key"], c_i64), d.wns)


def run(d, solution: bool = True, grids: bool = True, timing: bool = True, batches: bool = True,
        max_nets: int = 0, snap_batch=None, threads: int = 1) -> dict:
    """Sequential oracle over design ``d`` (gen.synth.Design).  Returns numpy arrays:
    net_cost, wire_ptr/wires, via_ptr/vias, wire_dem, via_dem, sink_delay, net_cap,
    net_rc, batch_of, n_nodes, elapsed_s, nets_run.  ``snap_batch`` (int32 per net):
    paper-style snapshot batches (NEXT #1, reading R31) instead of sequential commits.
    ``threads`` > 1: mode 2, the nets of each conflict-free batch on that many
    host threads (OpenMP); exact by SURVEY §8(c) c.2, so every output equals mode 1's."""
    lib = _load()
    keep = []
    g = _grid(d, keep)
    n = _nets(d, keep)
    N, NP = d.n_nets, d.n_pins
    ue = d.unit_edges_total() if d.seg_xy.size else 0
    res = dict(net_cost=np.empty(N, np.float64), n_nodes=np.zeros(N, np.int32))
    if solution:
        res.update(wire_ptr=np.zeros(N + 1, np.int64), wires=np.zeros((max(ue, 1), 5), np.int32),
                   via_ptr=np.zeros(N + 1, np.int64), vias=np.zeros((max(ue + N, 1), 4), np.int32))
    if grids:
        res.update(wire_dem=np.zeros(d.wire_cap.shape[0], np.int32), via_dem=np.zeros(d.via_cap.shape[0], np.int32))
    if timing:
        res.update(sink_delay=np.zeros(NP, np.float64), net_cap=np.zeros(N, np.float64), net_rc=np.zeros(N, np.float64))
    if batches:
        res.update(batch_of=np.full(N, -1, np.int32))
    o = OOut()
    o.max_wires = res["wires"].shape[0] if solution else 0
    o.max_vias = res["vias"].shape[0] if solution else 0
    o.max_nets_to_run = max_nets
    o.threads = int(threads)
    if snap_batch is not None:
        snap_batch = np.ascontiguousarray(snap_batch, np.int32)
        keep.append(snap_batch)
        o.snap_batch = _ptr(snap_batch, c_i32)
    for k, ct in (("net_cost", c_f64), ("wire_ptr", c_i64), ("wires", c_i32), ("via_ptr", c_i64), ("vias", c_i32),
                  ("wire_dem", c_i32), ("via_dem", c_i32), ("sink_delay", c_f64), ("net_cap", c_f64),
                  ("net_rc", c_f64), ("batch_of", c_i32), ("n_nodes", c_i32)):
        if k in res:
            setattr(o, k, _ptr(res[k], ct))
    t0 = time.perf_counter()
    rc = lib.oracle_run(ctypes.byref(g), ctypes.byref(n), ctypes.byref(o))
    res["wall_s"] = time.perf_counter() - t0
    if rc != 0:
        raise OracleError(o.err.decode())
    if solution:
        res["wires"] = res["wires"][: res["wire_ptr"][-1]]
        res["vias"] = res["vias"][: res["via_ptr"][-1]]
    res["elapsed_s"] = o.elapsed_s
    res["nets_run"] = o.nets_run
    return res


def tables(d):
    lib = _load()
    keep = []
    g = _grid(d, keep)
    VR = np.zeros(d.L * d.L, np.float64)
    n = d.delta_hi - d.delta_lo + 1
    Mp, Mz = np.zeros(n, np.float64), np.zeros(n, np.float64)
    ravg = c_f64()
    lib.oracle_tables(ctypes.byref(g), _ptr(VR, c_f64), _ptr(Mp, c_f64), _ptr(Mz, c_f64), ctypes.byref(ravg))
    return VR.reshape(d.L, d.L), Mp, Mz, ravg.value


def pin_weight(d, slack: float, wns: float) -> float:
    lib = _load()
    keep = []
    g = _grid(d, keep)
    return lib.oracle_pin_weight(ctypes.byref(g), slack, wns)


def tree(d, net: int):
    """Oracle's LA tree of one net: array [n_nodes][7] = x, y, parent, len, edir, height, npins
    (preorder ids, root = 0; edir 0=E 1=W 2=N 3=S = direction parent -> node)."""
    lib = _load()
    keep = []
    g = _grid(d, keep)
    n = _nets(d, keep)
    ue = d.unit_edges_total() + 2
    out = np.zeros((ue, 7), np.int32)
    cnt = c_i32()
    err = ctypes.create_string_buffer(256)
    rc = lib.oracle_tree(ctypes.byref(g), ctypes.byref(n), net, _ptr(out, c_i32), ue, ctypes.byref(cnt), err)
    if rc != 0:
        raise OracleError(err.value.decode())
    return out[: cnt.value]


def net_dp(d, net: int) -> dict:
    """O2/O3/O6 internals of one net on the design's initial demand (nodes in oracle_tree's
    preorder ids): ur, wd per node; f, dlc, gp (G' of the chosen span), cb, ct [node][L];
    entry [node][L][4] (son layers).  Exposed for the look-ahead pins."""
    lib = _load()
    keep = []
    g = _grid(d, keep)
    n = _nets(d, keep)
    M = d.unit_edges_total() + 2
    L = d.L
    ur, wd = np.zeros(M, np.float64), np.zeros(M, np.float64)
    f, dlc, gp = (np.zeros((M, L), np.float64) for _ in range(3))
    cb, ct = np.zeros((M, L), np.int32), np.zeros((M, L), np.int32)
    entry = np.zeros((M, L, 4), np.int32)
    cnt = c_i32()
    err = ctypes.create_string_buffer(256)
    rc = lib.oracle_net_dp(ctypes.byref(g), ctypes.byref(n), net, M, ctypes.byref(cnt), _ptr(ur, c_f64),
                           _ptr(wd, c_f64), _ptr(f, c_f64), _ptr(dlc, c_f64), _ptr(gp, c_f64), _ptr(cb, c_i32),
                           _ptr(ct, c_i32), _ptr(entry, c_i32), err)
    if rc != 0:
        raise OracleError(err.value.decode())
    k = cnt.value
    return dict(ur=ur[:k], wd=wd[:k], f=f[:k], dlc=dlc[:k], gp=gp[:k], cb=cb[:k], ct=ct[:k], entry=entry[:k])


def pre_timing(d, r_h: float = float("nan"), r_v: float = float("nan"), c_h: float = float("nan"),
               c_v: float = float("nan")):
    """Pre-assignment pi-model timing on the 2D LA trees (PAPER §III-B l.283-286, Alg. 1 inputs
    r_avg / c_avg l.240-241; reading R44): per-direction unit R / C (NaN =
    mean over that direction's routable layers), definitional Elmore (la_oracle.cpp
    pre_timing_net).  Returns (sink_delay[n_pins] ps, driver slots 0; net_cap[n_nets] fF)."""
    lib = _load()
    keep = []
    g = _grid(d, keep)
    n = _nets(d, keep)
    delay = np.zeros(int(d.pin_ptr[-1]), np.float64)
    cap = np.zeros(d.n_nets, np.float64)
    err = ctypes.create_string_buffer(256)
    rc = lib.oracle_pre_timing(ctypes.byref(g), ctypes.byref(n), r_h, r_v, c_h, c_v, _ptr(delay, c_f64),
                               _ptr(cap, c_f64), err)
    if rc != 0:
        raise OracleError(err.value.decode())
    return delay, cap


def evaluate(d, wire_dem, via_dem, wires, vias) -> dict:
    """Evaluation of a 3D solution by the plain definitions.

    PAPER §II-E Eq. (3) (l.178-182): a GCell edge on layer l with demand d and capacity c
    overflows by ofw(l) * e^{s (d - c)}, s = 0.5 (s_pos) if c > 0 else 1.5 (s_zero); tof_wire
    is the sum over every wire edge of every layer (l.169 "total overflow of all the GCell
    edges").  Eq. (2) (l.175-177): max{0, d - c}, summed: legacy_wire.  The via-cut grid of
    reading R11 is evaluated the same way with ofw of the cut's lower layer (R36).  Sums of
    floating-point terms are exactly rounded (math.fsum), so the library's binned sum is
    compared against the correctly rounded total.  wirelength[l] = unit wire edges on layer l,
    via_cuts = sum of (t - b) over via stacks, wire_cap = sum over wires of c[l] * length.
    Grids are in API layout (wire edges per layer, by lower endpoint, row-major; via cuts
    [k][y][x]); wires [n][5] (x1, y1, x2, y2, l); vias [n][4] (x, y, b, t).
    """
    import math
    wd = np.asarray(wire_dem, np.int64)
    vd = np.asarray(via_dem, np.int64)
    wc = np.asarray(d.wire_cap, np.int64)
    vc = np.asarray(d.via_cap, np.int64)
    sizes = d.wire_layer_sizes()
    offs = np.concatenate([[0], np.cumsum(sizes)])
    X, Y = d.X, d.Y

    def terms(dem, cap, ofw_l):
        delta = (dem - cap).astype(np.float64)
        s = np.where(cap > 0, d.s_pos, d.s_zero)
        return [ofw_l * math.exp(sv * dv) for sv, dv in zip(s.tolist(), delta.tolist())]

    tw, lw = [], 0
    for l in range(d.L):
        a, b = offs[l], offs[l + 1]
        tw.extend(terms(wd[a:b], wc[a:b], float(d.ofw[l])))
        lw += int(np.maximum(wd[a:b] - wc[a:b], 0).sum())
    tv, lv = [], 0
    n_cut = X * Y
    for k in range(d.L - 1):
        a, b = k * n_cut, (k + 1) * n_cut
        tv.extend(terms(vd[a:b], vc[a:b], float(d.ofw[k])))
        lv += int(np.maximum(vd[a:b] - vc[a:b], 0).sum())
    wires = np.asarray(wires, np.int64).reshape(-1, 5)
    vias = np.asarray(vias, np.int64).reshape(-1, 4)
    length = np.abs(wires[:, 2] - wires[:, 0]) + np.abs(wires[:, 3] - wires[:, 1])
    wl = [int(length[wires[:, 4] == l].sum()) for l in range(16)]
    wire_cap = math.fsum(float(d.c[l]) * float(n) for l, n in zip(wires[:, 4].tolist(), length.tolist()))
    return {"tof_wire": math.fsum(tw), "tof_via": math.fsum(tv), "legacy_wire": lw, "legacy_via": lv,
            "wirelength": wl, "via_cuts": int((vias[:, 3] - vias[:, 2]).sum()), "wire_cap": wire_cap,
            "n_wire_terms": len(tw), "n_via_terms": len(tv)}


def paper_batches(pin_ptr, pin_slack, seg_ptr, seg_xy, wns, criticality, alpha=0.7, th=3, max_batch=1 << 20):
    """Alg. 1 lines 3-10 (PAPER §III-A l.213-262) written out step by step
    in plain Python; readings R31 (GetBatches = size cap), R33 (slack bands (f_{k-1} WNS, f_k WNS]),
    R42 (f_k = 1 - 0.01 k^2: 1, 0.99, 0.96, ...), R43 (non-critical: 2D wirelength ascending).
    Returns (batch id per net, number of batches)."""
    n = len(pin_ptr) - 1
    net_slack, wl = [], []
    for j in range(n):
        sinks = [float(pin_slack[p]) for p in range(int(pin_ptr[j]) + 1, int(pin_ptr[j + 1]))]
        net_slack.append(min(sinks) if sinks else float("inf"))      # l.217: minimum over its pins
        w = 0
        for s in range(int(seg_ptr[j]), int(seg_ptr[j + 1])):
            x1, y1, x2, y2 = (int(v) for v in seg_xy[s])
            w += abs(x2 - x1) + abs(y2 - y1)
        wl.append(w)
    # line 3: Divide
    Nc = [j for j in range(n) if criticality[j] > th]
    Ns = [j for j in range(n) if criticality[j] <= th and wns < 0 and net_slack[j] < alpha * wns]
    Nn = [j for j in range(n) if j not in set(Nc) | set(Ns)]
    # line 4: PartitionAndSort(N_c): [C, C], [C/2, C), [C/4, C/2), ...
    subsets = []
    if Nc:
        C = max(criticality[j] for j in Nc)
        bands = {}
        for j in Nc:
            c = criticality[j]
            k = 0
            if c < C:
                k = 1
                while c < C / 2 ** k:
                    k += 1
            bands.setdefault(k, []).append(j)
        for k in sorted(bands):
            subsets.append(sorted(bands[k], key=lambda j: (-criticality[j], net_slack[j], j)))
    # line 5: PartitionAndSort(N_s): slack == WNS, then (f_{k-1} WNS, f_k WNS]
    if Ns:
        bands = {}
        for j in Ns:
            s = net_slack[j]
            k = 0
            if not s <= wns:
                k = 1
                while k < 10 and not s <= (1.0 - 0.01 * k * k) * wns:
                    k += 1
            bands.setdefault(k, []).append(j)
        for k in sorted(bands):
            subsets.append(sorted(bands[k], key=lambda j: (net_slack[j], j)))
    # line 6: Sort(N_n)
    if Nn:
        subsets.append(sorted(Nn, key=lambda j: (wl[j], j)))
    # lines 7-10: GetBatches per subset, Concat
    batch = [0] * n
    nb = 0
    for sub in subsets:
        for i in range(0, len(sub), max_batch):
            for j in sub[i:i + max_batch]:
                batch[j] = nb
            nb += 1
    return np.array(batch, np.int32), nb
