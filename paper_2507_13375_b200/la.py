"""Thin ctypes binding of the C ABI in include/la.h (argument marshalling only).

Every step of the hot path runs in libgapla.so's CUDA kernels.  If the library
cannot be loaded this module raises at import time: there is no CPU fallback.

The functions keep the C names (la_init_grid, la_load_nets, la_assign_batch,
la_commit_demand, la_eval_timing, ...); ``LayerAssigner`` is a small
convenience wrapper over them that takes a ``gen.synth.Design``-like object
(any object with the attributes of la_grid_desc / la_net_desc).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_PKG, "lib", os.environ.get("GAPLA_SO", "libgapla.so"))   # GAPLA_SO: A/B builds in lib/

P = ctypes.POINTER
c_i32, c_i64, c_u8, c_f64, c_void_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint8, ctypes.c_double, ctypes.c_void_p


class LaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


STATUS = {0: "LA_OK", -1: "LA_EINVAL", -2: "LA_ESTATE", -3: "LA_ENOMEM", -4: "LA_ECUDA", -5: "LA_ENCCL", -6: "LA_ERANGE"}
LA_OK, LA_EINVAL, LA_ESTATE, LA_ENOMEM, LA_ECUDA, LA_ENCCL, LA_ERANGE = 0, -1, -2, -3, -4, -5, -6


class la_grid_desc(ctypes.Structure):
    _fields_ = [("X", c_i32), ("Y", c_i32), ("L", c_i32),
                ("dir", P(c_u8)), ("routable", P(c_u8)), ("r", P(c_f64)), ("c", P(c_f64)), ("vr", P(c_f64)),
                ("ofw", P(c_f64)), ("s_pos", c_f64), ("s_zero", c_f64),
                ("wire_cap", P(c_i32)), ("via_cap", P(c_i32)), ("wire_dem0", P(c_i32)), ("via_dem0", P(c_i32)),
                ("W_D", c_f64), ("W_CAP", c_f64), ("W_CONG", c_f64), ("W_VIA", c_f64), ("r_avg", c_f64),
                ("logit_k", c_f64), ("logit_b", c_f64), ("w_floor", c_f64), ("delta_lo", c_i32), ("delta_hi", c_i32),
                ("device", c_i32), ("rank", c_i32), ("world", c_i32), ("nccl_id", c_void_p), ("stream", c_void_p)]


class la_net_desc(ctypes.Structure):
    _fields_ = [("n_nets", c_i64), ("pin_ptr", P(c_i64)), ("pin_x", P(c_i32)), ("pin_y", P(c_i32)),
                ("pin_layer", P(c_u8)), ("pin_cap", P(c_f64)), ("pin_slack", P(c_f64)),
                ("seg_ptr", P(c_i64)), ("seg_xy", P(c_i32)), ("r_drv", P(c_f64)), ("order_key", P(c_i64)),
                ("wns", c_f64)]


class la_eval(ctypes.Structure):
    _fields_ = [("tof_wire", c_f64), ("tof_via", c_f64), ("legacy_wire", c_i64), ("legacy_via", c_i64),
                ("wirelength", c_i64 * 16), ("via_cuts", c_i64), ("wire_cap", c_f64), ("out_of_domain", c_i64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["wirelength"] = list(self.wirelength)
        return d


class la_stats(ctypes.Structure):
    _fields_ = [("n_nets", c_i64), ("n_pins", c_i64), ("n_nodes", c_i64), ("n_sinks", c_i64),
                ("wirelength", c_i64), ("footprint", c_i64), ("n_batches", c_i32), ("max_height", c_i32),
                ("max_batch_nets", c_i64), ("max_net_nodes", c_i64), ("via_cuts", c_i64), ("launches", c_i64),
                ("load_ms", c_f64), ("batch_ms", c_f64), ("wire_state_words", c_i64), ("via_state_words", c_i64),
                ("h2d_bytes", c_i64), ("d2h_bytes", c_i64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class la_profile(ctypes.Structure):
    _fields_ = [("assign_launches", c_i64), ("commit_launches", c_i64), ("elmore_launches", c_i64),
                ("reconcile_calls", c_i64), ("assign_ms", c_f64), ("commit_ms", c_f64), ("elmore_ms", c_f64),
                ("reconcile_ms", c_f64), ("eval_launches", c_i64), ("eval_ms", c_f64),
                ("pretime_launches", c_i64), ("order_calls", c_i64), ("pretime_ms", c_f64), ("order_ms", c_f64),
                ("order_kernel_ms", c_f64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA library is required; there is no CPU fallback)")
    lib = ctypes.CDLL(SO_PATH)
    sig = {
        "la_init_grid": ([P(la_grid_desc), P(c_void_p)], c_i32),
        "la_load_nets": ([c_void_p, P(la_net_desc), P(c_i32)], c_i32),
        "la_assign_batch": ([c_void_p, c_i32], c_i32),
        "la_commit_demand": ([c_void_p, c_i32], c_i32),
        "la_assign_all": ([c_void_p], c_i32),
        "la_set_schedule": ([c_void_p, c_i32], c_i32),
        "la_set_tracing": ([c_void_p, c_i32], c_i32),
        "la_eval_overflow": ([c_void_p, P(la_eval)], c_i32),
        "la_set_snapshot_batches": ([c_void_p, P(c_i32), c_i64], c_i32),
        "la_batch_extent": ([c_void_p, c_i32, P(c_i64), P(c_i64)], c_i32),
        "la_get_decisions": ([c_void_p, c_i32, P(ctypes.c_uint32), P(c_f64)], c_i32),
        "la_put_decisions": ([c_void_p, c_i32, P(ctypes.c_uint32), P(c_f64)], c_i32),
        "la_paper_batches": ([c_void_p, P(la_net_desc), P(c_i32), c_f64, c_i32, c_i64, P(c_i32), P(c_i32)], c_i32),
        "la_pre_timing": ([c_void_p, c_f64, c_f64, c_f64, c_f64, P(c_f64), P(c_f64)], c_i32),
        "la_get_trace": ([c_void_p, P(c_i64)], c_i32),
        "la_eval_timing": ([c_void_p, P(c_f64), P(c_f64), P(c_f64)], c_i32),
        "la_get_solution": ([c_void_p, P(c_i64), P(c_i64), P(c_i64), P(c_i32), P(c_i64), P(c_i32), P(c_f64)], c_i32),
        "la_get_demand": ([c_void_p, P(c_i32), P(c_i32)], c_i32),
        "la_get_batches": ([c_void_p, P(c_i32)], c_i32),
        "la_reset": ([c_void_p], c_i32),
        "la_get_stats": ([c_void_p, P(la_stats)], c_i32),
        "la_sync": ([c_void_p], c_i32),
        "la_destroy": ([c_void_p], None),
        "la_last_error": ([], ctypes.c_char_p),
        "la_shard_range": ([c_i64, c_i32, c_i32, P(c_i64), P(c_i64)], None),
        "la_set_profiling": ([c_void_p, c_i32], c_i32),
        "la_get_profile": ([c_void_p, P(la_profile), c_i32], c_i32),
        "la_nccl_unique_id": ([c_void_p], c_i32),
        "la_fp64_peak": ([c_i32, P(c_f64)], c_i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = _load()
EXPORTS = ("la_init_grid", "la_load_nets", "la_assign_batch", "la_commit_demand", "la_assign_all", "la_eval_timing",
           "la_get_solution", "la_get_demand", "la_get_batches", "la_reset", "la_get_stats", "la_sync", "la_destroy",
           "la_last_error", "la_shard_range", "la_set_profiling", "la_get_profile", "la_nccl_unique_id",
           "la_set_schedule", "la_set_tracing", "la_get_trace", "la_eval_overflow", "la_set_snapshot_batches",
           "la_paper_batches", "la_batch_extent", "la_get_decisions", "la_put_decisions", "la_fp64_peak",
           "la_pre_timing")


def _check(st):
    if st != LA_OK:
        raise LaError(st, _lib.la_last_error().decode(errors="replace"))


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(P(ct))


# ---------------------------------------------------------------- C names ---
def la_init_grid(desc: la_grid_desc):
    ctx = c_void_p()
    _check(_lib.la_init_grid(ctypes.byref(desc), ctypes.byref(ctx)))
    return ctx


def la_load_nets(ctx, desc: la_net_desc) -> int:
    nb = c_i32()
    _check(_lib.la_load_nets(ctx, ctypes.byref(desc), ctypes.byref(nb)))
    return nb.value


def la_assign_batch(ctx, k: int):
    _check(_lib.la_assign_batch(ctx, k))


def la_commit_demand(ctx, k: int):
    _check(_lib.la_commit_demand(ctx, k))


def la_assign_all(ctx):
    _check(_lib.la_assign_all(ctx))


def la_eval_timing(ctx, sink_delay=None, net_cap=None, net_rc=None):
    _check(_lib.la_eval_timing(ctx, _p(sink_delay, c_f64), _p(net_cap, c_f64), _p(net_rc, c_f64)))


def la_get_solution(ctx, n_nets: int):
    nw, nv = c_i64(), c_i64()
    _check(_lib.la_get_solution(ctx, ctypes.byref(nw), ctypes.byref(nv), None, None, None, None, None))
    wire_ptr = np.zeros(n_nets + 1, np.int64)
    via_ptr = np.zeros(n_nets + 1, np.int64)
    wires = np.zeros((max(nw.value, 1), 5), np.int32)
    vias = np.zeros((max(nv.value, 1), 4), np.int32)
    cost = np.zeros(n_nets, np.float64)
    _check(_lib.la_get_solution(ctx, ctypes.byref(nw), ctypes.byref(nv), _p(wire_ptr, c_i64), _p(wires, c_i32),
                                _p(via_ptr, c_i64), _p(vias, c_i32), _p(cost, c_f64)))
    return dict(wire_ptr=wire_ptr, wires=wires[: nw.value], via_ptr=via_ptr, vias=vias[: nv.value], net_cost=cost)


def la_get_demand(ctx, wire_dem=None, via_dem=None):
    _check(_lib.la_get_demand(ctx, _p(wire_dem, c_i32), _p(via_dem, c_i32)))


def la_get_batches(ctx, out):
    _check(_lib.la_get_batches(ctx, _p(out, c_i32)))


LA_SCHED_DATAFLOW, LA_SCHED_BATCH = 0, 1


def la_set_schedule(ctx, schedule: int):
    _check(_lib.la_set_schedule(ctx, int(schedule)))


def la_eval_overflow(ctx) -> dict:
    out = la_eval()
    _check(_lib.la_eval_overflow(ctx, ctypes.byref(out)))
    return out.as_dict()


def la_set_snapshot_batches(ctx, batch_of):
    if batch_of is None:
        _check(_lib.la_set_snapshot_batches(ctx, None, 0))
        return
    b = np.ascontiguousarray(batch_of, np.int32)
    _check(_lib.la_set_snapshot_batches(ctx, b.ctypes.data_as(P(c_i32)), b.shape[0]))


def net_desc_of(d, keep) -> la_net_desc:
    """la_net_desc over the arrays of design ``d`` (converted copies are appended to ``keep``)."""
    def arr(a, dt):
        x = np.ascontiguousarray(a, dtype=dt)
        keep.append(x)
        return x

    n = la_net_desc()
    n.n_nets = d.n_nets
    n.pin_ptr = _p(arr(d.pin_ptr, np.int64), c_i64)
    n.pin_x, n.pin_y = _p(arr(d.pin_x, np.int32), c_i32), _p(arr(d.pin_y, np.int32), c_i32)
    n.pin_layer = _p(arr(d.pin_layer, np.uint8), c_u8)
    n.pin_cap, n.pin_slack = _p(arr(d.pin_cap, np.float64), c_f64), _p(arr(d.pin_slack, np.float64), c_f64)
    n.seg_ptr = _p(arr(d.seg_ptr, np.int64), c_i64)
    n.seg_xy = _p(arr(np.asarray(d.seg_xy).reshape(-1), np.int32), c_i32)
    n.r_drv = _p(arr(d.r_drv, np.float64), c_f64)
    n.order_key = _p(arr(d.order_key, np.int64), c_i64)
    n.wns = d.wns
    return n


def la_paper_batches(ctx, d, criticality, alpha: float = 0.7, th: int = 3, max_batch: int = 1 << 20):
    """Alg. 1 lines 3-10 on the GPU (include/la.h): batch id per net (input order) and the batch count."""
    keep = []
    desc = net_desc_of(d, keep)
    crit = np.ascontiguousarray(criticality, np.int32)
    out = np.zeros(d.n_nets, np.int32)
    nb = c_i32(0)
    _check(_lib.la_paper_batches(ctx, ctypes.byref(desc), crit.ctypes.data_as(P(c_i32)), float(alpha), int(th),
                                 int(max_batch), out.ctypes.data_as(P(c_i32)), ctypes.byref(nb)))
    return out, int(nb.value)


def la_pre_timing(ctx, n_pins: int, n_nets: int, r_h=float("nan"), r_v=float("nan"), c_h=float("nan"),
                  c_v=float("nan")):
    """Pre-assignment pi-model timing on the loaded 2D trees (include/la.h): (sink_delay, net_cap)."""
    delay = np.zeros(n_pins, np.float64)
    cap = np.zeros(n_nets, np.float64)
    _check(_lib.la_pre_timing(ctx, float(r_h), float(r_v), float(c_h), float(c_v), _p(delay, c_f64), _p(cap, c_f64)))
    return delay, cap


def la_get_decisions(ctx, batch: int):
    """Host transport: this rank's packed decisions and net costs of ``batch`` (after assign)."""
    nodes, nets = c_i64(0), c_i64(0)
    _check(_lib.la_batch_extent(ctx, batch, ctypes.byref(nodes), ctypes.byref(nets)))
    dec = np.zeros(nodes.value, np.uint32)
    cost = np.zeros(nets.value, np.float64)
    _check(_lib.la_get_decisions(ctx, batch, dec.ctypes.data_as(P(ctypes.c_uint32)), cost.ctypes.data_as(P(c_f64))))
    return dec, cost


def la_put_decisions(ctx, batch: int, dec, cost):
    dec = np.ascontiguousarray(dec, np.uint32)
    cost = np.ascontiguousarray(cost, np.float64)
    _check(_lib.la_put_decisions(ctx, batch, dec.ctypes.data_as(P(ctypes.c_uint32)), cost.ctypes.data_as(P(c_f64))))


def la_set_tracing(ctx, enable: bool):
    _check(_lib.la_set_tracing(ctx, 1 if enable else 0))


def la_get_trace(ctx, n_nets: int):
    out = np.zeros((n_nets, 5), np.int64)
    _check(_lib.la_get_trace(ctx, out.ctypes.data_as(P(c_i64))))
    return out


def la_reset(ctx):
    _check(_lib.la_reset(ctx))


def la_get_stats(ctx) -> dict:
    s = la_stats()
    _check(_lib.la_get_stats(ctx, ctypes.byref(s)))
    return s.as_dict()


def la_sync(ctx):
    _check(_lib.la_sync(ctx))


def la_fp64_peak(device: int = 0) -> float:
    """FP64 vector-pipe peak of the device, lane ops per second (measurement aid)."""
    v = c_f64(0.0)
    _check(_lib.la_fp64_peak(int(device), ctypes.byref(v)))
    return v.value


def la_destroy(ctx):
    _lib.la_destroy(ctx)


def la_shard_range(n: int, world: int, rank: int):
    b, e = c_i64(), c_i64()
    _lib.la_shard_range(n, world, rank, ctypes.byref(b), ctypes.byref(e))
    return b.value, e.value


def la_set_profiling(ctx, enable: bool):
    _check(_lib.la_set_profiling(ctx, 1 if enable else 0))


def la_get_profile(ctx, reset: bool = True) -> dict:
    p = la_profile()
    _check(_lib.la_get_profile(ctx, ctypes.byref(p), 1 if reset else 0))
    return p.as_dict()


def la_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.la_nccl_unique_id(ctypes.cast(buf, c_void_p)))
    return buf.raw


# ------------------------------------------------------------ convenience ---
class LayerAssigner:
    """Owns one la_ctx.  ``d`` is a gen.synth.Design (or any object with the same
    attributes).  Host arrays are converted once and kept alive for the calls."""

    def __init__(self, d, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 stream: int | None = None):
        self._keep = []
        k = self._keep

        def arr(a, dt):
            if a is None:
                return None
            x = np.ascontiguousarray(a, dtype=dt)
            k.append(x)
            return x

        self.d = d
        g = la_grid_desc()
        g.X, g.Y, g.L = d.X, d.Y, d.L
        g.dir = _p(arr(d.dir, np.uint8), c_u8)
        g.routable = _p(arr(d.routable, np.uint8), c_u8)
        g.r, g.c = _p(arr(d.r, np.float64), c_f64), _p(arr(d.c, np.float64), c_f64)
        g.vr, g.ofw = _p(arr(d.vr, np.float64), c_f64), _p(arr(d.ofw, np.float64), c_f64)
        g.s_pos, g.s_zero = d.s_pos, d.s_zero
        g.wire_cap, g.via_cap = _p(arr(d.wire_cap, np.int32), c_i32), _p(arr(d.via_cap, np.int32), c_i32)
        g.wire_dem0 = _p(arr(d.wire_dem0, np.int32), c_i32)
        g.via_dem0 = _p(arr(d.via_dem0, np.int32), c_i32)
        g.W_D, g.W_CAP, g.W_CONG, g.W_VIA, g.r_avg = d.W_D, d.W_CAP, d.W_CONG, d.W_VIA, d.r_avg
        g.logit_k, g.logit_b, g.w_floor = d.logit_k, d.logit_b, d.w_floor
        g.delta_lo, g.delta_hi = d.delta_lo, d.delta_hi
        g.device, g.rank, g.world = device, rank, world
        if nccl_id is not None:
            self._nid = ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
            g.nccl_id = ctypes.cast(self._nid, c_void_p)
        g.stream = stream
        self.grid_desc = g
        self.ctx = la_init_grid(g)
        self.n_batches = None

    def net_desc(self, d=None) -> la_net_desc:
        return net_desc_of(d or self.d, self._keep)

    def load(self, d=None, snapshot_batches=None) -> int:
        """la_load_nets; ``snapshot_batches`` (int32 per net): paper-style batches (NEXT #1)."""
        if snapshot_batches is not None:
            la_set_snapshot_batches(self.ctx, snapshot_batches)
        self.n_batches = la_load_nets(self.ctx, self.net_desc(d))
        return self.n_batches

    def assign_batch(self, k):
        la_assign_batch(self.ctx, k)

    def commit_demand(self, k):
        la_commit_demand(self.ctx, k)

    def assign_all(self):
        la_assign_all(self.ctx)

    def set_schedule(self, schedule: int):
        la_set_schedule(self.ctx, schedule)

    def eval_timing(self):
        d = self.d
        sd = np.zeros(d.n_pins, np.float64)
        nc = np.zeros(d.n_nets, np.float64)
        nr = np.zeros(d.n_nets, np.float64)
        la_eval_timing(self.ctx, sd, nc, nr)
        return dict(sink_delay=sd, net_cap=nc, net_rc=nr)

    def eval_overflow(self):
        """la_eval_overflow: Eq. (3)/(2) total overflow, wirelength per layer, via cuts, wire C."""
        return la_eval_overflow(self.ctx)

    def solution(self):
        return la_get_solution(self.ctx, self.d.n_nets)

    def demand(self):
        wd = np.zeros(self.d.wire_cap.shape[0], np.int32)
        vd = np.zeros(self.d.via_cap.shape[0], np.int32)
        la_get_demand(self.ctx, wd, vd)
        return wd, vd

    def batches(self):
        out = np.zeros(self.d.n_nets, np.int32)
        la_get_batches(self.ctx, out)
        return out

    def reset(self):
        la_reset(self.ctx)

    def stats(self):
        return la_get_stats(self.ctx)

    def profiling(self, enable: bool):
        la_set_profiling(self.ctx, enable)

    def profile(self, reset: bool = True):
        return la_get_profile(self.ctx, reset)

    def sync(self):
        la_sync(self.ctx)

    def close(self):
        if self.ctx:
            la_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self):
        """Whole hot path: every batch (assign + commit) then Elmore; returns all outputs."""
        self.assign_all()
        out = self.eval_timing()
        out.update(self.solution())
        wd, vd = self.demand()
        out.update(wire_dem=wd, via_dem=vd, batch_of=self.batches())
        return out
