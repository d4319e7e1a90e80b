"""Small design builders shared by the tests (input construction only)."""
from __future__ import annotations

import copy
import json
import os

import numpy as np

from gen import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def single_net(d: synth.Design, net: int) -> synth.Design:
    """Design with the same grid/tech/weights and only net ``net``."""
    e = copy.copy(d)
    a, b = int(d.pin_ptr[net]), int(d.pin_ptr[net + 1])
    s0, s1 = int(d.seg_ptr[net]), int(d.seg_ptr[net + 1])
    e.pin_ptr = np.array([0, b - a], np.int64)
    e.pin_x, e.pin_y = d.pin_x[a:b].copy(), d.pin_y[a:b].copy()
    e.pin_layer, e.pin_cap, e.pin_slack = d.pin_layer[a:b].copy(), d.pin_cap[a:b].copy(), d.pin_slack[a:b].copy()
    e.seg_ptr = np.array([0, s1 - s0], np.int64)
    e.seg_xy = d.seg_xy[s0:s1].copy()
    e.r_drv = d.r_drv[net:net + 1].copy()
    e.order_key = np.zeros(1, np.int64)
    return e


def randomize_state(d: synth.Design, rng: np.random.Generator, wire_caps=(0, 1, 2, 3), via_caps=(0, 2, 4),
                    wire_dem=4, via_dem=3) -> synth.Design:
    """Random capacities (zeros included, so s_zero is exercised) and initial demand."""
    e = copy.copy(d)
    e.wire_cap = rng.choice(np.array(wire_caps, np.int32), size=d.wire_cap.shape[0]).astype(np.int32)
    e.via_cap = rng.choice(np.array(via_caps, np.int32), size=d.via_cap.shape[0]).astype(np.int32)
    e.wire_dem0 = rng.integers(0, wire_dem + 1, size=d.wire_cap.shape[0]).astype(np.int32)
    e.via_dem0 = rng.integers(0, via_dem + 1, size=d.via_cap.shape[0]).astype(np.int32)
    return e


def tiny_pool(seed: int, L: int, n: int = 400, X: int = 6, Y: int = 6, pin_max: int = 4, rdrv_mode: int = 0):
    return synth.generate(n_nets=n, X=X, Y=Y, L=L, seed=seed, pin_max=pin_max, rdrv_mode=rdrv_mode,
                          name=f"tiny_pool_{seed}")


def fixture_design(fx, tech, **weights) -> synth.Design:
    d = synth.empty_design(16, 16, tech["L"])
    d.dir = np.array(tech["dir"], np.uint8)
    d.r = np.array(tech["r"], np.float64)
    d.c = np.array(tech["c"], np.float64)
    d.vr = np.array(tech["vr"], np.float64)
    d.routable = np.array(fx["routable"], np.uint8)
    n_wire = sum((d.X - 1) * d.Y if d.dir[l] == 0 else d.X * (d.Y - 1) for l in range(d.L))
    d.wire_cap = np.full(n_wire, 10, np.int32)
    for k, v in weights.items():
        setattr(d, k, v)
    return synth.with_nets(d, [dict(pins=[tuple(p) for p in fx["pins"]], segs=[tuple(s) for s in fx["segs"]])])


def rebuild_demand(d: synth.Design, wires, vias):
    """Demand grids rebuilt from a solution (O8 by definition): +1 per unit edge of
    every wire on its layer, +1 per via cut."""
    wd = np.zeros(d.wire_cap.shape[0], np.int64)
    vd = np.zeros(d.via_cap.shape[0], np.int64)
    offs = np.concatenate([[0], np.cumsum(d.wire_layer_sizes())])
    for (x1, y1, x2, y2, l) in np.asarray(wires, np.int64):
        if y1 == y2:
            xs = np.arange(x1, x2)
            wd[offs[l] + y1 * (d.X - 1) + xs] += 1
        else:
            ys = np.arange(y1, y2)
            wd[offs[l] + ys * d.X + x1] += 1
    for (x, y, b, t) in np.asarray(vias, np.int64):
        for k in range(b, t):
            vd[(k * d.Y + y) * d.X + x] += 1
    if d.wire_dem0 is not None:
        wd += d.wire_dem0
    if d.via_dem0 is not None:
        vd += d.via_dem0
    return wd.astype(np.int32), vd.astype(np.int32)


# Canonical outputs of one whole run (SURVEY §8(d) d.5 "parity at config 5 compares hashes"): the
# arrays, their dtypes and byte order are fixed here so the oracle's golden hashes
# (tools/oracle_golden.py) and the GPU run hash the same bytes.  Floating-point outputs are hashed
# as their IEEE bit patterns.  No method arithmetic.
HASH_KEYS = (("wire_ptr", "<i8"), ("wires", "<i4"), ("via_ptr", "<i8"), ("vias", "<i4"), ("wire_dem", "<i4"),
             ("via_dem", "<i4"), ("batch_of", "<i4"), ("net_cost", "<f8"), ("sink_delay", "<f8"),
             ("net_cap", "<f8"), ("net_rc", "<f8"))
HASH_CHUNKS = 64


def output_hashes(res) -> dict:
    """SHA-256 of every canonical output array, plus per-chunk hashes (HASH_CHUNKS equal slices
    along axis 0) so a mismatch can be localised without the oracle's arrays."""
    import hashlib
    out = {}
    for k, dt in HASH_KEYS:
        a = np.ascontiguousarray(np.asarray(res[k]).astype(dt, copy=False))
        n = a.shape[0]
        out[k] = {"sha256": hashlib.sha256(a.tobytes()).hexdigest(), "shape": list(a.shape),
                  "chunks": [hashlib.sha256(a[n * i // HASH_CHUNKS: n * (i + 1) // HASH_CHUNKS].tobytes()).hexdigest()[:16]
                             for i in range(HASH_CHUNKS)]}
    return out


def compare_hashes(got: dict, want: dict) -> list:
    """Mismatch report: per array, the shape difference or the first differing chunk and its
    element range."""
    bad = []
    for k, _ in HASH_KEYS:
        g, w = got[k], want[k]
        if g["sha256"] == w["sha256"]:
            continue
        if g["shape"] != w["shape"]:
            bad.append(f"{k}: shape {g['shape']} != {w['shape']}")
            continue
        n = w["shape"][0]
        first = next(i for i in range(HASH_CHUNKS) if g["chunks"][i] != w["chunks"][i])
        bad.append(f"{k}: first differing chunk {first} = elements [{n * first // HASH_CHUNKS}, "
                   f"{n * (first + 1) // HASH_CHUNKS})")
    return bad
