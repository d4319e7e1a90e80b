"""World-size-2 CPU (gloo) tests of the multi-GPU reconcile protocol.

The N > 1 path shards the nets of every conflict-free batch over the ranks with la_shard_range
(contiguous chunks), every rank packs the decisions of its own chunk into a batch-wide array
whose other slots are 0, and ONE sum all-reduce makes every rank hold every decision (a sum of
disjoint one-hot slots is an all-gather); each rank then commits the whole batch, so the integer
demand replicas stay identical.  These tests run that protocol over gloo with two processes, the
shard ranges coming from the real C-ABI library, the decisions from the CPU oracle (test
infrastructure), and check: the chunks partition every batch, the all-reduced decisions equal the
full decision array on both ranks, the fp64 net costs survive the sum bit-exactly (x + 0 == x),
and the demand replicas built from the reconciled decisions are identical and equal the oracle's.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import synth
from helpers import rebuild_demand


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(d, ref):
    """Per-net decision words: for every wire (x1,y1,x2,y2,l) of net j one u32 word
    (l + 1) | valid, in the oracle's per-net wire order; and one word per via stack (b | t << 4 | 1 << 8)."""
    wires, vias = ref["wires"], ref["vias"]
    wdec = (wires[:, 4].astype(np.int64) + 1) | (1 << 8)
    vdec = vias[:, 2].astype(np.int64) | (vias[:, 3].astype(np.int64) << 4) | (1 << 8)
    return wdec, vdec


def _worker(rank, world, port, d, ref, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_13375_b200 import la
        batch_of = ref["batch_of"]
        nb = int(batch_of.max()) + 1 if len(batch_of) else 0
        wdec_full, vdec_full = _pack(d, ref)
        wp, vp = ref["wire_ptr"], ref["via_ptr"]
        got_w = np.zeros_like(wdec_full)
        got_v = np.zeros_like(vdec_full)
        got_cost = np.zeros(d.n_nets, np.float64)
        owner = np.zeros(d.n_nets, np.int64)
        for b in range(nb):
            nets = np.nonzero(batch_of == b)[0]            # the batch's nets (input order)
            s0, s1 = la.la_shard_range(len(nets), world, rank)
            mine = nets[s0:s1]
            bw = np.zeros_like(wdec_full)
            bv = np.zeros_like(vdec_full)
            bc = np.zeros(d.n_nets, np.float64)
            bo = np.zeros(d.n_nets, np.int64)
            for j in mine:
                bw[wp[j]:wp[j + 1]] = wdec_full[wp[j]:wp[j + 1]]
                bv[vp[j]:vp[j + 1]] = vdec_full[vp[j]:vp[j + 1]]
                bc[j] = ref["net_cost"][j]
                bo[j] = 1
            tw, tv, tc, to = (torch.from_numpy(a) for a in (bw, bv, bc, bo))
            for t in (tw, tv, tc, to):
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
            got_w += tw.numpy()
            got_v += tv.numpy()
            got_cost += tc.numpy()
            owner += to.numpy()
        # replicated commit from the reconciled decisions (O8), on every rank
        wires = ref["wires"].copy()
        wires[:, 4] = (got_w & 0xff) - 1
        vias = ref["vias"].copy()
        vias[:, 2] = got_v & 0xf
        vias[:, 3] = (got_v >> 4) & 0xf
        wdem, vdem = rebuild_demand(d, wires, vias)
        out_q.put((rank, got_w, got_v, got_cost, owner, wdem, vdem))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def design_and_ref():
    from oracle import oracle
    d = synth.make_config(1)
    return d, oracle.run(d)


def test_two_rank_reconcile_equals_full_solution(design_and_ref):
    d, ref = design_and_ref
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, ref, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wfull, vfull = _pack(d, ref)
    for rank, got_w, got_v, got_cost, owner, wdem, vdem in res:
        assert np.all(owner == 1), "every net is assigned by exactly one rank"
        assert np.array_equal(got_w, wfull) and np.array_equal(got_v, vfull)
        assert np.array_equal(got_cost.view(np.int64), ref["net_cost"].view(np.int64)), "x + 0 must be exact"
        assert np.array_equal(wdem, ref["wire_dem"]) and np.array_equal(vdem, ref["via_dem"])
    # replicas identical across ranks
    assert np.array_equal(res[0][5], res[1][5]) and np.array_equal(res[0][6], res[1][6])


def test_shards_balance_each_batch(design_and_ref):
    """Per batch, the two chunks differ by at most one net and are contiguous in batch order."""
    from paper_2507_13375_b200 import la
    _, ref = design_and_ref
    batch_of = ref["batch_of"]
    for b in range(int(batch_of.max()) + 1):
        n = int((batch_of == b).sum())
        (a0, a1), (b0, b1) = la.la_shard_range(n, 2, 0), la.la_shard_range(n, 2, 1)
        assert a0 == 0 and a1 == b0 and b1 == n and abs((a1 - a0) - (b1 - b0)) <= 1
