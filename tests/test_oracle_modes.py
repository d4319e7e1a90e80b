"""Oracle mode 2 (the nets of each conflict-free batch on several host threads)
against mode 1 (sequential priority order), bit for bit.  Exactness is SURVEY §8(c) c.2: nets of
one batch have disjoint footprints.  Mode 2 produces the full-size golden hashes
(tools/oracle_golden.py), so it is pinned to mode 1 here, at config 3's full size included."""
import numpy as np
import pytest

from gen import synth
from oracle import oracle

INT_KEYS = ("wire_ptr", "wires", "via_ptr", "vias", "wire_dem", "via_dem", "batch_of", "n_nodes")
FP_KEYS = ("net_cost", "sink_delay", "net_cap", "net_rc")


def same(a, b):
    for k in INT_KEYS:
        assert np.array_equal(a[k], b[k]), k
    for k in FP_KEYS:
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k


@pytest.mark.parametrize("threads", [2, 3, 8])
def test_mode2_equals_mode1_small(threads):
    for d in (synth.make_config(1), synth.make_config(2, n_nets=30_000),
              synth.generate(8000, 24, 24, 6, seed=77, pin_max=16, rdrv_mode=1, name="dense")):
        same(oracle.run(d, threads=threads), oracle.run(d))


def test_mode2_equals_mode1_config3_full():
    """Config 3 (1M nets, 1024^2, L = 10, criticality-weighted, r_drv > 0) at full size."""
    d = synth.make_config(3)
    same(oracle.run(d, threads=8), oracle.run(d))


def test_mode2_prefix_and_errors():
    d = synth.make_config(2, n_nets=20_000)
    a, b = oracle.run(d, max_nets=5000, threads=4), oracle.run(d, max_nets=5000)
    same(a, b)
    bad = synth.with_nets(synth.empty_design(8, 8, 4), [dict(pins=[(0, 0, 0, 1, 0), (3, 3, 0, 1, 0)], segs=[(0, 0, 2, 0)])])
    with pytest.raises(oracle.OracleError, match="not on the route"):
        oracle.run(bad, threads=4)
