"""Debug helper (GPU box): where do GPU and oracle disagree?  Not part of the product."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from gen import synth
from oracle import oracle
from paper_2507_13375_b200 import la


def per_net_mismatch(got, ref, n):
    bad = np.zeros(n, bool)
    wp = ref["wire_ptr"]
    for k in ("wires",):
        a, b = got[k], ref[k]
        diff = np.any(a != b, axis=1)
        idx = np.nonzero(diff)[0]
        nets = np.searchsorted(wp, idx, side="right") - 1
        bad[nets] = True
    return bad


def run(d, sched):
    A = la.LayerAssigner(d, device=0)
    A.load()
    A.set_schedule(sched)
    out = A.run()
    st = A.stats()
    A.close()
    return out, st


def main():
    cases = [("cfg2", synth.make_config(2))]
    for name, d in cases:
        ref = oracle.run(d)
        npins = np.diff(d.pin_ptr)
        for sched in (la.LA_SCHED_BATCH, la.LA_SCHED_DATAFLOW):
            got, st = run(d, sched)
            same_w = np.array_equal(got["wires"], ref["wires"]) if got["wires"].shape == ref["wires"].shape else False
            msg = f"{name} sched={sched} wires_equal={same_w} cost_eq={np.array_equal(got['net_cost'], ref['net_cost'])}"
            if got["wires"].shape == ref["wires"].shape and not same_w:
                bad = per_net_mismatch(got, ref, d.n_nets)
                cbad = got["net_cost"] != ref["net_cost"]
                msg += f" bad_nets={bad.sum()} cost_bad={cbad.sum()} pins_of_bad={np.bincount(npins[bad])[:20].tolist()}"
                i = int(np.nonzero(cbad)[0][0]) if cbad.any() else -1
                if i >= 0:
                    msg += f" first_cost_bad net {i} pins {npins[i]} got {got['net_cost'][i]} ref {ref['net_cost'][i]}"
            print(msg, flush=True)


if __name__ == "__main__":
    main()
