"""Golden SHA-256 hashes of the CPU oracle's outputs at full size (SURVEY §8(d)
d.5: "Parity at config 5 compares hashes").  Calls only gen/ (seeded input) and oracle/ (mode 2:
the nets of each conflict-free batch on all host threads, exact by SURVEY §8(c) c.2 and checked
bit-equal to mode 1 by tests/test_oracle_modes.py).  Writes tests/golden/oracle_hashes_cfg{k}.json.

    python tools/oracle_golden.py 4 5
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from gen import synth  # noqa: E402
from helpers import output_hashes  # noqa: E402
from oracle import oracle  # noqa: E402


def main(cfgs):
    threads = os.cpu_count() or 1
    for k in cfgs:
        t0 = time.time()
        d = synth.make_config(k)
        tg = time.time() - t0
        t0 = time.time()
        r = oracle.run(d, threads=threads)
        tr = time.time() - t0
        h = output_hashes(r)
        rec = {"_source": "tools/oracle_golden.py: oracle.run(synth.make_config(%d), threads=%d) (mode 2); "
                          "hashes of tests/helpers.py HASH_KEYS" % (k, threads),
               "workload": d.name, "n_nets": d.n_nets, "n_pins": d.n_pins,
               "oracle_wall_s": round(tr, 1), "oracle_dp_s": round(r["elapsed_s"], 1), "generate_s": round(tg, 1),
               "threads": threads, "host": platform.processor() or platform.machine(),
               "n_batches": int(r["batch_of"].max()) + 1, "hashes": h}
        with open(os.path.join(ROOT, "tests", "golden", f"oracle_hashes_cfg{k}.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print(f"cfg{k}: {d.n_nets} nets, oracle {tr:.1f} s on {threads} threads, {rec['n_batches']} batches", flush=True)
        del r, d


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4, 5])
