"""Mutation check of the oracle's pins (VERDICT r1 'next round' item 1).

Applies one plausible slip at a time to a scratch copy of oracle/la_oracle.cpp, rebuilds the
oracle from that copy, runs tests/test_oracle_pins.py against it, and reports whether a pin
turned red.  The tree under oracle/ is restored afterwards.

    python tools/oracle_mutations.py
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "la_oracle.cpp")
SO = os.path.join(ROOT, "oracle", "liboracle.so")

MUTATIONS = [
    ("look-ahead dropped: cost' = cost (P:448-453)",
     "double cp = cost + o.B * st.ur[n];", "double cp = cost;"),
    ("ur from the parent's edge length (O3, R6)",
     "st.ur[T.par[n]] + C.r_avg * T.len[n];", "st.ur[T.par[n]] + C.r_avg * T.len[T.par[n]];"),
    ("ur(root) = 0 instead of r_drv (O3, R6)",
     "(nets->r_drv ? nets->r_drv[net] : 0.0)", "0.0"),
    ("Eq. (3) table not clamped above (R20)",
     "if (delta > C.g->delta_hi) delta = C.g->delta_hi;", "if (delta > C.g->delta_hi + 100) delta = C.g->delta_hi;"),
    ("son tie-break: highest j (R21)",
     "if (jb < 0 || cp < cpb) {", "if (jb < 0 || cp <= cpb) {"),
    ("span key without t - b (R21)",
     "(Gp == bGp && (t - b < bt - bb || (t - b == bt - bb && b < bb)))", "(Gp == bGp && b < bb)"),
    ("vcong counted for [b, b] (R10)",
     "for (int k = b; k < t; k++) V = V + kap[k];", "for (int k = b; k <= t && k < L - 1; k++) V = V + kap[k];"),
    ("pin-via delay with the wrong layer pair (Alg. 3 l.4-7)",
     "F0 = F0 + wq * (N->pin_cap[q] * C.VR[(size_t)N->pin_layer[q] * L + l]);",
     "F0 = F0 + wq * (N->pin_cap[q] * C.VR[(size_t)N->pin_layer[q] * L + 0]);"),
]


def main() -> int:
    orig = open(SRC).read()
    backup = SRC + ".orig"
    shutil.copy(SRC, backup)
    bad = 0
    try:
        for name, a, b in MUTATIONS:
            assert a in orig, name
            open(SRC, "w").write(orig.replace(a, b, 1))
            if os.path.exists(SO):
                os.remove(SO)
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-p", "no:cacheprovider"],
                               cwd=ROOT, capture_output=True, text=True)
            last = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
            caught = r.returncode != 0
            bad += not caught
            print(f"{'CAUGHT ' if caught else 'MISSED '} {name}: {last}", flush=True)
    finally:
        shutil.move(backup, SRC)
        if os.path.exists(SO):
            os.remove(SO)
        subprocess.check_call([sys.executable, "-c", "from oracle import oracle; oracle.build()"], cwd=ROOT)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
