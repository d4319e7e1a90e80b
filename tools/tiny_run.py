"""Debug helper: one small run through the C ABI (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import synth
from paper_2507_13375_b200 import la
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
sched = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d = synth.make_config(2, n_nets=n)
A = la.LayerAssigner(d, device=0)
A.load()
A.set_schedule(sched)
A.assign_all()
A.sync()
print("ok", A.stats()["max_net_nodes"])
A.close()
