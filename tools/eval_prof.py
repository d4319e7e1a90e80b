"""The evaluator (la_eval_overflow) of config 5 between cudaProfilerStart/Stop, for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from gen import synth  # noqa: E402
from paper_2507_13375_b200 import la  # noqa: E402

d = synth.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
A = la.LayerAssigner(d, device=0)
A.load()
A.assign_all()
A.eval_overflow()
A.sync()
torch.cuda.profiler.start()
A.eval_overflow()
A.sync()
torch.cuda.profiler.stop()
A.close()
