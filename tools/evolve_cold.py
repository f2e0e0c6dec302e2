"""Cold adiabatic evolution in a fresh process (plans and templates empty; NVRTC disk cache as
left by earlier runs): wall time of one 20-step TFIM evolution, then a second one (warm)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import evolution

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
evolution.STEP_WINDOW = int(sys.argv[2]) if len(sys.argv) > 2 else evolution.STEP_WINDOW
cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.05, 1.0)
q.uniform_state(10)
torch.cuda.synchronize()
for label, hz in (("cold", 1.0), ("warm", 0.9)):
    t0 = time.perf_counter()
    st = q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, hz), q.Schedule.linear(), cfg)
    torch.cuda.synchronize()
    print(f"n={n} window={evolution.STEP_WINDOW} {label}: {(time.perf_counter() - t0) * 1e3:.0f} ms", flush=True)
    del st
    torch.cuda.empty_cache()
