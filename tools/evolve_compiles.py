"""How many pass kernels an adiabatic evolution compiles when an evolution with another field
strength ran before (debug aid: python tools/evolve_compiles.py n)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import jit

n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.05, 1.0)
for h in (0.9, 1.0, 1.1):
    before = len(jit._cache)
    t0 = time.perf_counter()
    q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, h), q.Schedule.linear(), cfg)
    torch.cuda.synchronize()
    print(f"h={h}: {1e3 * (time.perf_counter() - t0):.0f} ms, new kernels {len(jit._cache) - before}", flush=True)
