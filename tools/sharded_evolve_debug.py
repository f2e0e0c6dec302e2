"""Debug aid: per-step cost of a sharded-resident adiabatic evolution (compiles, wall time)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import jit
from paper_2009_01845_b200 import sharding as sd
from paper_2009_01845_b200.evolution import _time_steps, trotter_step_circuit

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 2
h0, h1 = q.build_x(n), q.build_tfim(n, 1.0)
cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.01, 1.0)
sh = sd.uniform_sharded(n, shards)
for k, (t, dt) in enumerate(_time_steps(cfg)):
    s_ = min(max(t / cfg.T, 0.0), 1.0)
    c = trotter_step_circuit(q.combine(h0, 1 - s_, h1, s_), dt)
    before = len(jit._cache)
    t0 = time.perf_counter()
    sd.apply_sharded(sh, c)
    torch.cuda.synchronize()
    if k < 5 or k % 20 == 0:
        print(f"step {k}: {1e3 * (time.perf_counter() - t0):.1f} ms, new kernels {len(jit._cache) - before}", flush=True)
