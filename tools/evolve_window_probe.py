"""Host-side profile of adiabatic_evolve at small n (host-bound sizes): wall time per window
size, new kernels compiled in the timed run, and a cProfile of the heaviest calls."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import evolution, jit

for n in [int(a) for a in sys.argv[1:]] or [26]:
    for w in (1, 4):
        evolution.STEP_WINDOW = w
        cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.05, 1.0)
        q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 0.9), q.Schedule.linear(), cfg)
        torch.cuda.synchronize()
        c0 = len(jit._cache)
        t0 = time.perf_counter()
        st = q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 1.0), q.Schedule.linear(), cfg)
        torch.cuda.synchronize()
        print(f"n={n} w={w}: {(time.perf_counter() - t0) * 1e3:.1f} ms, new kernels {len(jit._cache) - c0}", flush=True)
        pr = cProfile.Profile()
        pr.enable()
        st = q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 1.1), q.Schedule.linear(), cfg)
        torch.cuda.synchronize()
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(18)
        del st
        torch.cuda.empty_cache()
