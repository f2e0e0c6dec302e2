"""Host-side profile of a time-dependent adiabatic evolution (the per-step planning / kernel
specialisation / launch path), cProfile sorted by cumulative time.  argv: n (26)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q

n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.05, 1.0)
q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 0.9), q.Schedule.linear(), cfg)  # warm-up: kernels
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
st = q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 1.0), q.Schedule.linear(), cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
