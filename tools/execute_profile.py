"""Host-side profile of Circuit.execute on a small state (python tools/execute_profile.py n)."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01845_b200 as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
c = q.variational_circuit(n, 5, np.random.default_rng(42).uniform(0, 6.28, n * 11), fused=True)
for _ in range(3):
    c.execute()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    c.execute()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
