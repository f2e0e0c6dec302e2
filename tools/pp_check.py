"""Quick check of the ping-pong 2-qubit-gate passes: fused vs per-gate at n (argv[1], default 22)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.verify import max_abs_diff

n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
engine.FIRST_RUN_BATCH = False
for name, c in [("var", q.variational_circuit(n, 3, np.random.default_rng(1).uniform(0, 6, n * 7), fused=True)),
                ("trotter", q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)),
                ("grid", q.random_grid_circuit(2, n // 2, 6, 3))]:
    a = c.execute(q.uniform_state(n))
    b = c.execute(q.uniform_state(n), fuse=False)
    torch.cuda.synchronize()
    print(name, n, "passes", c.plan().n_passes, "max|diff|", max_abs_diff(a, b), flush=True)
