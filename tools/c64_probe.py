"""Device time of complex64 plans (n = 30): grid 3x10, four Trotter steps, variational L5 --
run with QSB_C64_WIDE_MIN_CODE=0 / default to compare the 256 x 32 rule."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine

n = 30
step = q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)
params = np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11)
for name, circ in (("grid", q.random_grid_circuit(3, 10, 20, 42)),
                   ("trotter4", q.Circuit(n).add([g for _ in range(4) for g in step.queue])),
                   ("variational", q.variational_circuit(n, 5, params, fused=True))):
    st = q.uniform_state(n, q.Precision.F32)
    plan = engine.plan_for_state(st, circ.queue)
    holder = {}
    engine.run_plan(st, plan, holder)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        engine.run_plan(st, plan, holder)
    b.record()
    torch.cuda.synchronize()
    print(f"c64 {name}: {a.elapsed_time(b) / 3:.2f} ms, {plan.n_passes} passes "
          f"(QSB_C64_WIDE_MIN_CODE={os.environ.get('QSB_C64_WIDE_MIN_CODE', 'default')})", flush=True)
