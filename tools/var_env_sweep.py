"""Variational-30 L5 fused (c128 / c64) and grid 3x10 c128 device time per circuit, warm -- run
under different QSB_* env settings to compare kernel-generation switches."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine

n = 30
params = np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11)
env = {k: v for k, v in os.environ.items() if k.startswith("QSB_")}
for name, circ, prec in (("var c128", q.variational_circuit(n, 5, params, fused=True), q.Precision.F64),
                         ("grid c128", q.random_grid_circuit(3, 10, 20, 42), q.Precision.F64)):
    st = q.uniform_state(n, prec)
    plan = engine.plan_for_state(st, circ.queue)
    holder = {}
    for _ in range(2):
        engine.run_plan(st, plan, holder)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        engine.run_plan(st, plan, holder)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{name}: {best:.2f} ms {env}", flush=True)
    del st
    torch.cuda.empty_cache()
