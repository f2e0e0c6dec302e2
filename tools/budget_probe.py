"""Measured device time of plans with a per-pass FP-work cap (fusion._plan_passes fp_budget)
against the greedy plan, for the n = 30 workloads: is spreading gate arithmetic over the passes
worth it?"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat
from paper_2009_01845_b200 import engine, fusion, jit

n = 30
params = np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11)
step = q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)
cases = [("var c128", q.variational_circuit(n, 5, params, fused=True), q.Precision.F64),
         ("var c64", q.variational_circuit(n, 5, params, fused=True), q.Precision.F32),
         ("grid c128", q.random_grid_circuit(3, 10, 20, 42), q.Precision.F64),
         ("trotter4 c128", q.Circuit(n).add([g for _ in range(4) for g in step.queue]), q.Precision.F64)]
only = os.environ.get("ONLY")
for name, circ, prec in cases:
    if only and only not in name:
        continue
    dt = prec.qsb_dtype
    geo = engine.default_geometry(dt)
    gates = [g for g in (fusion.normalize(s, n, i) for i, s in enumerate(circ.queue)) if g is not None]
    base = fusion.sandwich_diagonals(fusion.merge_1q_runs(gates))
    st = q.uniform_state(n, prec)
    for slack in [float(x) for x in os.environ.get("SLACKS", "0,4").split(",")]:
        cand = fusion.merge_2q_runs(fusion.merge_single_qubit(base, slack))
        for budget in [None] + [float(x) for x in os.environ.get("BUDGETS", "128,96,80,72").split(",")]:
            plan = fusion._plan_passes(fusion.Plan(n, dt), cand, n, dt, geo, True, None, fp_budget=budget)
            steps = [s for s in plan.steps if isinstance(s, fusion.PassStep)]
            jit.precompile(steps, dt)
            holder = {}
            engine.run_plan(st, plan, holder)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                engine.run_plan(st, plan, holder)
            b.record()
            torch.cuda.synchronize()
            costs = [round(sum(fusion.matrix_cost(g.matrix) for g in s.gates if g.kind in ("g1", "g2"))) for s in steps]
            print(f"{name} slack {slack} budget {budget}: {a.elapsed_time(b) / 3:.2f} ms, {len(steps)} passes, "
                  f"est {fusion.plan_estimate(plan):.2f}, costs {costs}", flush=True)
    del st
    torch.cuda.empty_cache()
