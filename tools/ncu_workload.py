"""ncu target: the fused plan of one BASELINE workload, run twice (the first run compiles the
specialised pass kernels; profile the second with -s <passes> -c ...).
argv: workload (qft|variational|trotter|trotter4|grid) n precision(f64|f32)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine


def build(workload, n):
    if workload == "qft":
        return q.qft_circuit(n)
    if workload == "variational":
        params = np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11)
        return q.variational_circuit(n, 5, params, fused=True)
    if workload == "trotter":
        h = q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5)
        return q.trotter_step_circuit(h, 0.05)
    if workload == "trotter4":  # four steps as one circuit, as evolve() plans them
        h = q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5)
        step = q.trotter_step_circuit(h, 0.05)
        return q.Circuit(n).add([g for _ in range(4) for g in step.queue])
    if workload == "grid":
        rows = 3 if n % 3 == 0 else 2
        return q.random_grid_circuit(rows, n // rows, 20, 42)
    raise SystemExit(f"unknown workload {workload}")


if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "variational"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 28
    prec = q.Precision.F64 if (len(sys.argv) < 4 or sys.argv[3] == "f64") else q.Precision.F32
    st = q.uniform_state(n, prec)
    plan = engine.plan_for_state(st, build(wl, n).queue)
    engine.run_plan(st, plan)
    torch.cuda.synchronize()
    engine.run_plan(st, plan)
    torch.cuda.synchronize()
    print("done", plan.n_passes, len(plan.steps))
