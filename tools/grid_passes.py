"""Per-pass device times of the random grid circuit (3 x n/3, 20 cycles, c128) with gate kinds,
layout changes and kernel geometry; run with QSB_JIT_PROBE=nogates|notransposes|nostores to
split the time (probe kernels compute wrong results)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.fusion import PassStep

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
c = q.random_grid_circuit(3, n // 3, 20, 42)
st = q.uniform_state(n)
plan = engine.plan_for_state(st, c.queue)
holder = {}
engine.run_plan(st, plan, holder)
torch.cuda.synchronize()
evs = []
engine.run_plan(st, plan, holder, events=evs)
torch.cuda.synchronize()
per = [a.elapsed_time(b) for a, b in evs]
ps = [s for s in plan.steps if isinstance(s, PassStep)]
print(f"probe={os.environ.get('QSB_JIT_PROBE', 'full')} grid-{n}: {sum(per):.1f} ms in {len(ps)} passes "
      f"({len(plan.steps) - len(ps)} stand-alone gates)")
rows = []
for x, s in zip(per, ps):
    kinds = {}
    for g in s.gates:
        kinds[g.kind] = kinds.get(g.kind, 0) + 1
    rows.append(f"{x:.2f}[{s.n_gates}g/{s.n_transposes}t {kinds.get('g2', 0)}x2q]")
print("  " + " ".join(rows))
