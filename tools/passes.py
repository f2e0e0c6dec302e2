"""Per-pass device times of a BASELINE workload plan (argv: workload n [f64|f32]) with kernel
geometry (register bits), gate count, layout changes and the gate-code estimate per thread."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.fusion import PassStep, matrix_cost
from ncu_workload import build

wl = sys.argv[1] if len(sys.argv) > 1 else "trotter"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
prec = q.Precision(sys.argv[3]) if len(sys.argv) > 3 else q.Precision.F64
st = q.uniform_state(n, prec)
plan = engine.plan_for_state(st, build(wl, n).queue)
holder = {}
engine.run_plan(st, plan, holder)
torch.cuda.synchronize()
runs = []
for _ in range(3):
    evs = []
    engine.run_plan(st, plan, holder, events=evs)
    torch.cuda.synchronize()
    runs.append([a.elapsed_time(b) for a, b in evs])
per = [sorted(x)[1] for x in zip(*runs)]  # median of three
ps = [s for s in plan.steps if isinstance(s, PassStep)]
print(f"{wl}-{n} {prec.value}: {sum(per):.2f} ms in {len(ps)} passes")
for x, s in zip(per, ps):
    code = sum(matrix_cost(g.matrix) for g in s.gates if g.kind in ("g1", "g2")) * (1 << int(s.words[3]))
    print(f"  {x:6.2f} ms  nreg={int(s.words[3])} {s.n_gates:3d}g {s.n_transposes}t code/thread~{code:.0f}")
