"""ncu target: JIT pass kernels of QFT-n (warm the JIT cache first, then one plan run)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
prec = q.Precision.F64 if (len(sys.argv) < 3 or sys.argv[2] == "f64") else q.Precision.F32
st = q.uniform_state(n, prec)
plan = engine.plan_for_state(st, q.qft_circuit(n).queue)
engine.run_plan(st, plan)  # compiles
torch.cuda.synchronize()
engine.run_plan(st, plan)  # profiled launches
torch.cuda.synchronize()
print("done")
