"""QFT-30 c128 device time per circuit (plan resident, warm) -- run under different QSB_* env
settings to compare kernel-generation switches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine

n = 30
st = q.uniform_state(n)
plan = engine.plan_for_state(st, q.qft_circuit(n).queue)
holder = {}
for _ in range(3):
    engine.run_plan(st, plan, holder)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4):
        engine.run_plan(st, plan, holder)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / 4)
env = {k: v for k, v in os.environ.items() if k.startswith("QSB_")}
print(f"QFT-30 c128 {best:.3f} ms  {env}", flush=True)
