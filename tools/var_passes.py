"""Per-pass device times of variational-n (fused layers, L=5) with gate/transposition counts.
Run three times with QSB_JIT_PROBE unset / nogates / notransposes to split each pass's time into
gate bodies, layout changes and the memory stream (probe kernels compute wrong results)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.fusion import PassStep

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
prec = q.Precision(sys.argv[2]) if len(sys.argv) > 2 else q.Precision.F64
params = np.random.default_rng(42).uniform(0, 2 * np.pi, n * 11)
c = q.variational_circuit(n, 5, params, fused=True)
st = q.uniform_state(n, prec)
plan = engine.plan_for_state(st, c.queue)
holder = {}
for _ in range(2):
    engine.run_plan(st, plan, holder)
torch.cuda.synchronize()
evs = []
engine.run_plan(st, plan, holder, events=evs)
torch.cuda.synchronize()
per = [a.elapsed_time(b) for a, b in evs]
ps = [s for s in plan.steps if isinstance(s, PassStep)]
nbytes = 2 * (1 << n) * prec.itemsize
print(f"probe={os.environ.get('QSB_JIT_PROBE', 'full')} variational-{n} {prec.value}: {sum(per):.2f} ms")
for x, s in zip(per, ps):
    kinds = {}
    for g in s.gates:
        kinds[g.kind] = kinds.get(g.kind, 0) + 1
    geo = "x".join(str(int(w)) for w in s.words[2:4])
    print(f"  {x:6.2f} ms {nbytes / x / 1e6:5.0f} GB/s  {s.n_gates:3d}g {s.n_transposes}t {kinds} K,nreg={geo}"
          f"{' ext' if s.ext_perm else ''}")
