"""Per-pass device times of the QFT-n plan (c128 and c64) with the default JIT geometry."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.fusion import PassStep

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for prec in (q.Precision.F64, q.Precision.F32):
    st = q.uniform_state(n, prec)
    plan = engine.plan_for_state(st, q.qft_circuit(n).queue)
    holder = {}
    for _ in range(3):
        engine.run_plan(st, plan, holder)
    torch.cuda.synchronize()
    evs = []
    engine.run_plan(st, plan, holder, events=evs)
    torch.cuda.synchronize()
    nbytes = 2 * (1 << n) * prec.itemsize
    per = [a.elapsed_time(b) for a, b in evs]
    ps = [s for s in plan.steps if isinstance(s, PassStep)]
    print(f"QFT-{n} {prec.value}: {sum(per):.2f} ms, passes " + ", ".join(
        f"{x:.2f} ms ({nbytes / x / 1e6:.0f} GB/s, {s.n_gates}g/{s.n_transposes}t{'/ext' if s.ext_perm else ''})"
        for x, s in zip(per, ps)), flush=True)
    del st, holder
    torch.cuda.empty_cache()
