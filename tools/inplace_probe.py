"""Why a plan's run differs from the sum of its passes timed alone: per-pass times inside
run_plan (events), the same pass programs launched in place (src = dst) and out of place."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat
from paper_2009_01845_b200 import engine, fusion, jit

n = 30
step = q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)
circ = q.Circuit(n).add([g for _ in range(4) for g in step.queue])
st = q.uniform_state(n, q.Precision.F64)
plan = engine.plan_for_state(st, circ.queue)
holder: dict = {}
for _ in range(2):
    engine.run_plan(st, plan, holder)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    engine.run_plan(st, plan, holder)
b.record()
torch.cuda.synchronize()
print(f"run_plan: {a.elapsed_time(b) / 3:.2f} ms per 4 steps", flush=True)
evs: list = []
engine.run_plan(st, plan, holder, events=evs)
torch.cuda.synchronize()
inplan = [x.elapsed_time(y) for x, y in evs]
src = st.raw_tensor
dst = torch.empty_like(src)
stream = torch.cuda.current_stream().cuda_stream
passes = [s for s in plan.steps if isinstance(s, fusion.PassStep)]


def t(words, s, d, reps=3):
    c, co = jit.compile_words(words, nat.QSB_C128)
    jit.run(words, nat.QSB_C128, s, d, n, stream, c, co)
    a.record()
    for _ in range(reps):
        jit.run(words, nat.QSB_C128, s, d, n, stream, c, co)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


tot = [0.0, 0.0, 0.0]
for i, p in enumerate(passes):
    ip = t(p.words, src.data_ptr(), src.data_ptr()) if not p.ext_perm else float("nan")
    op = t(p.words, src.data_ptr(), dst.data_ptr())
    tot[0] += inplan[i]
    tot[1] += ip if ip == ip else op
    tot[2] += op
    print(f"pass {i:2d} ext {int(p.ext_perm)} in-plan {inplan[i]:6.3f}  alone in-place {ip:6.3f}  alone out-of-place {op:6.3f}", flush=True)
print("sums: in-plan %.2f  in-place %.2f  out-of-place %.2f" % tuple(tot))
