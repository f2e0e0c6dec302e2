"""A window of four time-dependent Trotter steps planned from a template vs planned afresh:
same passes?  same device time?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine, evolution, fusion, jit

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
h0, h1 = q.build_x(n), q.build_tfim(n, 1.0)


def window(s0, hz=1.0):
    hh = q.build_tfim(n, hz)
    c = q.Circuit(n)
    for j in range(4):
        s = s0 + j * 0.05
        c.add(list(evolution.trotter_step_circuit(q.combine(h0, 1 - s, hh, s), 0.05).queue))
    return c


st = q.uniform_state(n)
A, B = window(0.3, 0.9), window(0.5)
fusion.PLAN_TEMPLATES = False
fresh = engine.plan_for_state(st, B.queue)
fusion.PLAN_TEMPLATES = True
engine.plan_for_state(st, A.queue)
tpl = engine.plan_for_state(st, B.queue)
print("template stats", fusion.TEMPLATE_STATS, "recipes", jit.RECIPE_STATS)
pf = [s for s in fresh.steps if isinstance(s, fusion.PassStep)]
pt = [s for s in tpl.steps if isinstance(s, fusion.PassStep)]
print("passes fresh", len(pf), "template", len(pt))
for i, (a, b) in enumerate(zip(pf, pt)):
    same_len = len(a.words) == len(b.words)
    ka = jit.coefficients_only(a.words, 1)[0]
    kb = jit.coefficients_only(b.words, 1)[0]
    ca = sum(fusion.matrix_cost(g.matrix) for g in a.gates if g.kind in ("g1", "g2"))
    cb = sum(fusion.matrix_cost(g.matrix) for g in b.gates if g.kind in ("g1", "g2"))
    kj = b.jit[0].name if b.jit else None
    print(f"pass {i}: len {len(a.words)}/{len(b.words)} same-structure {ka == kb} cost {ca}/{cb} "
          f"kernel fresh {a.jit[0].name if a.jit else None} tpl {kj}")


def t(plan):
    holder = {}
    engine.run_plan(st, plan, holder)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(3):
        engine.run_plan(st, plan, holder)
    ev1.record()
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / 3


for _ in range(2):
    print(f"fresh {t(fresh):.2f} ms  template {t(tpl):.2f} ms")
