"""Device time of each 4-step window of adiabatic_evolve (n = 30 TFIM, 20 steps), plan
templates on vs off, with per-pass times of one window and the template counters."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine, fusion, jit

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
if len(sys.argv) > 2:
    from paper_2009_01845_b200 import evolution

    evolution.STEP_WINDOW = int(sys.argv[2])
orig = engine.run_plan
records = []


def timed(state, plan, holder=None, stream=None, events=None):
    evs = []
    orig(state, plan, holder, stream, evs)
    records.append((plan, evs))


engine.run_plan = timed
cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.05, 1.0)
for use in (True, True):
    fusion.PLAN_TEMPLATES = use
    jit.RECIPES = use
    q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 0.9), q.Schedule.linear(), cfg)
    torch.cuda.synchronize()
    records.clear()
    s0 = dict(fusion.TEMPLATE_STATS)
    t0 = time.perf_counter()
    q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 1.0), q.Schedule.linear(), cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    per = [sum(a.elapsed_time(b) for a, b in evs) for _, evs in records]
    d = {k: fusion.TEMPLATE_STATS[k] - s0[k] for k in s0}
    print(f"templates {use}: wall {wall * 1e3:.0f} ms, windows (device ms) {[round(x, 1) for x in per]}, template {d}",
          flush=True)
    plan, evs = records[2]
    ps = [s for s in plan.steps if isinstance(s, fusion.PassStep)]
    for s, (a, b) in zip(ps, evs):
        print(f"   {a.elapsed_time(b):6.2f} ms len {len(s.words)} flags {int(s.words[7])} nreg {int(s.words[3])} "
              f"kernel {s.jit[0].name if s.jit else None} cost {sum(fusion.matrix_cost(g.matrix) for g in s.gates if g.kind in ('g1', 'g2'))}",
              flush=True)
