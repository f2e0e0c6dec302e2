"""Largest single-GPU states: QFT-33 c128 (137 GB, no room for an out-of-place scratch -> the
final SWAPs run as in-place half-sweeps) and the 3x11 random grid (BASELINE config 4's circuit
on one B200), device time per circuit."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.fusion import PassStep, GateStep

q.set_max_qubits(36)
n = 33
for name, circ in [("QFT-33 c128", q.qft_circuit(n)), ("grid 3x11 20 cycles c128", q.random_grid_circuit(3, 11, 20, 42))]:
    st = q.uniform_state(n)
    plan = engine.plan_for_state(st, circ.queue)
    holder = {}
    engine.run_plan(st, plan, holder)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    engine.run_plan(st, plan, holder)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    sweeps = plan.state_sweeps()
    print(f"{name}: {ms:.1f} ms, passes={sum(isinstance(s, PassStep) for s in plan.steps)} "
          f"gate steps={sum(isinstance(s, GateStep) for s in plan.steps)} sweeps={sweeps:.1f} "
          f"eff {sweeps * 2 * (1 << n) * 16 / ms / 1e6:.0f} GB/s, norm {q.norm(st):.12f}", flush=True)
    del st, holder
    torch.cuda.empty_cache()
