"""Per-pass device times at n = 33 complex128 (137 GB, no room for an out-of-place scratch: the
per-GPU shard size of the 36-qubit / 8-GPU target): QFT-33, the 3x11 grid (BASELINE config 4's
circuit) and one TFIM Trotter step, with each pass's tile bits, next to an identity pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.fusion import GateStep, PassStep

q.set_max_qubits(36)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
which = sys.argv[2:] or ["qft", "trotter", "grid"]
sweep = 2 * (1 << n) * 16
st = q.uniform_state(n)
_step = q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)
# trotter4: four steps as one circuit, as evolve() plans them (evolution.STEP_WINDOW)
circs = {"qft": q.qft_circuit(n), "trotter": _step, "grid": q.random_grid_circuit(3, n // 3, 20, 42)}
for _w in (2, 4, 6, 8):  # trotterK: K steps as one circuit
    circs[f"trotter{_w}"] = q.Circuit(n).add([g for _ in range(_w) for g in _step.queue])
for name in which:
    if name == "qft-api":
        # through Circuit.execute's engine.run_gates: no room for a scratch buffer, so the
        # SWAPs become a qubit relabelling kept on the state; the canonical read is timed apart
        circ = circs["qft"]
        cache, holder = {}, {}
        engine.run_gates(st, circ.queue, None, holder, cache)
        st._canonicalize()
        torch.cuda.synchronize()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        plan = engine.run_gates(st, circ.queue, None, holder, cache)
        b.record()
        st._canonicalize()
        c.record()
        torch.cuda.synchronize()
        print(f"qft-{n} via run_gates: {a.elapsed_time(b):.1f} ms ({plan.n_passes} passes, {len(plan.steps)} steps, "
              f"SWAPs as relabels); canonical read (in-place SWAP kernels) {b.elapsed_time(c):.1f} ms", flush=True)
        continue
    circ = circs[name]
    plan = engine.plan_for_state(st, circ.queue)
    holder = {}
    engine.run_plan(st, plan, holder)
    torch.cuda.synchronize()
    evs = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    engine.run_plan(st, plan, holder, events=evs)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    ps = [s for s in plan.steps if isinstance(s, PassStep)]
    gs = [s for s in plan.steps if isinstance(s, GateStep)]
    print(f"{name}-{n}: {ms:.1f} ms, {len(ps)} passes + {len(gs)} gate steps, sweeps {plan.state_sweeps():.1f}, "
          f"eff {plan.state_sweeps() * sweep / ms / 1e6:.0f} GB/s" + (f", {ms / int(name[7:]):.1f} ms per step" if name.startswith("trotter") and name[7:] else ""),
          flush=True)
    for x, s in zip([a_.elapsed_time(b_) for a_, b_ in evs], ps):
        print(f"   {x:8.2f} ms  {sweep / x / 1e6:6.0f} GB/s  gates={s.n_gates:3d} tr={s.n_transposes} ext={int(s.ext_perm)} "
              f"tile={list(s.tile_pos)}", flush=True)
