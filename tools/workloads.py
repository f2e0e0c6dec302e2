"""Time the BASELINE workloads on one GPU (device time, CUDA events): variational-n (fused
layers, c128/c64), a Trotter adiabatic step, the random grid circuit, and sampling."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.fusion import PassStep


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def plan_stats(plan):
    ps = [s for s in plan.steps if isinstance(s, PassStep)]
    return f"steps={len(plan.steps)} passes={len(ps)} sweeps={plan.state_sweeps():.2f} jit={sum(1 for s in ps if s.jit)}"


def run_circuit(name, circ, n, prec):
    st = q.uniform_state(n, prec)
    t0 = time.time()
    plan = engine.plan_for_state(st, circ.queue)
    tp = time.time() - t0
    holder = {}
    ms = timed(lambda: engine.run_plan(st, plan, holder))
    sweep_bytes = 2 * (1 << n) * prec.itemsize
    evs = []
    engine.run_plan(st, plan, holder, events=evs)
    torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in evs]
    ps = [s for s in plan.steps if isinstance(s, PassStep)]
    print(f"{name:28s} n={n} {prec.value} gates={len(circ.queue)} {plan_stats(plan)} plan={tp*1e3:.0f}ms "
          f"run={ms:.2f} ms  eff={plan.state_sweeps() * sweep_bytes / ms / 1e6:.0f} GB/s", flush=True)
    print("    per pass ms: " + " ".join(f"{x:.2f}{'' if (s.jit is not None and not s.no_jit) else '(I)'}[{s.n_gates}g/{s.n_transposes}t]"
                                      for x, s in zip(per, ps)), flush=True)
    del st, holder
    torch.cuda.empty_cache()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    rng = np.random.default_rng(42)
    params = rng.uniform(0, 2 * math.pi, n * 11)
    for prec in (q.Precision.F64, q.Precision.F32):
        run_circuit("variational L5 fused", q.variational_circuit(n, 5, params, fused=True), n, prec)
        run_circuit("variational L5 unfused", q.variational_circuit(n, 5, params, fused=False), n, prec)
    h = q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5)
    run_circuit("trotter step dt=0.05", q.trotter_step_circuit(h, 0.05), n, q.Precision.F64)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from oracle import statevec as ov
    from plan_helpers import spec_tuples_to_specs

    rows = 3 if n % 3 == 0 else 2
    cols = n // rows
    grid = q.random_grid_circuit(rows, cols, 20, 42)
    run_circuit(f"grid {rows}x{cols} 20 cycles", grid, rows * cols, q.Precision.F64)
    # Trotter-form energy (EnergyCallback / CLI final_energy): 2n terms
    st = q.uniform_state(n)
    ms = timed(lambda: q.expectation(h, st), reps=2)
    from paper_2009_01845_b200.hamiltonians import _EXPECT_CACHE, _fold_single_terms

    folded = len(_fold_single_terms(h.terms))
    passes = max((len(v) for v in _EXPECT_CACHE.values()), default=folded)
    print(f"expectation <H> ({len(h.terms)} terms -> {folded} folded terms in {passes} read-only passes) n={n}: "
          f"{ms:.1f} ms ({passes * (1 << n) * 16 / ms / 1e6:.0f} GB/s of state reads)", flush=True)
    del st
    # sampling
    st = q.qft_circuit(n).execute(q.basis_state(n, 12345))
    for shots in (100000, 1000000):
        ms = timed(lambda: q.sample(st, range(n), shots, 42), reps=1)
        print(f"sample all {n} qubits {shots} shots: {ms:.1f} ms", flush=True)
    ms = timed(lambda: q.sample(st, (0, 3, 5), 100000, 42), reps=1)
    print(f"sample 3-qubit marginal 1e5 shots: {ms:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
