"""Randomised check of the planner + specialised kernels: random circuits (dense 1/2-qubit
unitaries, controlled 2-qubit unitaries, controlled rotations, phase gates, SWAPs, CZ / CNOT, repeated structures with fresh
parameters for the plan templates) at n = 20-23, fused passes vs per-gate kernels, complex128
(<= 1e-12) and complex64 (<= 1e-5).  argv: number of circuits (default 40)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200.verify import max_abs_diff

engine.FIRST_RUN_BATCH = False
count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
worst = {"f64": 0.0, "f32": 0.0}
for trial in range(count):
    rng = np.random.default_rng(1000 + trial)
    n = int(rng.integers(20, 24))
    layout = [(int(rng.integers(9)), int(rng.integers(n - 2)), int(rng.integers(n))) for _ in range(int(rng.integers(40, 160)))]
    for rep in range(2):  # the same structure twice: the second plan comes from the template
        r = np.random.default_rng(trial * 7 + rep)
        c = q.Circuit(n)
        for kind, a, b in layout:
            if kind == 0:
                u, _ = np.linalg.qr(r.standard_normal((4, 4)) + 1j * r.standard_normal((4, 4)))
                c.add(q.Unitary(u, a, a + 1))
            elif kind == 1:
                u, _ = np.linalg.qr(r.standard_normal((2, 2)) + 1j * r.standard_normal((2, 2)))
                c.add(q.Unitary(u, a))
            elif kind == 2 and b != a:
                c.add(q.RX(a, float(r.uniform(0, 6)), controls=(b,)))
            elif kind == 3:
                c.add(q.CZPow(a, a + 1, float(r.uniform(0, 1))))
            elif kind == 4:
                c.add(q.SWAP(a, (a + 5) % n))
            elif kind == 5:
                c.add(q.CZ(a, (a + 2) % n))
            elif kind == 6:
                c.add(q.CNOT(a, (a + 1) % n))
            elif kind == 7 and b not in (a, a + 1):
                u, _ = np.linalg.qr(r.standard_normal((4, 4)) + 1j * r.standard_normal((4, 4)))
                c.add(q.Unitary(u, a, a + 1, controls=(b,)))
            else:
                c.add(q.RZ(a, float(r.uniform(0, 6))))
        for prec, tol in (("f64", 1e-12), ("f32", 1e-5)):
            p = q.Precision(prec)
            start = q.uniform_state(n, p)
            a_ = c.execute(start, precision=p)
            b_ = c.execute(start, precision=p, fuse=False)
            err = max_abs_diff(a_.tensor, b_.tensor)
            worst[prec] = max(worst[prec], err)
            if err > tol:
                print(f"FAIL trial {trial} rep {rep} n={n} {prec}: {err:.3e}", flush=True)
                sys.exit(1)
            del a_, b_, start
    torch.cuda.empty_cache()
print(f"FUZZ_OK {count} structures x 2 parameter sets; worst |fused - per-gate| f64 {worst['f64']:.2e}, "
      f"f32 {worst['f32']:.2e}", flush=True)
