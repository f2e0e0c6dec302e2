"""complex64 energy at n: fused expectation passes vs the per-term kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import hamiltonians as hm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = q.uniform_state(n, q.Precision.F32)
h = q.combine(q.build_x(n), 0.4, q.build_tfim(n, 1.0), 0.6)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        v = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, v


fused = timed(lambda: q.expectation(h, st))
orig = hm._expectation_passes
hm._expectation_passes = lambda *a: None
per_term = timed(lambda: q.expectation(h, st))
hm._expectation_passes = orig
print(f"c64 energy n={n}: fused {fused[0]:.1f} ms ({fused[1]:.9f}), per-term {per_term[0]:.1f} ms ({per_term[1]:.9f})")
