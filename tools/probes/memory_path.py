"""Memory-path ceiling: identity fused passes (TMA tile loads -> registers -> stores, no gates)
vs the single-gate streaming kernel (k_general1, plain loads) on the same 2^30 c128 state,
CUDA-event timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat, engine
from paper_2009_01845_b200.fusion import GEOMETRY_JIT, PassStep, compile_pass


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n = 30
st = q.uniform_state(n)
nbytes = 2 * (1 << n) * 16
dt = nat.QSB_C128
geo = GEOMETRY_JIT[dt]
K = geo.K
for name, T in [("contig", set(range(K))), ("low4+mid", set(range(4)) | set(range(14, 14 + K - 4))),
                ("low4+top", set(range(4)) | set(range(30 - (K - 4), 30))),
                ("low6+top", set(range(6)) | set(range(30 - (K - 6), 30)))]:
    words, _ = compile_pass([], T, n, dt, geo)
    step = PassStep(words, [], tuple(sorted(T)), False, 0, 0)
    ms = timed(lambda: engine._launch_pass(step, words, dt, st.data_ptr, st.data_ptr, n, nat.stream_ptr()))
    print(f"identity pass {name:10s} {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)
for g in (q.H(3), q.H(20), q.RY(29, 0.3)):
    ms = timed(lambda: q.apply_gate(st, g))
    print(f"single gate {g.kind.value}{tuple(g.targets)} {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)
x = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
ms = timed(lambda: x.copy_(st.tensor))
print(f"torch copy {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)
