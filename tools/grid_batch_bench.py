"""Device time of qsb_apply_batch (grid-synchronised walk) per gate at several state sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat
from paper_2009_01845_b200 import engine

for n in (14, 16, 18, 20, 22, 24):
    c = q.variational_circuit(n, 5, np.random.default_rng(1).uniform(0, 6, n * 11), fused=False)
    st = q.uniform_state(n)
    packed = engine.pack_specs(c.queue, n)
    for _ in range(2):
        engine._apply_gate_batch(st.data_ptr, n, nat.QSB_C128, packed, nat.stream_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        engine._apply_gate_batch(st.data_ptr, n, nat.QSB_C128, packed, nat.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    g = len(c.queue)
    print(f"n={n}: {g} gates {ms:.3f} ms = {1e3 * ms / g:.2f} us/gate "
          f"({2 * (1 << n) * 16 * g / ms / 1e6:.0f} GB/s of gate sweeps)", flush=True)
