"""Bit-permuting copy at n = 30 c128 (17 GB): the QFT's bit reversal and a random permutation,
device time per call and GB/s (read + write)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200.sharding import CudaBackend

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
be = CudaBackend(q.Precision.F64)
src = q.uniform_state(n).tensor
for name, perm in [("reversal", list(range(n))[::-1]), ("random", [int(x) for x in np.random.default_rng(1).permutation(n)]),
                   ("identity", list(range(n)))]:
    out = be.permute(src, n, perm)
    del out
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = be.permute(src, n, perm)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"permute {name} n={n}: {ms:.2f} ms, {2 * (1 << n) * 16 / ms / 1e6:.0f} GB/s", flush=True)
    del out
