"""Debug aid: batch vs per-gate kernels, per-gate divergence (python tools/batch_diff.py n prec)."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import paper_2009_01845_b200 as q  # noqa: E402
from paper_2009_01845_b200 import _native as nat  # noqa: E402
from paper_2009_01845_b200 import engine  # noqa: E402
from paper_2009_01845_b200.fusion import normalize  # noqa: E402
from test_gpu_parity import _random_spec  # noqa: E402

n, prec = int(sys.argv[1]), sys.argv[2]
rng = np.random.default_rng(1000 + n)
specs = [_random_spec(q, n, rng) for _ in range(150)]
ngates = [g for g in (normalize(s, n, i) for i, s in enumerate(specs)) if g is not None]
psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
precision = q.Precision(prec)
a = q.from_amplitudes(psi, precision=precision)
b = q.from_amplitudes(psi, precision=precision)
for k, g in enumerate(ngates):
    engine._apply_gate_batch(a.data_ptr, n, precision.qsb_dtype, engine.pack_gate_batch([g]), nat.stream_ptr())
    engine._apply_gate_step(b.data_ptr, n, precision.qsb_dtype, g, nat.stream_ptr())
    d = np.max(np.abs(a.amplitudes - b.amplitudes))
    if d:
        print(k, g.kind, g.targets, g.controls, "max diff", d)
        print(np.round(g.matrix, 3))
        break
else:
    print("all", len(ngates), "gates equal")
