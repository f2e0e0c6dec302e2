"""Device-synchronised time of exact sampling on a QFT-n state (argv n, default 30): all qubits
1e5 / 1e6 shots and a 3-qubit marginal, plus a digest of the samples (equal across builds)."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = q.qft_circuit(n).execute(q.basis_state(n, 12345))
for qubits, shots in ((range(n), 100000), (range(n), 1000000), ((0, 3, 5), 100000)):
    res = q.sample(st, qubits, shots, 42)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        res = q.sample(st, qubits, shots, 42)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    dig = hashlib.sha1(np.ascontiguousarray(np.asarray(res.samples)).tobytes()).hexdigest()[:12]
    print(f"n={n} qubits={len(list(qubits))} shots={shots}: {best * 1e3:.1f} ms digest {dig}", flush=True)
