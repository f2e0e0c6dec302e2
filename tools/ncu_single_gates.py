"""ncu target: the stand-alone single-gate kernels (one launch per gate, fuse=False) on a 2^n
c128 state: H (general 1q body), CZPow (diagonal body, 1/4 of the state), SWAP (permutation
body, 1/2), RY (real 1q), CNOT, fSim-like Unitary (general 2q)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
st = q.uniform_state(n)
th, ph = math.pi / 2, math.pi / 6
fsim = np.array([[1, 0, 0, 0], [0, math.cos(th), -1j * math.sin(th), 0],
                 [0, -1j * math.sin(th), math.cos(th), 0], [0, 0, 0, np.exp(-1j * ph)]])
gates = [q.H(3), q.H(n - 2), q.CZPow(1, n - 1, 0.3), q.SWAP(0, n - 1), q.RY(5, 0.7), q.CNOT(2, 9),
         q.Unitary(fsim, 4, 11)]
for rep in range(2):
    for g in gates:
        q.apply_gate(st, g)
torch.cuda.synchronize()
print("done")
