"""ncu / timing target: sample(all n qubits) and a 3-qubit marginal on a QFT-n state (argv n)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
st = q.qft_circuit(n).execute(q.basis_state(n, 12345))
for _ in range(2):
    q.sample(st, range(n), 100000, 42)
    q.sample(st, (0, 3, 5), 100000, 42)
torch.cuda.synchronize()
print("done")
