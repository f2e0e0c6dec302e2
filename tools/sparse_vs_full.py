import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import measurement as M
n = 30
st = q.qft_circuit(n).execute(q.basis_state(n, 12345))
for shots in (100000, 300000, 1000000, 3000000):
    for mode in ("sparse", "full"):
        def run():
            probs = M.device_marginal(st, tuple(range(n)))
            if mode == "sparse":
                return M.device_sample_exact(probs, shots, 42)
            cum = M.device_cdf(probs); del probs
            return M.device_sample(cum, shots, 42)
        r = run(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter(); r = run(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
        print(shots, mode, f"{best*1e3:.1f} ms", int(r.sum().item()) % 1000003, flush=True)
