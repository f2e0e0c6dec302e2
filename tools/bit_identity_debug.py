import os, sys, math
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
engine.FUSION_DEFAULT = False
n = 20
rng = np.random.default_rng(31)
psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
def sv(p): return q.StateVector(n, torch.from_numpy(p).cuda(), q.Precision.F64) if hasattr(q, "StateVector") else None
from paper_2009_01845_b200.state import upload
def mk(): return q.StateVector(n, upload(psi.copy()), q.Precision.F64)
circuits = {"qft": q.qft_circuit(n), "var": q.variational_circuit(n, 2, rng.uniform(0, 6, n * 5), fused=True), "grid": q.random_grid_circuit(4, 5, 6, 3)}
for name, c in circuits.items():
    a = c.execute(mk()).amplitudes
    b = q.execute_sharded(c, 2, initial=mk()).amplitudes
    print(name, "equal" if np.array_equal(a, b) else f"diff {np.max(np.abs(a-b)):.2e}", flush=True)
    if not np.array_equal(a, b):
        gates = list(c.queue)
        lo, hi = 1, len(gates)
        while lo < hi:
            mid = (lo + hi) // 2
            cc = q.Circuit(n).add(gates[:mid])
            x = cc.execute(mk()).amplitudes; y = q.execute_sharded(cc, 2, initial=mk()).amplitudes
            if np.array_equal(x, y): lo = mid + 1
            else: hi = mid
        g = gates[lo - 1]
        print("  first differing prefix length", lo, "gate", g.kind, g.targets, g.controls, getattr(g, "params", None), flush=True)
