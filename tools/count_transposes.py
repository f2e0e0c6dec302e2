"""Layout changes (transposes) per pass of the BASELINE workloads at n = 30 (CPU only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, sys
import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat
from paper_2009_01845_b200.fusion import plan_circuit, PassStep, GEOMETRY_JIT
n = 30
circs = {"qft": q.qft_circuit(n), "var": q.variational_circuit(n, 5, np.random.default_rng(42).uniform(0, 2*np.pi, n*11), fused=True),
         "grid": q.random_grid_circuit(3, 10, 20, 42)}
terms = q.combine(q.build_x(n), 0.4, q.build_tfim(n, 1.0), 0.6)
from paper_2009_01845_b200.evolution import trotter_step_circuit
try:
    circs["trotter"] = trotter_step_circuit(terms, 0.05)
except Exception as e:
    print("trotter", e)
for name, c in circs.items():
    for dt in (nat.QSB_C128, nat.QSB_C64):
        plan = plan_circuit(c.queue, n, dt, geometry=GEOMETRY_JIT[dt])
        ps = [s for s in plan.steps if isinstance(s, PassStep)]
        print(name, dt, "passes", len(ps), "transposes", sum(s.n_transposes for s in ps), [s.n_transposes for s in ps])
