"""Data-moving steps of the sharded schedules at the BASELINE multi-GPU configs: the reference
planner's single-qubit reshuffles (sharding.py:152-216) vs the batched all-to-all schedule."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import sharding as sd
from paper_2009_01845_b200.evolution import trotter_step_circuit


def trotter_steps(n, steps=20, dt=0.05):
    h0, h1 = q.build_x(n), q.build_tfim(n, 1.0)
    c = q.Circuit(n)
    for k in range(steps):
        s = min(max((k + 0.5) * dt / 1.0, 0.0), 1.0)
        c.add(list(trotter_step_circuit(q.combine(h0, 1 - s, h1, s), dt).queue))
    return c


def row(name, c, shards):
    ref = sd.plan(c, shards)
    bat = sd.plan_batched(c, shards)
    ks = [s.k for s in bat.steps if isinstance(s, sd.Exchange)]
    print(f"{name:28s} x{shards}: reference {ref.n_reshuffles:3d} reshuffles = {ref.shard_fraction_moved():6.2f} "
          f"shards sent | batched {bat.n_exchanges:3d} exchanges (k={ks[:12]}{'...' if len(ks) > 12 else ''}) = "
          f"{bat.shard_fraction_moved():6.2f} shards sent")


for shards in (2, 4, 8):
    row("QFT-33", q.qft_circuit(33), shards)
    row("grid 3x11, 20 cycles", q.random_grid_circuit(3, 11, 20, 42), shards)
    row("variational-34 L5 fused", q.variational_circuit(34, 5, np.random.default_rng(42).uniform(0, 6.28, 34 * 11),
                                                         fused=True), shards)
q.set_max_qubits(36)
for n in (34, 36):
    row(f"TFIM-{n} one Trotter step", trotter_steps(n, 1), 8)
    row(f"TFIM-{n} adiabatic, 20 steps", trotter_steps(n), 8)
