"""Small-state latency: Circuit.execute below the fused-pass size (one qsb_apply_batch launch
per 64 gates, state in shared memory) against one qsb_apply_matrix launch per gate.
Usage: python tools/small_latency.py"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2009_01845_b200 as q  # noqa: E402
from paper_2009_01845_b200 import _native as nat  # noqa: E402
from paper_2009_01845_b200 import engine  # noqa: E402


def wall(fn, reps):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def main():
    for n, fused in ((6, False), (10, False), (12, False), (12, True)):
        params = np.random.default_rng(42).uniform(0, 2 * np.pi, n * 11)
        c = q.variational_circuit(n, 5, params, fused=fused)
        plan = c.plan()
        gates = [s.gate for s in plan.steps]
        st = q.zero_state(n)
        per_gate = wall(lambda: [engine._apply_gate_step(st.data_ptr, n, nat.QSB_C128, g, nat.stream_ptr())
                                 for g in gates], 20)
        batched = wall(lambda: c.execute(), 50)
        packed = engine.pack_gate_batch(gates)
        device = wall(lambda: engine._apply_gate_batch(st.data_ptr, n, nat.QSB_C128, packed, nat.stream_ptr()), 200)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        engine._apply_gate_batch(st.data_ptr, n, nat.QSB_C128, packed, nat.stream_ptr())
        ev1.record()
        torch.cuda.synchronize()
        print(f"variational n={n} L=5 fused={fused}: {len(gates)} gates; per-gate launches {per_gate:.3f} ms, "
              f"execute (batched) {batched:.3f} ms, batch call {device:.3f} ms, batch kernels {ev0.elapsed_time(ev1):.3f} ms")


def mid_sizes():
    """Fused-pass sizes: a re-executed circuit (plan cached) and a fresh parameter set each call
    (re-planned; the specialised kernels come from the source-keyed cache)."""
    for n in (14, 16, 20):
        rng = np.random.default_rng(7)
        c = q.variational_circuit(n, 5, rng.uniform(0, 2 * np.pi, n * 11), fused=True)
        t = time.perf_counter()
        c.execute()
        torch.cuda.synchronize()
        first = (time.perf_counter() - t) * 1e3
        cached = wall(lambda: c.execute(), 20)
        fresh = wall(lambda: q.variational_circuit(n, 5, rng.uniform(0, 2 * np.pi, n * 11), fused=True).execute(), 5)
        g = c.capture()
        replay = wall(lambda: g.execute(), 20)
        print(f"variational n={n} L=5 fused: passes {c.plan().n_passes}; graph replay execute {replay:.3f} ms, "
              f"first execute (grid batch) {first:.3f} ms, "
              f"execute (plan cached) {cached:.3f} ms, "
              f"new parameters each call {fresh:.3f} ms")


if __name__ == "__main__":
    mid_sizes()
    main()
