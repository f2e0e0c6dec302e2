"""Probe: identity-pass bandwidth for tiles whose contiguous low run is 128 B (L=3 c128 / L=4 c64)
vs 256 B (L=4 / L=5), and the QFT-n plan under each contiguity setting (pass count, device
time).  argv: n (default 30)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math

import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat, engine, fusion
from paper_2009_01845_b200.fusion import compile_pass, PassStep


def timed(fn, reps=5):
    fn()
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    for prec in (q.Precision.F64, q.Precision.F32):
        dt = prec.qsb_dtype
        st = q.uniform_state(n, prec)
        nbytes = 2 * (1 << n) * prec.itemsize
        geo0 = fusion.GEOMETRY[dt]
        K = geo0.K
        st_ptr = st.data_ptr
        for L in (geo0.L - 1, geo0.L, geo0.L + 2):
            shapes = {
                f"low{L}+top": set(range(L)) | set(range(n - (K - L), n)),
                f"low{L}+mid": set(range(L)) | set(range(12, 12 + K - L)),
                f"low{L}+split": set(range(L)) | set(range(8, 8 + (K - L) // 2)) | set(range(n - (K - L + 1) // 2, n)),
            }
            for name, T in shapes.items():
                words, info = compile_pass([], T, n, dt)
                step = PassStep(words, [], tuple(sorted(T)), False, 0, 0)
                ms = timed(lambda: engine._launch_pass(step, words, dt, st_ptr, st_ptr, n, nat.stream_ptr()))
                print(f"{prec.value} identity {name:14s} {ms:7.3f} ms {nbytes / ms / 1e6:8.1f} GB/s jit={step.jit is not None}",
                      flush=True)
        for L in (geo0.L - 1, geo0.L):
            fusion.GEOMETRY[dt] = fusion.TileGeometry(geo0.K, geo0.G, L)
            plan = engine.plan_for_state(st, q.qft_circuit(n).queue)
            holder = {}
            evs = []
            ms = timed(lambda: engine.run_plan(st, plan, holder))
            engine.run_plan(st, plan, holder, events=evs)
            torch.cuda.synchronize()
            per = [a.elapsed_time(b) for a, b in evs]
            print(f"{prec.value} QFT-{n} L={L}: passes={plan.n_passes} steps={len(plan.steps)} {ms:.2f} ms/circuit; "
                  f"per pass " + ", ".join(f"{x:.2f}" for x in per) + " ms  ("
                  + ", ".join(f"{nbytes / x / 1e6:.0f}" for x in per) + " GB/s)", flush=True)
            del holder
        fusion.GEOMETRY[dt] = geo0
        # correctness spot check of the L-1 plan on a basis state: QFT|k> = e^{2 pi i jk/2^n}/2^{n/2}
        fusion.GEOMETRY[dt] = fusion.TileGeometry(geo0.K, geo0.G, geo0.L - 1)
        k = 123457
        bs = q.basis_state(n, k, prec)
        out = q.qft_circuit(n).execute(bs)
        fusion.GEOMETRY[dt] = geo0
        idx = torch.tensor(np.random.default_rng(0).integers(0, 1 << n, 4096), device="cuda")
        got = out.tensor[idx].cpu().numpy()
        j = idx.cpu().numpy().astype(np.float64)
        # QFT ends with the bit-reversing SWAPs: amplitude index j holds e^{2 pi i j k / 2^n}
        ang = 2 * np.pi * ((j * k) % (1 << n)) / (1 << n)
        want = np.exp(1j * ang) / math.sqrt(1 << n)
        print(f"{prec.value} L={geo0.L - 1} QFT-{n}|{k}> max err {np.max(np.abs(got - want)):.3e}", flush=True)
        del st, out, bs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
