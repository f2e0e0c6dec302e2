"""Micro-probe of the fused pass kernel: identity passes with different tile shapes (memory
path only) vs the real QFT passes (memory + compute).  Prints ms and GB/s per launch."""

import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat, engine
from paper_2009_01845_b200.fusion import compile_pass, plan_circuit, PassStep


def time_words(state, words, reps=5, step=None):
    lib = nat.lib()
    st = nat.stream_ptr()
    n = state.n_qubits
    dt = state.precision.qsb_dtype

    def launch():
        if step is not None:
            engine._launch_pass(step, words, dt, state.data_ptr, state.data_ptr, n, st)
        else:
            nat.check(lib.qsb_run_pass(state.data_ptr, state.data_ptr, n, dt, words.ctypes.data, len(words), st))

    for _ in range(2):
        launch()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        launch()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    for prec in (q.Precision.F64, q.Precision.F32):
        st = q.uniform_state(n, prec)
        dt = prec.qsb_dtype
        nbytes = 2 * (1 << n) * prec.itemsize
        K = nat.lib().qsb_pass_max_tile_bits(dt)
        L = 4 if prec is q.Precision.F64 else 5
        shapes = {
            "contig": set(range(K)),
            "low+top": set(range(L)) | set(range(n - (K - L), n)),
            "low+mid": set(range(L)) | set(range(10, 10 + K - L)),
            "low6+top": set(range(6)) | set(range(n - (K - 6), n)),
        }
        for name, T in shapes.items():
            words, info = compile_pass([], T, n, dt)
            ms = time_words(st, words, step=PassStep(words, [], tuple(sorted(T)), False, 0, 0))
            print(f"{prec.value} identity {name:9s} {ms:7.3f} ms  {nbytes / ms / 1e6:8.1f} GB/s", flush=True)
        plan = plan_circuit(q.qft_circuit(n).queue, n, dt)
        for i, s in enumerate(plan.steps):
            if isinstance(s, PassStep) and not s.ext_perm:
                ms = time_words(st, s.words)
                mj = time_words(st, s.words, step=s)
                print(f"{prec.value} qft pass {i} gates={s.n_gates} piv={s.n_pivots} tr={s.n_transposes} "
                      f"interp {ms:7.3f} ms {nbytes / ms / 1e6:7.1f} GB/s | jit {mj:7.3f} ms {nbytes / mj / 1e6:7.1f} GB/s",
                      flush=True)
        del st
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
