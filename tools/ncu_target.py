"""Launch sequence for ncu captures: one identity pass (pure TMA/HBM streaming) followed by
the QFT-n fused plan (argv: n, precision)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat, engine
from paper_2009_01845_b200.fusion import compile_pass

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
prec = q.Precision.F64 if (len(sys.argv) < 3 or sys.argv[2] == "f64") else q.Precision.F32
st = q.uniform_state(n, prec)
dt = prec.qsb_dtype
K = nat.lib().qsb_pass_max_tile_bits(dt)
words, _ = compile_pass([], set(range(4)) | set(range(n - K + 4, n)), n, dt)
nat.check(nat.lib().qsb_run_pass(st.data_ptr, st.data_ptr, n, dt, words.ctypes.data, len(words), nat.stream_ptr()))
plan = engine.plan_for_state(st, q.qft_circuit(n).queue)
engine.run_plan(st, plan)
torch.cuda.synchronize()
print("done", plan.n_passes)
