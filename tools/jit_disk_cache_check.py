"""Process-level check of the on-disk cubin cache: the first process compiles, the second loads."""
import os
import subprocess
import sys
import tempfile
import time

code = r'''
import sys, time, numpy as np
sys.path.insert(0, %r)
import torch
import paper_2009_01845_b200 as q
c = q.variational_circuit(24, 2, np.random.default_rng(1).uniform(0, 6, 24 * 5), fused=True)
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
from paper_2009_01845_b200 import engine
engine.prepare_plan(24, q.Precision.F64, c.queue, None, {})
torch.cuda.synchronize()
print("prepare", round(time.perf_counter() - t, 2))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with tempfile.TemporaryDirectory() as d:
    env = dict(os.environ, QSB_JIT_CACHE_DIR=d)
    for k in range(2):
        out = subprocess.run([sys.executable, "-c", code % root], env=env, capture_output=True, text=True)
        print(f"process {k}: {out.stdout.strip()} {out.stderr.strip()[-300:]}")
    print("cached cubins:", sum(len(f) for _, _, f in os.walk(d)))
