"""SURVEY.md section 8(e)'s invariant at BASELINE config 4's size: the random 3 x 11 grid circuit
(33 qubits c128, 20 cycles) run sharded over 8 shards (in-process, the batched all-to-all
schedule) against the same circuit on the whole 137 GB state on one B200.

Both states cannot be resident at once (2 x 137 GB), so the 1-GPU state is reduced to
fingerprints first -- per 2^26-amplitude chunk f_c = sum_i w_i psi_i with w_i = e^{2 pi i
frac(i alpha)} (alpha = the golden ratio), plus 2^20 amplitudes at seeded random indices -- and
freed; the sharded state is canonicalised (global qubits 0..2, locals in order: shard c is then
the c-th slice of the state vector) and fingerprinted the same way.  Prints CHECK_OK on success.
argv: n (33), shards (8), cycles (20)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine
from paper_2009_01845_b200 import sharding as sd

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 20
q.set_max_qubits(max(n, q.max_qubits()))
CH = 1 << min(26, n - 3)
ALPHA = (math.sqrt(5.0) - 1.0) / 2.0
rows = 3 if n % 3 == 0 else 2
circuit = q.random_grid_circuit(rows, n // rows, cycles, 42)
idx = np.sort(np.random.default_rng(7).choice(1 << n, size=1 << 20, replace=False))


def fingerprints(chunks):
    """chunks: iterable of (global offset, device tensor) covering the canonical vector."""
    out = {}
    for off, t in chunks:
        for s in range(0, t.numel(), CH):
            i = torch.arange(off + s, off + s + CH, dtype=torch.float64, device=t.device)
            ph = torch.remainder(i * ALPHA, 1.0) * (2 * math.pi)
            w = torch.polar(torch.ones_like(ph), ph)
            out[off + s] = complex((w * t[s:s + CH]).sum().item())
            del i, ph, w
    return out


def samples(chunks):
    vals = np.empty(len(idx), dtype=np.complex128)
    for off, t in chunks:
        sel = np.nonzero((idx >= off) & (idx < off + t.numel()))[0]
        if len(sel):
            vals[sel] = t[torch.from_numpy(idx[sel] - off).to(t.device)].cpu().numpy()
    return vals


# 1 GPU, the whole state (137 GB at n = 33: in-place passes, SWAP-free circuit)
st = q.zero_state(n)
engine.run_gates(st, circuit.queue, None, {}, {})
torch.cuda.synchronize()
fa, va = fingerprints([(0, st.tensor)]), samples([(0, st.tensor)])
norm_a = q.norm(st)
del st
torch.cuda.empty_cache()

# sharded: 8 in-process shards, batched exchanges
plan = sd.plan_batched(circuit, shards)
sh = sd.run_sharded(circuit, shards, None, q.Precision.F64, None, sd.LocalComm(), None, {}, plan)
torch.cuda.synchronize()
sd.canonicalize(sh)
torch.cuda.synchronize()
nl = sh.n_local
order = sd._canonical_shard_ids(sh)
chunks = [(c << nl, sh.shards[s_id]) for c, s_id in enumerate(order)]
fb, vb = fingerprints(chunks), samples(chunks)
norm_b = sd.norm_sharded(sh)
df = max(abs(fa[k] - fb[k]) for k in fa)
dv = float(np.max(np.abs(va - vb)))
print(f"n={n} shards={shards} exchanges={plan.n_exchanges} (reference plan: {sd.plan(circuit, shards).n_reshuffles} "
      f"reshuffles) chunk fingerprints max|diff|={df:.3e} sampled amplitudes max|diff|={dv:.3e} "
      f"norms {norm_a:.15f} {norm_b:.15f}", flush=True)
ok = df <= 1e-10 and dv <= 1e-12 and abs(norm_a - norm_b) <= 1e-12
print("CHECK_OK" if ok else "CHECK_FAILED", flush=True)
