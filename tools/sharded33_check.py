"""SURVEY.md section 8(e)'s invariant at BASELINE config 4's size: the random 3 x 11 grid circuit
(33 qubits c128, 20 cycles) run sharded over 8 shards (in-process, the batched all-to-all
schedule) against the same circuit on the whole 137 GB state on one B200.

Both states cannot be resident at once (2 x 137 GB), so the 1-GPU state is reduced to
fingerprints first -- per 2^26-amplitude chunk f_c = sum_i w_i psi_i with w_i = e^{2 pi i
frac(i alpha)} (alpha = the golden ratio), plus 2^20 amplitudes at seeded random indices -- and
freed; the sharded state is fingerprinted the same way in its own layout (each element's
canonical index through the shards' logical qubit map), without a canonicalising copy.  Prints CHECK_OK on success.
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
idx = np.sort(np.random.default_rng(7).choice(1 << n, size=min(1 << 20, 1 << (n - 2)), replace=False))


def fingerprints(chunks):
    """Per canonical 2^26-amplitude bucket: sum of w_i psi_i over the amplitudes whose canonical
    index i falls in the bucket.  chunks: (canonical index map, device tensor) pairs covering
    the state vector; the map turns local element indices (int64 tensor) into canonical ones,
    so the buckets do not depend on the layout."""
    acc = None
    for cmap, t in chunks:
        if acc is None:
            acc = torch.zeros((1 << n) // CH, dtype=torch.complex128, device=t.device)
        for s in range(0, t.numel(), CH):
            loc = torch.arange(s, s + CH, dtype=torch.int64, device=t.device)
            ci = cmap(loc)
            ph = torch.remainder(ci.to(torch.float64) * ALPHA, 1.0) * (2 * math.pi)
            w = torch.polar(torch.ones_like(ph), ph)
            acc.index_add_(0, ci // CH, w * t[s:s + CH])
            del loc, ci, ph, w
    return {k: complex(v) for k, v in enumerate(acc.cpu().numpy())}


# 1 GPU, the whole state (137 GB at n = 33: in-place passes, SWAP-free circuit)
st = q.zero_state(n)
engine.run_gates(st, circuit.queue, None, {}, {})
torch.cuda.synchronize()
fa = fingerprints([(lambda l: l, st.tensor)])
va = st.tensor[torch.from_numpy(idx).cuda()].cpu().numpy()
norm_a = q.norm(st)
del st
torch.cuda.empty_cache()

# sharded: 8 in-process shards, batched exchanges, passes in place (as on a 137 GB shard of the
# 36-qubit target); fingerprinted in its own layout through the logical qubit map (no
# canonicalisation copy)
engine.scratch_fits = lambda nbytes: nbytes <= engine.GRID_BATCH_MAX_STATE_BYTES
plan = sd.plan_batched(circuit, shards)
sh = sd.run_sharded(circuit, shards, None, q.Precision.F64, None, sd.LocalComm(), None, {}, plan)
torch.cuda.synchronize()
g, nl = sh.n_global, sh.n_local
gq, lq = sh.global_qubits, sh.local_qubits


def shard_map(s_id):
    base = sum(((s_id >> (g - 1 - j)) & 1) << (n - 1 - q_) for j, q_ in enumerate(gq))

    def cmap(l):
        i = torch.full_like(l, base)
        for m, q_ in enumerate(lq):
            i |= ((l >> (nl - 1 - m)) & 1) << (n - 1 - q_)
        return i
    return cmap


chunks = [(shard_map(s_id), t) for s_id, t in sh.shards.items()]
fb = fingerprints(chunks)
# the sampled canonical indices in (shard, local) coordinates
s_of = np.zeros(len(idx), dtype=np.int64)
l_of = np.zeros(len(idx), dtype=np.int64)
for j, q_ in enumerate(gq):
    s_of |= ((idx >> (n - 1 - q_)) & 1) << (g - 1 - j)
for m, q_ in enumerate(lq):
    l_of |= ((idx >> (n - 1 - q_)) & 1) << (nl - 1 - m)
vb = np.empty(len(idx), dtype=np.complex128)
for s_id, t in sh.shards.items():
    sel = np.nonzero(s_of == s_id)[0]
    vb[sel] = t[torch.from_numpy(l_of[sel]).cuda()].cpu().numpy()
norm_b = sd.norm_sharded(sh)
df = max(abs(fa[k] - fb[k]) for k in fa)
dv = float(np.max(np.abs(va - vb)))
print(f"n={n} shards={shards} exchanges={plan.n_exchanges} (reference plan: {sd.plan(circuit, shards).n_reshuffles} "
      f"reshuffles) chunk fingerprints max|diff|={df:.3e} sampled amplitudes max|diff|={dv:.3e} "
      f"norms {norm_a:.15f} {norm_b:.15f} final globals {gq}", flush=True)
ok = df <= 1e-10 and dv <= 1e-12 and abs(norm_a - norm_b) <= 1e-12
print("CHECK_OK" if ok else "CHECK_FAILED", flush=True)
