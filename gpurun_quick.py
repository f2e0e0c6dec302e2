import numpy as np, sys, time
sys.path.insert(0, '.')
import torch
import paper_2009_01845_b200 as q
from oracle import statevec as ov
for n in (13, 16):
    rng = np.random.default_rng(1)
    psi = rng.standard_normal(1<<n) + 1j*rng.standard_normal(1<<n); psi /= np.linalg.norm(psi)
    c = q.qft_circuit(n)
    t = time.time()
    got = c.execute(q.from_amplitudes(psi)).amplitudes
    print("qft", n, "err", np.max(np.abs(got - ov.run(ov.qft(n), n, psi))), "t", time.time()-t, flush=True)
    got2 = c.execute(q.from_amplitudes(psi), fuse=False).amplitudes
    print("qft unfused", n, "err", np.max(np.abs(got2 - ov.run(ov.qft(n), n, psi))), flush=True)
