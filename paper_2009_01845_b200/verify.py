"""Size-independent checks of device states: used by bench.py to verify
the state it times and by the CLI's --verify at sizes the CPU cannot reach.  Everything runs on
the device in chunks; nothing here is a CPU fallback of a kernel.

* `dft_column_error`: QFT(n)|k> = sum_j e^{2 pi i jk / 2^n} / 2^{n/2} |j> -- the reference's own
  known-answer test (/root/reference/pkg/tests/test_circuit.py:189-201), exact for any n;
* `max_abs_diff`: max |a - b| of two device states (fused passes vs per-gate kernels, sharded vs
  single-GPU)."""

from __future__ import annotations

import math

from . import _native as nat

CHUNK = 1 << 26


def dft_column_error(state, k: int, chunk: int = CHUNK) -> float:
    """max_j |psi_j - e^{2 pi i jk / 2^n} / 2^{n/2}| (j*k mod 2^n in exact int64 arithmetic, the
    phase and the exponential in float64)."""
    torch = nat.torch_mod()
    n = state.n_qubits
    t = state.tensor
    dim = 1 << n
    amp = 1.0 / math.sqrt(dim)
    worst = torch.zeros((), dtype=torch.float64, device=t.device)
    for s in range(0, dim, chunk):
        j = torch.arange(s, min(dim, s + chunk), dtype=torch.int64, device=t.device)
        ph = ((j * k) % dim).to(torch.float64) * (2.0 * math.pi / dim)
        want = torch.polar(torch.full_like(ph, amp), ph)
        worst = torch.maximum(worst, (t[s:s + chunk].to(torch.complex128) - want).abs().max())
    return float(worst.item())


def max_abs_diff(a, b, chunk: int = CHUNK) -> float:
    """max |a_i - b_i| of two device tensors (or StateVectors) of the same length."""
    torch = nat.torch_mod()
    a = getattr(a, "tensor", a)
    b = getattr(b, "tensor", b)
    worst = torch.zeros((), dtype=torch.float64, device=a.device)
    for s in range(0, a.numel(), chunk):
        d = (a[s:s + chunk].to(torch.complex128) - b[s:s + chunk].to(torch.complex128)).abs().max()
        worst = torch.maximum(worst, d)
    return float(worst.item())
