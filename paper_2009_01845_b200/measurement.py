"""Shot sampling on the device (drop-in for /root/reference/pkg/src/qsim/measurement.py).

Pipeline, every stage a qsb200 kernel and bit-compatible with the reference's numpy path
(SURVEY.md Appendix B):
  qsb_probabilities   |a|^2 with numpy's complex-abs formula          (measurement.py:50)
  qsb_marginal        numpy's add.reduce order over unmeasured qubits  (measurement.py:52-58)
  qsb_cumsum_normalized  the exact sequential cumsum, in parallel      (measurement.py:81-82)
  qsb_sample          PCG64 draws + searchsorted(side="right") + clip  (measurement.py:83-86)
The generator state is seeded on the host exactly as numpy.random.default_rng(seed) does
(numpy's PCG64 seeding is used for the 128-bit (state, inc) pair only; all draws are made
on the device with jump-ahead).
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ShapeError

RNG_ALGORITHM = "pcg64"


@dataclass
class MeasurementResult:
    """Outcomes over an ordered qubit subset (qubits[0] = MSB of each sample)."""

    n_shots: int
    qubits: tuple
    samples: np.ndarray
    seed: int
    registers: dict = field(default_factory=dict)
    rng_algorithm: str = RNG_ALGORITHM

    def binary(self) -> np.ndarray:
        k = len(self.qubits)
        shifts = np.arange(k - 1, -1, -1, dtype=np.int64)
        return ((self.samples[:, None] >> shifts[None, :]) & 1).astype(np.uint8)


def _validate_qubits(state, qubits):
    qubits = tuple(int(q) for q in qubits)
    if not qubits:
        raise ShapeError("measurement needs at least one qubit")
    if len(set(qubits)) != len(qubits):
        raise ShapeError(f"duplicate measurement qubits {qubits}")
    for q in qubits:
        if not 0 <= q < state.n_qubits:
            raise ShapeError(f"qubit {q} out of range for {state.n_qubits} qubits")
    return qubits


def _f64(n):
    torch = nat.torch_mod()
    return torch.empty(n, dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))


def device_probabilities(state):
    """float64 |a|^2 of every amplitude, on the device."""
    p = _f64(state.n_amps)
    nat.check(
        nat.lib().qsb_probabilities(state.data_ptr, state.n_amps, state.precision.qsb_dtype, p.data_ptr(),
                                    nat.stream_ptr()),
        "probabilities",
    )
    return p


def device_marginal(state, qubits):
    """Marginal distribution over `qubits` as a float64 CUDA tensor (length 2**len(qubits))."""
    qubits = _validate_qubits(state, qubits)
    n = state.n_qubits
    lib = nat.lib()
    k = len(qubits)
    kept = np.array([n - 1 - q for q in qubits], dtype=np.int32)
    if k < n and int(kept.min()) >= 8:
        # the 8 lowest bits are summed out: leaf sums straight from the amplitudes
        out = _f64(1 << k)
        scratch = _f64(int(lib.qsb_marginal_scratch_doubles(n, k)))
        nat.check(lib.qsb_marginal_amps(state.data_ptr, state.precision.qsb_dtype, n, k, kept.ctypes.data,
                                        out.data_ptr(), scratch.data_ptr(), nat.stream_ptr()), "marginal")
        return out
    probs = device_probabilities(state)
    if qubits == tuple(range(n)):
        return probs
    out = _f64(1 << k)
    scratch = _f64(int(lib.qsb_marginal_scratch_doubles(n, k)))
    nat.check(
        lib.qsb_marginal(probs.data_ptr(), n, k, kept.ctypes.data, out.data_ptr(), scratch.data_ptr(),
                         nat.stream_ptr()),
        "marginal",
    )
    del probs, scratch
    return out


def marginal_probabilities(state, qubits) -> np.ndarray:
    """Outcome probabilities over `qubits` (others traced out), float64 even for f32 states."""
    return device_marginal(state, qubits).cpu().numpy()


def pcg64_seed_state(seed: int):
    """(state, inc) of numpy.random.default_rng(seed)'s PCG64, as four uint64 halves."""
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m


def device_cdf(probs, normalize: bool = True):
    """Normalised cumulative distribution, bit-identical to numpy's cumsum(p) / cumsum(p)[-1];
    normalize=False: the exact sequential cumsum itself."""
    torch = nat.torch_mod()
    lib = nat.lib()
    n = probs.numel()
    cum = torch.empty_like(probs)
    nbytes = int(lib.qsb_cumsum_scratch_bytes(n))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=probs.device)
    nat.check(
        lib.qsb_cumsum(probs.data_ptr(), n, cum.data_ptr(), scratch.data_ptr(), nbytes, 1 if normalize else 0,
                       nat.stream_ptr()),
        "cumsum",
    )
    return cum


def device_sample_counts(cum, n_shots: int, seed: int):
    """#{i : cum[i] <= u_k} for the n_shots draws u_k of default_rng(seed), unclipped."""
    torch = nat.torch_mod()
    out = torch.empty(int(n_shots), dtype=torch.int64, device=cum.device)
    sh, sl, ih, il = pcg64_seed_state(seed)
    nat.check(
        nat.lib().qsb_sample_counts(cum.data_ptr(), cum.numel(), sh, sl, ih, il, int(n_shots), out.data_ptr(),
                                    nat.stream_ptr()),
        "sample_counts",
    )
    return out


def device_sample(cum, n_shots: int, seed: int):
    torch = nat.torch_mod()
    out = torch.empty(int(n_shots), dtype=torch.int64, device=cum.device)
    sh, sl, ih, il = pcg64_seed_state(seed)
    nat.check(
        nat.lib().qsb_sample(cum.data_ptr(), cum.numel(), sh, sl, ih, il, int(n_shots), out.data_ptr(),
                             nat.stream_ptr()),
        "sample",
    )
    return out


def sample(state, qubits, n_shots: int, seed: int, registers: dict | None = None) -> MeasurementResult:
    """Draw `n_shots` outcomes by inverse-CDF sampling (measurement.py:61-87)."""
    if n_shots < 1:
        raise ValueError(f"n_shots must be >= 1, got {n_shots}")
    qubits = _validate_qubits(state, qubits)
    regs = dict(registers or {})
    for name, reg in regs.items():
        missing = set(reg) - set(qubits)
        if missing:
            raise ShapeError(f"register {name!r} references unmeasured qubits {sorted(missing)}")
        regs[name] = tuple(reg)
    n = state.n_qubits
    if SPARSE_CDF and qubits == tuple(range(n)) and (1 << n) >= SPARSE_CDF_MIN and n_shots < (1 << 32):
        # every qubit in order: the probabilities and the scan's block sums in one pass
        probs, bsums = device_probabilities_block_sums(state)
        samples = device_sample_exact(probs, n_shots, seed, bsums).cpu().numpy()
        return MeasurementResult(int(n_shots), qubits, samples, int(seed), regs)
    probs = device_marginal(state, qubits)
    if SPARSE_CDF and probs.numel() >= SPARSE_CDF_MIN and n_shots < (1 << 32):
        samples = device_sample_exact(probs, n_shots, seed).cpu().numpy()
    else:
        cum = device_cdf(probs)
        del probs
        samples = device_sample(cum, n_shots, seed).cpu().numpy()
    return MeasurementResult(int(n_shots), qubits, samples, int(seed), regs)


# sample() draws through qsb_sample_exact (no CDF: row starts of the drawn blocks, a 16-element
# walk per draw) for marginals of at least SPARSE_CDF_MIN outcomes.  Measured at 2^30 outcomes
# (tools/sparse_vs_full.py): 1e5 / 3e5 / 1e6 / 3e6 shots 17.2 / 18.8 / 20.8 / 21.4 ms against
# 27.1-28.5 ms through the full CDF; QSB_SPARSE_CDF=0: always the full CDF
SPARSE_CDF = os.environ.get("QSB_SPARSE_CDF", "1") != "0"
SPARSE_CDF_MIN = 1 << 16


def device_probabilities_block_sums(state):
    """(probabilities, approximate 4096-element block sums) of a state in one pass."""
    n = state.n_amps
    probs = _f64(n)
    bsums = _f64((n + 4095) // 4096)
    nat.check(nat.lib().qsb_probabilities_block_sums(state.data_ptr, n, state.precision.qsb_dtype, probs.data_ptr(),
                                                     bsums.data_ptr(), nat.stream_ptr()), "probabilities")
    return probs, bsums


def device_sample_exact(probs, n_shots: int, seed: int, block_sums=None):
    """The draws of sample() straight from the probabilities: the exact scan's block
    boundaries route every draw to its 4096-element block, the exact values before that block's
    16-element rows route it to a row, and the row is walked with fl(c + p) (bit-identical to
    device_cdf + device_sample)."""
    torch = nat.torch_mod()
    lib = nat.lib()
    n = probs.numel()
    cum = torch.empty(((n + 4095) // 4096) * 256, dtype=probs.dtype, device=probs.device)  # row starts
    nbytes = int(lib.qsb_sample_exact_scratch_bytes(n, int(n_shots)))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=probs.device)
    out = torch.empty(int(n_shots), dtype=torch.int64, device=probs.device)
    sh, sl, ih, il = pcg64_seed_state(seed)
    if block_sums is not None:
        nat.check(lib.qsb_sample_exact_bsums(probs.data_ptr(), block_sums.data_ptr(), n, cum.data_ptr(),
                                             scratch.data_ptr(), nbytes, sh, sl, ih, il, int(n_shots), out.data_ptr(),
                                             nat.stream_ptr()), "sample_exact")
        return out
    nat.check(lib.qsb_sample_exact(probs.data_ptr(), n, cum.data_ptr(), scratch.data_ptr(), nbytes, sh, sl, ih, il,
                                   int(n_shots), out.data_ptr(), nat.stream_ptr()), "sample_exact")
    return out


def collapse(state, qubits, outcome: int) -> float:
    """Project `state` in place onto `outcome` of `qubits` (qubits[0] = MSB of the outcome, as
    in `sample`) and renormalise; returns the outcome's probability.

    Extension beyond the reference (which has no mid-circuit measurement): the
    probability is the bit-exact marginal of `marginal_probabilities`, the kept amplitudes are
    scaled by 1/sqrt(p) in the state's precision, all others become exact zeros."""
    qubits = _validate_qubits(state, qubits)
    k = len(qubits)
    outcome = int(outcome)
    if not 0 <= outcome < (1 << k):
        raise ShapeError(f"outcome {outcome} out of range for {k} qubits")
    p = float(device_marginal(state, qubits)[outcome].item())
    if p <= 0.0:
        raise ValueError(f"outcome {outcome} has probability 0")
    n = state.n_qubits
    mask = value = 0
    for j, q in enumerate(qubits):
        bit = 1 << (n - 1 - q)
        mask |= bit
        if (outcome >> (k - 1 - j)) & 1:
            value |= bit
    nat.check(nat.lib().qsb_collapse(state.data_ptr, state.n_amps, state.precision.qsb_dtype, mask, value,
                                     1.0 / np.sqrt(p), nat.stream_ptr()), "collapse")
    return p


def measure(state, qubits, seed: int) -> int:
    """Mid-circuit measurement: draw one outcome exactly as `sample(state, qubits, 1, seed)` and
    collapse the state onto it (in place).  Returns the outcome."""
    outcome = int(sample(state, qubits, 1, seed).samples[0])
    collapse(state, qubits, outcome)
    return outcome


def frequencies(result: MeasurementResult, register: str | None = None) -> dict:
    """Outcome counts, optionally projected onto a named register (measurement.py:90-103)."""
    samples = result.samples
    if register is not None:
        if register not in result.registers:
            raise KeyError(register)
        reg = result.registers[register]
        k = len(result.qubits)
        pos = np.array([result.qubits.index(q) for q in reg], dtype=np.int64)
        bits = (samples[:, None] >> (k - 1 - pos)[None, :]) & 1
        weights = 1 << np.arange(len(reg) - 1, -1, -1, dtype=np.int64)
        samples = bits @ weights
    values, counts = np.unique(samples, return_counts=True)
    return {int(v): int(c) for v, c in zip(values, counts)}
