"""Device-resident state vectors (drop-in for /root/reference/pkg/src/qsim/state.py).

Basis convention kept from the reference (state.py:1-6, 34-36): qubit q is bit n-1-q of the
basis index, qubit 0 is the most significant bit.

The amplitudes live in HBM as one contiguous torch CUDA tensor (complex64 / complex128);
torch only provides the allocation and the stream, every numeric operation is a qsb200 kernel.
`StateVector.amplitudes` keeps the reference's numpy contract: reading it copies the state to
the host (a fresh array each time), assigning a numpy array uploads it.
"""

from __future__ import annotations

import enum
import math
import os

import numpy as np

from . import _native as nat
from .errors import CapacityError, ShapeError, SimulationError

# The reference caps states at 34 qubits (state.py:15).  The distributed (sharded) path and
# BASELINE config 5 need 36; lift the cap with set_max_qubits() or QSB_MAX_QUBITS.
MAX_QUBITS = 34
_cap = int(os.environ.get("QSB_MAX_QUBITS", MAX_QUBITS))


def max_qubits() -> int:
    return _cap


def set_max_qubits(n: int) -> None:
    """Raise (or restore) the qubit cap enforced by StateVector / zero_state / Circuit."""
    global _cap
    if n < 1 or n > 40:
        raise ValueError(f"qubit cap must lie in [1, 40], got {n}")
    _cap = int(n)


def _check_cap(n_qubits: int):
    if not 1 <= n_qubits <= _cap:
        raise CapacityError(f"n_qubits must be within [1, {_cap}], got {n_qubits}")


class Precision(enum.Enum):
    """Complex width of the amplitudes (state.py:18-31)."""

    F32 = "f32"
    F64 = "f64"

    @property
    def complex_dtype(self) -> np.dtype:
        return np.dtype(np.complex128 if self is Precision.F64 else np.complex64)

    @property
    def norm_atol(self) -> float:
        return 1e-10 if self is Precision.F64 else 1e-4

    @property
    def torch_dtype(self):
        torch = nat.torch_mod()
        return torch.complex128 if self is Precision.F64 else torch.complex64

    @property
    def qsb_dtype(self) -> int:
        return nat.QSB_C128 if self is Precision.F64 else nat.QSB_C64

    @property
    def itemsize(self) -> int:
        return 16 if self is Precision.F64 else 8


def bit_position(n_qubits: int, qubit: int) -> int:
    """Index bit that stores `qubit` (qubit 0 = most significant bit)."""
    return n_qubits - 1 - qubit


def _device():
    nat.require_cuda()
    torch = nat.torch_mod()
    return torch.device("cuda", torch.cuda.current_device())


def allocate(n_qubits: int, precision: Precision):
    """Uninitialised device buffer for 2**n amplitudes (the state allocator)."""
    torch = nat.torch_mod()
    try:
        return torch.empty(1 << n_qubits, dtype=precision.torch_dtype, device=_device())
    except RuntimeError as exc:  # torch.OutOfMemoryError is a RuntimeError
        raise CapacityError(
            f"cannot allocate a {n_qubits}-qubit {precision.value} state "
            f"({(1 << n_qubits) * precision.itemsize / 2**30:.1f} GiB): {exc}"
        ) from exc


# side streams for chunked device -> host copies (StateVector.copy_to_host)
COPY_STREAMS = 4
_COPY_STREAMS: dict = {}


def _copy_streams(k):
    torch = nat.torch_mod()
    key = (torch.cuda.current_device(), k)
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = [torch.cuda.Stream() for _ in range(k)]
    return _COPY_STREAMS[key]


class StateVector:
    """Dense 2**n amplitude vector resident in HBM (state.py:39-64).

    Constructed like the reference: StateVector(n_qubits, amplitudes, precision), where
    `amplitudes` may be a numpy array (uploaded) or a CUDA tensor (adopted without a copy).
    """

    __slots__ = ("n_qubits", "precision", "_t", "_layout")

    def __init__(self, n_qubits: int, amplitudes, precision: Precision = Precision.F64):
        _check_cap(n_qubits)
        self.n_qubits = int(n_qubits)
        self.precision = precision
        expected = (1 << self.n_qubits,)
        torch = nat.torch_mod()
        if isinstance(amplitudes, torch.Tensor):
            if tuple(amplitudes.shape) != expected:
                raise ShapeError(f"amplitude array has shape {tuple(amplitudes.shape)}, expected {expected}")
            if amplitudes.dtype != precision.torch_dtype:
                raise ShapeError(f"amplitude dtype {amplitudes.dtype} does not match precision {precision.value}")
            if not amplitudes.is_cuda:
                amplitudes = amplitudes.to(_device())
            self._t = amplitudes.contiguous()
        else:
            arr = np.asarray(amplitudes)
            if arr.shape != expected:
                raise ShapeError(f"amplitude array has shape {arr.shape}, expected {expected}")
            if arr.dtype != precision.complex_dtype:
                raise ShapeError(f"amplitude dtype {arr.dtype} does not match precision {precision.value}")
            self._t = upload(arr)
        # logical -> physical qubit map (None = canonical): a state too large for an
        # out-of-place scratch buffer takes uncontrolled SWAPs as relabels (engine.run_gates);
        # every canonical access below (tensor, data_ptr, amplitudes) applies the permutation
        # first, so callers always see the reference layout (state.py:1-6, 34-36)
        self._layout = None

    # -- numpy view (host copy) ------------------------------------------------------------
    @property
    def amplitudes(self) -> np.ndarray:
        self._canonicalize()
        return download(self._t)

    def copy_to_host(self, out, n_streams: int = COPY_STREAMS):
        """Write the amplitudes into `out` (a host torch tensor of 2**n elements and the state's
        dtype, pinned for an asynchronous copy) in `n_streams` chunks on side streams ordered
        after the current stream: several copy engines at once read the state back ~6% faster
        than one (measured 16 GB: 51.3 -> 54.9 GB/s).  Returns `out`; synchronise (or wait on
        the current stream after the call) before reading it."""
        torch = nat.torch_mod()
        self._canonicalize()
        src = self._t.reshape(-1)
        if out.numel() != src.numel() or out.dtype != src.dtype or out.is_cuda:
            raise ShapeError("copy_to_host needs a host tensor of the state's size and dtype")
        cur = torch.cuda.current_stream()
        k = max(1, int(n_streams)) if src.numel() >= (1 << 20) else 1
        streams = _copy_streams(k)
        chunk = -(-src.numel() // k)
        done = []
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                out[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
            done.append(s)
        for s in done:
            cur.wait_stream(s)
        src.record_stream(cur)
        return out

    @amplitudes.setter
    def amplitudes(self, values):
        arr = np.asarray(values)
        if arr.shape != (1 << self.n_qubits,) or arr.dtype != self.precision.complex_dtype:
            raise ShapeError("replacement amplitudes must keep shape and dtype")
        self._t = upload(arr)
        self._layout = None

    # -- device view -----------------------------------------------------------------------
    @property
    def tensor(self):
        """The CUDA tensor holding the amplitudes (mutated in place by the kernels)."""
        self._canonicalize()
        return self._t

    @property
    def data_ptr(self) -> int:
        self._canonicalize()
        return int(self._t.data_ptr())

    @property
    def raw_ptr(self) -> int:
        """Device pointer of the buffer in its current (possibly relabelled) layout (engine)."""
        return int(self._t.data_ptr())

    @property
    def raw_tensor(self):
        return self._t

    @property
    def layout(self):
        """Physical qubit of every logical qubit, or None when the buffer is canonical."""
        return self._layout

    @property
    def n_amps(self) -> int:
        return 1 << self.n_qubits

    def copy(self) -> "StateVector":
        dup = StateVector(self.n_qubits, self._t.clone(), self.precision)
        dup._layout = self._layout
        return dup

    def _canonicalize(self) -> None:
        """Apply a pending qubit relabelling: one bit-permuting copy when a scratch buffer fits,
        else in-place SWAP kernels (one half sweep per transposition)."""
        if self._layout is None:
            return
        from . import engine

        n = self.n_qubits
        phys = list(self._layout)
        self._layout = None
        if engine.scratch_fits(self.n_amps * self.precision.itemsize):
            dst = [0] * n  # physical qubit p (bit n-1-p) holds logical q: bit n-1-p -> bit n-1-q
            for q, p in enumerate(phys):
                dst[n - 1 - p] = n - 1 - q
            torch = nat.torch_mod()
            out = torch.empty_like(self._t)
            perm = np.ascontiguousarray(dst, dtype=np.int32)
            nat.check(nat.lib().qsb_permute_qubits(self._t.data_ptr(), out.data_ptr(), n, self.precision.qsb_dtype,
                                                   perm.ctypes.data, nat.stream_ptr()), "canonicalize")
            self._t = out
            return
        swap = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)
        where = {p: q for q, p in enumerate(phys)}  # physical -> logical
        for q in range(n):
            p = phys[q]
            if p == q:
                continue
            q2 = where[q]  # the logical qubit currently stored at physical q
            tb = np.array([n - 1 - p, n - 1 - q], dtype=np.int32)
            cb = np.zeros(1, dtype=np.int32)
            nat.check(nat.lib().qsb_apply_matrix(self._t.data_ptr(), n, self.precision.qsb_dtype, 2, tb.ctypes.data, 0,
                                                 cb.ctypes.data, swap.ctypes.data, nat.KERNEL_PERMUTATION,
                                                 nat.stream_ptr()), "canonicalize")
            phys[q], phys[q2] = q, p
            where[q], where[p] = q, q2

    def __repr__(self):
        return f"StateVector(n_qubits={self.n_qubits}, precision={self.precision.value}, device={self._t.device})"


def upload(arr: np.ndarray):
    torch = nat.torch_mod()
    dev = _device()
    host = torch.from_numpy(np.ascontiguousarray(arr))
    return host.to(dev, non_blocking=False)


def download(t) -> np.ndarray:
    """One device -> host copy into fresh host memory (the tensor .cpu() returns owns it)."""
    return t.detach().to("cpu").numpy()


def zero_state(n_qubits: int, precision: Precision = Precision.F64) -> StateVector:
    """|0...0> (state.py:67-75): memset + one store on the device."""
    _check_cap(n_qubits)
    return basis_state(n_qubits, 0, precision)


def basis_state(n_qubits: int, index: int, precision: Precision = Precision.F64) -> StateVector:
    """|index> with the reference's bit convention."""
    _check_cap(n_qubits)
    t = allocate(n_qubits, precision)
    nat.check(
        nat.lib().qsb_init_basis(t.data_ptr(), n_qubits, precision.qsb_dtype, int(index), nat.stream_ptr()),
        "zero_state",
    )
    return StateVector(n_qubits, t, precision)


def uniform_state(n_qubits: int, precision: Precision = Precision.F64) -> StateVector:
    """|+>^n: every amplitude 2**(-n/2), computed in float64 then cast like
    hamiltonians._plus_state (hamiltonians.py:115-117)."""
    _check_cap(n_qubits)
    t = allocate(n_qubits, precision)
    value = float(1.0 / np.sqrt(float(1 << n_qubits)))
    nat.check(
        nat.lib().qsb_init_uniform(t.data_ptr(), n_qubits, precision.qsb_dtype, value, 0.0, nat.stream_ptr()),
        "uniform_state",
    )
    return StateVector(n_qubits, t, precision)


def from_amplitudes(values, normalize: bool = False, precision: Precision | None = None) -> StateVector:
    """Wrap explicit amplitudes (state.py:78-106): verbatim copy unless `normalize`; precision
    inferred from the dtype (complex64/float32 -> F32) unless given."""
    torch = nat.torch_mod()
    if isinstance(values, torch.Tensor) and values.is_cuda:
        if values.dim() != 1:
            raise ShapeError(f"expected a flat amplitude array, got shape {tuple(values.shape)}")
        size = values.numel()
        small = values.dtype in (torch.complex64, torch.float32)
        arr = None
    else:
        arr = np.asarray(values)
        if arr.ndim != 1:
            raise ShapeError(f"expected a flat amplitude array, got shape {arr.shape}")
        size = arr.size
        small = arr.dtype in (np.dtype(np.complex64), np.dtype(np.float32))
    if size < 2 or size & (size - 1):
        raise ShapeError(f"amplitude count {size} is not a power of two >= 2")
    n_qubits = size.bit_length() - 1
    if n_qubits > _cap:
        raise CapacityError(f"{n_qubits} qubits exceed the cap of {_cap}")
    if precision is None:
        precision = Precision.F32 if small else Precision.F64
    if arr is not None:
        state = StateVector(n_qubits, arr.astype(precision.complex_dtype, copy=True), precision)
    else:
        state = StateVector(n_qubits, values.to(precision.torch_dtype).clone(), precision)
    if normalize:
        nrm = norm(state)
        if nrm == 0.0:
            raise ValueError("cannot normalize the zero vector")
        nat.check(
            nat.lib().qsb_scale(state.data_ptr, state.n_amps, precision.qsb_dtype, 1.0 / nrm, 0.0, nat.stream_ptr()),
            "from_amplitudes(normalize)",
        )
    return state


def _scalar_buffer(n_doubles: int):
    torch = nat.torch_mod()
    return torch.empty(n_doubles, dtype=torch.float64, device=_device())


def norm(state: StateVector) -> float:
    """Euclidean norm (state.py:109-111) as a deterministic device reduction."""
    out = _scalar_buffer(1)
    nat.check(
        nat.lib().qsb_norm2(state.data_ptr, state.n_amps, state.precision.qsb_dtype, out.data_ptr(), nat.stream_ptr()),
        "norm",
    )
    return float(math.sqrt(float(out.item())))


def overlap(a: StateVector, b: StateVector) -> complex:
    """<a|b>, conjugate-linear in a (state.py:114-122)."""
    if a.n_qubits != b.n_qubits:
        raise ShapeError(f"qubit counts differ: {a.n_qubits} vs {b.n_qubits}")
    if a.precision is not b.precision:
        raise ValueError("cannot mix f32 and f64 states in one operation")
    out = _scalar_buffer(2)
    nat.check(
        nat.lib().qsb_vdot(a.data_ptr, b.data_ptr, a.n_amps, a.precision.qsb_dtype, out.data_ptr(), nat.stream_ptr()),
        "overlap",
    )
    re, im = out.tolist()
    return complex(re, im)


def synchronize():
    nat.torch_mod().cuda.synchronize()


__all__ = [
    "MAX_QUBITS",
    "Precision",
    "StateVector",
    "basis_state",
    "bit_position",
    "from_amplitudes",
    "max_qubits",
    "norm",
    "overlap",
    "set_max_qubits",
    "uniform_state",
    "zero_state",
]

_ = SimulationError  # re-exported for callers catching device errors
