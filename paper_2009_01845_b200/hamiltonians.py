"""Trotter-form Hamiltonians (drop-in for the hot-path part of
/root/reference/pkg/src/qsim/hamiltonians.py).

In scope: TrotterHamiltonian (:62-93), build_x / build_tfim in Trotter form (:120-154),
combine (:157-174), the |+>^n ground state of build_x (:115-117) and the Trotter-form
expectation (:192-207) evaluated on the device.  The dense 2^N x 2^N form (capped at 12 qubits
and diagonalised with numpy.linalg.eigh in the reference) is outside the B200 hot path
(SURVEY.md section 2.1 row 6); asking for it raises FormError.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import CapacityError, FormError, ShapeError
from .state import Precision, StateVector, uniform_state

DENSE_MAX_QUBITS = 12
HERMITICITY_ATOL = 1e-10

_PX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_PZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)


class Form(enum.Enum):
    DENSE = "dense"
    TROTTER = "trotter"


def _require_hermitian(m, what):
    dev = np.max(np.abs(m - m.conj().T))
    if dev > HERMITICITY_ATOL:
        raise ShapeError(f"{what} is not Hermitian (deviation {dev:.2e})")


@dataclass
class TrotterHamiltonian:
    """Sum of <= 2-qubit Hermitian terms [(qubits, matrix), ...]."""

    n_qubits: int
    terms: list
    ground_state: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.n_qubits < 1:
            raise ShapeError(f"n_qubits must be >= 1, got {self.n_qubits}")
        clean = []
        for qubits, matrix in self.terms:
            qubits = tuple(int(q) for q in qubits)
            k = len(qubits)
            if k > 2:
                raise CapacityError(f"Trotter terms act on at most 2 qubits, got {qubits}")
            if k == 0 or len(set(qubits)) != k:
                raise ShapeError(f"bad term qubits {qubits}")
            for q in qubits:
                if not 0 <= q < self.n_qubits:
                    raise ShapeError(f"qubit {q} out of range for {self.n_qubits} qubits")
            m = np.asarray(matrix, dtype=np.complex128)
            if m.shape != (1 << k, 1 << k):
                raise ShapeError(f"term matrix shape {m.shape} does not fit {k} qubit(s)")
            _require_hermitian(m, f"term on {qubits}")
            clean.append((qubits, m))
        self.terms = clean

    @property
    def form(self) -> Form:
        return Form.TROTTER


def plus_state(n_qubits: int, precision: Precision = Precision.F64) -> StateVector:
    """|+>^n: the ground state of -sum X (hamiltonians.py:115-117), one fill kernel."""
    return uniform_state(n_qubits, precision)


def _dense_unsupported():
    raise FormError("the dense Hamiltonian form is outside the B200 hot path; use Form.TROTTER")


def build_x(n_qubits: int, form: Form = Form.TROTTER):
    """H = -sum_i X_i; ground state |+>^N (hamiltonians.py:120-132)."""
    if form is Form.DENSE:
        _dense_unsupported()
    if n_qubits < 2:
        raise ShapeError("Trotter form needs at least 2 qubits")
    ground = lambda precision=Precision.F64: plus_state(n_qubits, precision)  # noqa: E731
    ground.is_plus_state = True  # lets the sharded evolution build |+>^n shard by shard
    return TrotterHamiltonian(n_qubits, [((i,), -_PX) for i in range(n_qubits)], ground_state=ground)


def build_tfim(n_qubits: int, h: float, form: Form = Form.TROTTER):
    """Periodic transverse-field Ising chain, bond i = -(Z Z + h X I) on (i, i+1 mod N)
    (hamiltonians.py:135-154)."""
    if n_qubits < 2:
        raise ShapeError(f"the chain needs at least 2 qubits, got {n_qubits}")
    if form is Form.DENSE:
        _dense_unsupported()
    bond = -(np.kron(_PZ, _PZ) + h * np.kron(_PX, np.eye(2, dtype=np.complex128)))
    return TrotterHamiltonian(n_qubits, [((i, (i + 1) % n_qubits), bond) for i in range(n_qubits)])


def combine(a, coeff_a: float, b, coeff_b: float):
    """coeff_a * a + coeff_b * b; terms on identical qubit tuples merge, first-seen order
    (hamiltonians.py:157-174)."""
    if a.n_qubits != b.n_qubits:
        raise ShapeError(f"qubit counts differ: {a.n_qubits} vs {b.n_qubits}")
    if a.form is not b.form:
        raise FormError(f"cannot combine {a.form.value} with {b.form.value}")
    if a.form is not Form.TROTTER:
        _dense_unsupported()
    acc: dict = {}
    order = []
    for coeff, ham in ((coeff_a, a), (coeff_b, b)):
        for qubits, m in ham.terms:
            if qubits in acc:
                acc[qubits] = acc[qubits] + coeff * m
            else:
                acc[qubits] = coeff * m
                order.append(qubits)
    return TrotterHamiltonian(a.n_qubits, [(q, acc[q]) for q in order])


_EXPECT_CACHE: dict = {}


def _expectation_passes(bit_terms, state):
    """The terms (bit positions, MSB first) as read-only fused passes (jit expectation kernels:
    every term whose bits fit a tile is evaluated from the registers of that tile, one HBM read
    per pass instead of one per term).  None when the specialised kernels are unavailable or
    the state is too small."""
    from . import engine, jit
    from .fusion import plan_expectation

    from .fusion import TileGeometry

    n = state.n_qubits
    dtype = state.precision.qsb_dtype
    geo = engine.default_geometry(dtype)
    if dtype == nat.QSB_C64 and not geo.halves:
        # complex64: 512 consumers x 16 amplitudes (the accumulation is in double; 32 amplitudes
        # per thread would spill)
        geo = TileGeometry(geo.K, geo.G, geo.L, geo.nreg - 1)
    if not jit.available() or n < geo.K + 1 or geo.halves:
        return None
    key = (n, dtype, geo, tuple((tuple(b), np.asarray(m).tobytes()) for b, m in bit_terms))
    progs = _EXPECT_CACHE.get(key)
    if progs is None:
        progs = []
        for words in plan_expectation([(tuple(b), m) for b, m in bit_terms], n, dtype, geo):
            progs.append((words, jit.compile_words(words, dtype)))
        if len(_EXPECT_CACHE) > 16:
            _EXPECT_CACHE.clear()
        _EXPECT_CACHE[key] = progs
    torch = nat.torch_mod()
    total = None
    for words, (compiled, coeffs) in progs:
        part = torch.zeros(compiled.grid(), dtype=torch.float64, device=state.tensor.device)
        jit.run(words, dtype, state.data_ptr, part.data_ptr(), n, nat.stream_ptr(), compiled, coeffs)
        ssum = part.sum()
        total = ssum if total is None else total + ssum
    return float(total.item()) if total is not None else 0.0


def _expect_bit_terms(bit_terms, state) -> float:
    """sum_t <psi|H_t|psi> (real part) for terms given on bit positions (MSB of the matrix first)
    of a state-like object (StateVector or one shard)."""
    fused = _expectation_passes(bit_terms, state)
    if fused is not None:
        return fused
    torch = nat.torch_mod()
    ks = np.array([len(b) for b, _ in bit_terms], dtype=np.int32)
    bits = np.zeros(2 * max(1, len(bit_terms)), dtype=np.int32)
    mats = np.zeros(32 * max(1, len(bit_terms)), dtype=np.float64)
    for t, (b, m) in enumerate(bit_terms):
        if len(b) not in (1, 2):
            raise ShapeError(f"expectation supports 1- and 2-qubit terms, got {len(b)}")
        bits[2 * t] = b[0]
        bits[2 * t + 1] = b[-1]
        mm = np.ascontiguousarray(np.asarray(m, dtype=np.complex128))
        mats[32 * t:32 * t + 2 * mm.size] = mm.view(np.float64).reshape(-1)
    out = torch.empty(2, dtype=torch.float64, device=state.tensor.device)
    nat.check(nat.lib().qsb_expect_terms(state.data_ptr, state.n_qubits, state.precision.qsb_dtype, len(bit_terms),
                                         ks.ctypes.data, bits.ctypes.data, mats.ctypes.data, out.data_ptr(),
                                         nat.stream_ptr()),
              "expectation")
    return float(out[0].item())


def _fold_single_terms(terms):
    """Sum each 1-qubit term into a 2-qubit term on the same qubit (M2 + M1 (x) I, exact
    algebra): one read sweep per remaining term instead of one per term (TFIM + X: 2N -> N)."""
    terms = [(tuple(q), np.asarray(m, dtype=np.complex128)) for q, m in terms]
    pairs = [i for i, (q, _) in enumerate(terms) if len(q) == 2]
    out = {i: terms[i][1].copy() for i in pairs}
    keep = []
    eye = np.eye(2, dtype=np.complex128)
    for i, (q, m) in enumerate(terms):
        if len(q) == 2:
            continue
        host = next((j for j in pairs if q[0] in terms[j][0]), None)
        if host is None:
            keep.append((q, m))
            continue
        pos = terms[host][0].index(q[0])
        out[host] += np.kron(m, eye) if pos == 0 else np.kron(eye, m)
    return [(terms[i][0], out[i]) for i in pairs] + keep


def expectation(h, state: StateVector) -> float:
    """<psi|H|psi> (real part) on the device (hamiltonians.py:192-207): the terms are evaluated
    read-only (fused read passes, else `qsb_expect_terms` one sweep per term), no state copy (the
    reference copies the state and applies each term to the copy)."""
    if h.n_qubits != state.n_qubits:
        raise ShapeError(f"Hamiltonian has {h.n_qubits} qubits, state has {state.n_qubits}")
    if not isinstance(h, TrotterHamiltonian):
        _dense_unsupported()
    n = h.n_qubits
    terms = _fold_single_terms(h.terms)
    return _expect_bit_terms([(tuple(n - 1 - q for q in qs), m) for qs, m in terms], state)


def ground_state_vector(h, precision: Precision = Precision.F64) -> StateVector:
    """Attached ground-state constructor (|+>^N for build_x); other Hamiltonians need the dense
    eigen-solver, which is outside the hot path."""
    if getattr(h, "ground_state", None) is not None:
        return h.ground_state(precision)
    _dense_unsupported()
