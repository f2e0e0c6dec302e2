"""CPU ORACLE (test infrastructure only): numpy restatement of the reference state-vector path.

Gates are plain tuples (kind, targets, controls, params, matrix) so the oracle does not depend
on the product package.  Every body follows the reference implementation in
/root/reference/pkg/src/qsim; line numbers are cited per function.
"""

from __future__ import annotations

import cmath
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# ---- gate matrices: gates.py:82-122 ---------------------------------------------------------
_R2 = 1.0 / math.sqrt(2.0)
FIXED = {
    "H": np.array([[_R2, _R2], [_R2, -_R2]], dtype=complex),
    "X": np.array([[0, 1], [1, 0]], dtype=complex),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=complex),
    "Z": np.array([[1, 0], [0, -1]], dtype=complex),
    "CNOT": np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex),
    "CZ": np.diag([1, 1, 1, -1]).astype(complex),
    "SWAP": np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex),
}


def ry(t):  # gates.py:97-100
    c, s = math.cos(t / 2.0), math.sin(t / 2.0)
    return np.array([[c, -s], [s, c]], dtype=complex)


def rx(t):  # gates.py:103-106
    c, s = math.cos(t / 2.0), math.sin(t / 2.0)
    return np.array([[c, -1j * s], [-1j * s, c]], dtype=complex)


def rz(t):  # gates.py:109-110
    return np.diag([cmath.exp(-0.5j * t), cmath.exp(0.5j * t)])


def czpow(t):  # gates.py:113-114
    return np.diag([1.0, 1.0, 1.0, cmath.exp(1j * t)])


def vlayer(p):  # gates.py:117-122
    a, b, c, d = p
    return np.kron(ry(c), ry(d)) @ FIXED["CZ"] @ np.kron(ry(a), ry(b))


def matrix_of(kind, params=(), matrix=None):
    """gate_matrix (gates.py:275-289)."""
    if matrix is not None:
        return np.array(matrix, dtype=complex)
    if kind in FIXED:
        return FIXED[kind].copy()
    return {"RX": rx, "RY": ry, "RZ": rz, "CZPow": czpow}[kind](params[0]) if kind != "VariationalLayer" \
        else vlayer(params)


def gate(kind, targets, controls=(), params=(), matrix=None):
    return (kind, tuple(targets), tuple(controls), tuple(params), matrix_of(kind, params, matrix))


# ---- kernel: gates.py:334-469 ---------------------------------------------------------------
def classify(m):
    """classify_kernel (gates.py:340-352) -> 'diagonal' | 'permutation' | 'general'."""
    m = np.asarray(m)
    if np.count_nonzero(m - np.diag(np.diagonal(m))) == 0:
        return "diagonal"
    nz = m != 0
    if (nz.sum(1) == 1).all() and (nz.sum(0) == 1).all() and (np.abs(np.abs(m[nz]) - 1) <= 1e-12).all():
        return "permutation"
    return "general"


def _open_zero_bits(idx, positions):
    # gates.py:355-360: insert a zero bit at each ascending position
    for p in positions:
        lowmask = (1 << p) - 1
        idx = ((idx & ~lowmask) << 1) | (idx & lowmask)
    return idx


BLOCK = 1 << 15
PARALLEL_MIN = 1 << 17


def apply_matrix(amps, n, targets, matrix, controls=(), n_threads=1, kernel=None):
    """In-place Eq. (1) update with the reference's three bodies (gates.py:380-469)."""
    targets, controls = tuple(targets), tuple(controls)
    t = len(targets)
    m64 = np.ascontiguousarray(matrix, dtype=np.complex128)
    kernel = kernel or classify(m64)
    tb = [n - 1 - q for q in targets]
    cb = [n - 1 - q for q in controls]
    occupied = sorted(tb + cb)
    cmask = sum(1 << b for b in cb)
    dim = 1 << t
    off = np.array([sum(1 << tb[i] for i in range(t) if (j >> (t - 1 - i)) & 1) for j in range(dim)], dtype=np.int64)
    n_groups = 1 << (n - len(occupied))

    def bases(lo, hi):
        return _open_zero_bits(np.arange(lo, hi, dtype=np.int64), occupied) | cmask

    if kernel == "diagonal":
        d64 = np.diagonal(m64)
        rows = [j for j in range(dim) if d64[j] != 1.0]
        if not rows:
            return
        d = d64.astype(amps.dtype)

        def body(lo, hi):
            b = bases(lo, hi)
            for j in rows:
                amps[b + off[j]] *= d[j]
    elif kernel == "permutation":
        src = np.argmax(m64 != 0, axis=1)
        ph64 = m64[np.arange(dim), src]
        moved = [j for j in range(dim) if src[j] != j or ph64[j] != 1.0]
        if not moved:
            return
        ph = ph64.astype(amps.dtype)

        def body(lo, hi):
            b = bases(lo, hi)
            got = [amps[b + off[src[j]]] for j in moved]
            for row, j in zip(got, moved):
                amps[b + off[j]] = row * ph[j] if ph64[j] != 1.0 else row
    else:
        m = m64.astype(amps.dtype)

        def body(lo, hi):
            b = bases(lo, hi)
            idx = off[:, None] + b[None, :]
            amps[idx] = m @ amps[idx]

    if n_threads > 1 and n_groups >= PARALLEL_MIN:  # gates.py:363-377
        workers = min(n_threads, -(-n_groups // BLOCK))
        chunk = -(-n_groups // workers)

        def work(lo):
            for s in range(lo, min(lo + chunk, n_groups), BLOCK):
                body(s, min(s + BLOCK, lo + chunk, n_groups))

        with ThreadPoolExecutor(workers) as pool:
            list(pool.map(work, range(0, n_groups, chunk)))
    else:
        for s in range(0, n_groups, BLOCK):
            body(s, min(s + BLOCK, n_groups))


def run(gates, n, initial=None, dtype=np.complex128, n_threads=1):
    """Circuit.execute (circuit.py:96-125): |0..0> or a copy of `initial`, gates in order."""
    if initial is None:
        amps = np.zeros(1 << n, dtype=dtype)
        amps[0] = 1.0
    else:
        amps = np.array(initial, dtype=dtype, copy=True)
    for _kind, tg, ct, _p, m in gates:
        apply_matrix(amps, n, tg, m, ct, n_threads=n_threads)
    return amps


# ---- circuit builders: circuit.py:204-259 ---------------------------------------------------
def qft(n):
    out = []
    for q in range(n):
        out.append(gate("H", (q,)))
        for k in range(q + 1, n):
            out.append(gate("CZPow", (k, q), (), (math.pi / 2 ** (k - q),)))
    for q in range(n // 2):
        out.append(gate("SWAP", (q, n - 1 - q)))
    return out


def variational(n, layers, params, fused=False, wrap=True):
    p = np.asarray(params, dtype=float).ravel()
    out, k = [], 0
    for _ in range(layers):
        a, b = p[k:k + n], p[k + n:k + 2 * n]
        k += 2 * n
        if fused:
            out += [gate("VariationalLayer", (q, q + 1), (), (a[q], a[q + 1], b[q], b[q + 1])) for q in range(0, n, 2)]
        else:
            out += [gate("RY", (q,), (), (a[q],)) for q in range(n)]
            out += [gate("CZ", (q, q + 1)) for q in range(0, n, 2)]
            out += [gate("RY", (q,), (), (b[q],)) for q in range(n)]
        odd = [(q, q + 1) for q in range(1, n - 1, 2)] + ([(n - 1, 0)] if wrap and n > 2 else [])
        out += [gate("CZ", pr) for pr in odd]
    out += [gate("RY", (q,), (), (p[k + q],)) for q in range(n)]
    return out


def grid_supremacy(rows, cols, cycles, seed):
    """Random 'supremacy-style' circuit in reference GateSpec terms:
    per cycle a random sqrt(X)/sqrt(Y)/sqrt(W) Unitary on every qubit (no repeat per qubit),
    then fSim(pi/2, pi/6) Unitaries on couplers in the pattern ABCDCDAB; a final 1q layer."""
    rng = np.random.default_rng(seed)
    sx = np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]]) / 2
    sy = np.array([[1 + 1j, -1 - 1j], [1 + 1j, 1 + 1j]]) / 2
    w = (np.array([[1, 0], [0, 1]]) * 0 + np.array([[1, -np.sqrt(1j)], [np.sqrt(-1j), 1]])) / np.sqrt(2)
    singles = [sx, sy, w]
    th, ph = math.pi / 2, math.pi / 6
    fsim = np.array([[1, 0, 0, 0], [0, math.cos(th), -1j * math.sin(th), 0],
                     [0, -1j * math.sin(th), math.cos(th), 0], [0, 0, 0, cmath.exp(-1j * ph)]], dtype=complex)
    n = rows * cols
    q = lambda r, c: r * cols + c  # noqa: E731

    def couplers(kind):
        out = []
        for r in range(rows):
            for c in range(cols):
                if kind in "AB" and c + 1 < cols and (c % 2 == (0 if kind == "A" else 1)):
                    out.append((q(r, c), q(r, c + 1)))
                if kind in "CD" and r + 1 < rows and (r % 2 == (0 if kind == "C" else 1)):
                    out.append((q(r, c), q(r + 1, c)))
        return out

    pattern = "ABCDCDAB"
    last = [-1] * n
    out = []

    def layer1():
        for qq in range(n):
            choice = int(rng.integers(3))
            while choice == last[qq]:
                choice = int(rng.integers(3))
            last[qq] = choice
            out.append(gate("Unitary", (qq,), (), (), singles[choice]))

    for cyc in range(cycles):
        layer1()
        for a, b in couplers(pattern[cyc % len(pattern)]):
            out.append(gate("Unitary", (a, b), (), (), fsim))
    layer1()
    return out


# ---- measurement: measurement.py:36-87 ------------------------------------------------------
def probabilities(amps):
    return np.abs(amps.astype(np.complex128)) ** 2  # measurement.py:50


def marginal(amps, n, qubits):
    """marginal_probabilities (measurement.py:36-58)."""
    tensor = probabilities(amps).reshape([2] * n)
    other = tuple(q for q in range(n) if q not in qubits)
    if other:
        tensor = tensor.sum(axis=other)
    kept = sorted(qubits)
    return tensor.transpose([kept.index(q) for q in qubits]).ravel()


def sample(amps, n, qubits, n_shots, seed):
    """sample (measurement.py:61-87): sequential cumsum, PCG64 draws, searchsorted right."""
    probs = marginal(amps, n, tuple(qubits))
    cum = np.cumsum(probs)
    cum /= cum[-1]
    u = np.random.default_rng(seed).random(n_shots)
    s = np.searchsorted(cum, u, side="right").astype(np.int64)
    np.clip(s, 0, probs.size - 1, out=s)
    return s


# ---- Trotter: evolution.py:188-242, hamiltonians.py:120-174 ---------------------------------
PX = np.array([[0, 1], [1, 0]], dtype=complex)
PZ = np.array([[1, 0], [0, -1]], dtype=complex)


def x_terms(n):
    return [((i,), -PX) for i in range(n)]


def tfim_terms(n, h):
    bond = -(np.kron(PZ, PZ) + h * np.kron(PX, np.eye(2)))
    return [((i, (i + 1) % n), bond) for i in range(n)]


def combine(ta, ca, tb, cb):
    acc, order = {}, []
    for c, terms in ((ca, ta), (cb, tb)):
        for qs, m in terms:
            if qs in acc:
                acc[qs] = acc[qs] + c * m
            else:
                acc[qs] = c * m
                order.append(qs)
    return [(qs, acc[qs]) for qs in order]


def trotter_step(terms, dt):
    groups, sups = [], []
    for qs, m in terms:
        for g, s in zip(groups, sups):
            if not s & set(qs):
                g.append((qs, m))
                s.update(qs)
                break
        else:
            groups.append([(qs, m)])
            sups.append(set(qs))

    def ex(qs, m, tau):
        lam, v = np.linalg.eigh(m)
        return gate("Unitary", qs, (), (), (v * np.exp(-1j * lam * tau)) @ v.conj().T)

    if len(groups) == 1:
        return [ex(qs, m, dt) for qs, m in groups[0]]
    halves = [[ex(qs, m, dt / 2) for qs, m in g] for g in groups[:-1]]
    out = [x for h in halves for x in h]
    out += [ex(qs, m, dt) for qs, m in groups[-1]]
    for h in reversed(halves):
        out += h
    return out


def adiabatic(n, h_field, dt, T, amps=None):
    """adiabatic_evolve(build_x, build_tfim(h), linear schedule, Trotter) (evolution.py:351-383)."""
    psi = np.full(1 << n, 1.0 / np.sqrt(1 << n), dtype=np.complex128) if amps is None else amps.astype(np.complex128)
    n_full = int(math.floor(T / dt + 1e-9))
    steps = [(k * dt, dt) for k in range(n_full)]
    rem = T - n_full * dt
    if rem > 1e-9 * max(T, 1.0):
        steps.append((n_full * dt, rem))
    for t, tau in steps:
        s = min(max(t / T, 0.0), 1.0)
        terms = combine(x_terms(n), 1.0 - s, tfim_terms(n, h_field), s)
        psi = run(trotter_step(terms, tau), n, psi)
    return psi


def from_json(d):
    """Gate tuples from the reference's circuit JSON (circuit.py:265-312 format)."""
    import json as _json

    if isinstance(d, (str, bytes, np.ndarray)):
        d = _json.loads(str(d))
    out = []
    for e in d["gates"]:
        m = None
        if e.get("matrix") is not None:
            m = np.array([[complex(re, im) for re, im in row] for row in e["matrix"]])
        out.append(gate(e["name"], e["targets"], e.get("controls", ()), e.get("params", ()), m))
    return int(d["nqubits"]), out
