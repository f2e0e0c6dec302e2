"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors and
the CPU oracle.  Tolerances per BASELINE north star: 1e-12 per amplitude (complex128),
1e-5 (complex64); samples bit-exact."""

import hashlib
import json
import math

import numpy as np
import pytest

from conftest import circuit_from_json, golden, max_abs
from oracle import statevec as ov

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


def _sv(amps):
    import paper_2009_01845_b200 as q

    return q.from_amplitudes(np.asarray(amps))


# ---------------------------------------------------------------- single gates / apply_matrix
def test_single_gates_golden(cuda):
    g = golden("single_gates")
    for text, inp, out in zip(g["circuits"], g["inputs"], g["outputs"]):
        c = circuit_from_json(text)
        for fuse in (False, True):
            got = c.execute(_sv(inp), fuse=fuse).amplitudes
            assert max_abs(got, out) <= TOL64


@pytest.mark.parametrize("n", [8, 13, 16])
def test_apply_matrix_kernel_classes(cuda, n):
    import paper_2009_01845_b200 as q

    rng = np.random.default_rng(29 + n)
    amps = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    amps /= np.linalg.norm(amps)
    for spec in (q.X(3), q.SWAP(1, 6), q.CNOT(5, 2), q.CNOT(2, 5, controls=(0,)), q.Y(4)):
        fast, slow = amps.copy(), amps.copy()
        q.apply_matrix(fast, n, spec.targets, q.gate_matrix(spec), spec.controls, kernel=q.KernelClass.PERMUTATION)
        q.apply_matrix(slow, n, spec.targets, q.gate_matrix(spec), spec.controls, kernel=q.KernelClass.GENERAL)
        assert np.array_equal(fast, slow)
        ref = amps.copy()
        ov.apply_matrix(ref, n, spec.targets, q.gate_matrix(spec), spec.controls)
        assert np.array_equal(fast, ref)
    for spec in (q.Z(2), q.RZ(4, 0.9), q.CZ(1, 6), q.CZPow(0, 5, 2.2), q.CZ(3, 7, controls=(1,))):
        fast, slow = amps.copy(), amps.copy()
        q.apply_matrix(fast, n, spec.targets, q.gate_matrix(spec), spec.controls, kernel=q.KernelClass.DIAGONAL)
        q.apply_matrix(slow, n, spec.targets, q.gate_matrix(spec), spec.controls, kernel=q.KernelClass.GENERAL)
        assert max_abs(fast, slow) <= 1e-15
        ref = amps.copy()
        ov.apply_matrix(ref, n, spec.targets, q.gate_matrix(spec), spec.controls)
        assert max_abs(fast, ref) <= 1e-15


@pytest.mark.parametrize("t", [3, 4, 5])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_apply_matrix_three_to_five_targets(cuda, t, prec):
    """apply_matrix takes any 2^t x 2^t matrix (gates.py:380-469): general, diagonal and
    permutation bodies for 3-5 targets, with controls, against the oracle restatement."""
    import paper_2009_01845_b200 as q

    n = 11
    rng = np.random.default_rng(100 + t)
    dtype = np.complex128 if prec == "f64" else np.complex64
    tol = TOL64 if prec == "f64" else TOL32
    d = 1 << t
    z = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    unitary, _ = np.linalg.qr(z)
    phases = np.exp(1j * rng.uniform(0, 2 * np.pi, d))
    phases[::3] = 1.0
    diag = np.diag(phases)
    perm = np.zeros((d, d), dtype=np.complex128)
    order = rng.permutation(d)
    for r in range(d):
        perm[r, order[r]] = [1.0, -1.0, 1j, -1j][r % 4] if r % 2 else 1.0
    for mat in (unitary, diag, perm):
        qubits = [int(x) for x in rng.permutation(n)[:t + 1]]
        targets, controls = qubits[:t], qubits[t:]
        psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(dtype)
        want = psi.copy()
        ov.apply_matrix(want, n, targets, mat, controls)
        got = q.from_amplitudes(psi)
        q.apply_matrix(got, n, targets, mat, controls)
        assert max_abs(got.amplitudes, want) <= tol
        host = psi.copy()  # numpy callers: uploaded, transformed, written back in place
        q.apply_matrix(host, n, targets, mat, controls)
        assert max_abs(host, want) <= tol
        if mat is perm:
            assert np.array_equal(got.amplitudes, want)  # exact moves and +-1 / +-i phases
    with pytest.raises(q.ShapeError):
        q.apply_matrix(q.zero_state(12), 12, list(range(11)), np.eye(2048))


@pytest.mark.parametrize("t", [6, 8, 10])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_apply_matrix_six_to_ten_targets(cuda, t, prec):
    """apply_matrix with 6-10 targets (the dense shared-memory body), with a control and in
    scattered target order, against the oracle restatement."""
    import paper_2009_01845_b200 as q

    n = 13
    rng = np.random.default_rng(200 + t)
    dtype = np.complex128 if prec == "f64" else np.complex64
    tol = TOL64 if prec == "f64" else TOL32
    d = 1 << t
    unitary, _ = np.linalg.qr(rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d)))
    diag = np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, d)))
    for mat in (unitary, diag):
        qubits = [int(x) for x in rng.permutation(n)[:t + 1]]
        targets, controls = qubits[:t], qubits[t:]
        psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(dtype)
        want = psi.copy()
        ov.apply_matrix(want, n, targets, mat, controls)
        got = q.from_amplitudes(psi)
        q.apply_matrix(got, n, targets, mat, controls)
        assert max_abs(got.amplitudes, want) <= tol * (1 << (t - 5))  # sums of 2^t terms


def test_control_leaves_unset_half_untouched(cuda):
    import paper_2009_01845_b200 as q

    rng = np.random.default_rng(41)
    init = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    st = _sv(init)
    q.apply_gate(st, q.H(2, controls=(0,)))
    out = st.amplitudes
    assert np.array_equal(out[:8], init[:8])
    assert np.max(np.abs(out[8:] - init[8:])) > 1e-3


def test_apply_matrix_validation(cuda):
    import paper_2009_01845_b200 as q

    amps = q.zero_state(3).amplitudes
    with pytest.raises(q.ShapeError):
        q.apply_matrix(amps, 3, (0, 0), np.eye(4))
    with pytest.raises(q.ShapeError):
        q.apply_matrix(amps, 3, (5,), np.eye(2))
    with pytest.raises(q.ShapeError):
        q.apply_matrix(amps, 3, (0,), np.eye(4))


def test_states_basics(cuda):
    import paper_2009_01845_b200 as q

    assert np.array_equal(q.zero_state(2).amplitudes, [1, 0, 0, 0])
    s = q.zero_state(3, q.Precision.F32)
    assert s.amplitudes.dtype == np.complex64 and s.amplitudes[0] == 1
    for n in (1, 3, 5):
        st = q.zero_state(n)
        q.apply_gate(st, q.X(0))
        a = st.amplitudes
        assert a[1 << (n - 1)] == 1.0 and np.count_nonzero(a) == 1
    assert q.norm(q.from_amplitudes([2, 0])) == 2.0
    assert abs(q.norm(q.from_amplitudes([0.5] * 4)) - 1.0) < 1e-15
    plus = q.zero_state(1)
    q.apply_gate(plus, q.H(0))
    assert abs(q.overlap(q.zero_state(1), plus) - 1 / math.sqrt(2)) < 1e-15
    st = q.from_amplitudes([1, 1], normalize=True)
    assert np.allclose(st.amplitudes, [1 / math.sqrt(2)] * 2, atol=1e-15)
    with pytest.raises(ValueError):
        q.from_amplitudes([0, 0, 0, 0], normalize=True)
    with pytest.raises(ValueError):
        q.overlap(q.zero_state(2, q.Precision.F32), q.zero_state(2))
    u = q.uniform_state(5).amplitudes
    assert np.array_equal(u, np.full(32, 1 / np.sqrt(32)).astype(complex))
    dup = q.zero_state(2)
    cp = dup.copy()
    q.apply_gate(cp, q.X(1))
    assert dup.amplitudes[0] == 1.0


# ---------------------------------------------------------------- circuits
@pytest.mark.parametrize("fuse", [False, True])
def test_random_circuits_golden(cuda, fuse, mode):
    g = golden("random_circuits")
    for i, text in enumerate(g["circuits"]):
        c = circuit_from_json(text)
        got = c.execute(_sv(g[f"in{i}"]), fuse=fuse).amplitudes
        assert max_abs(got, g[f"out{i}"]) <= TOL64


@pytest.mark.parametrize("n", [10, 14])
@pytest.mark.parametrize("fuse", [False, True])
def test_qft_golden(cuda, n, fuse, mode):
    import paper_2009_01845_b200 as q

    g = golden("qft")
    c = q.qft_circuit(n)
    assert max_abs(c.execute(fuse=fuse).amplitudes, g[f"zero{n}"]) <= TOL64
    assert max_abs(c.execute(_sv(g[f"rin{n}"]), fuse=fuse).amplitudes, g[f"rout{n}"]) <= TOL64
    k = int(g[f"basisk{n}"])
    got = c.execute(q.basis_state(n, k), fuse=fuse).amplitudes
    assert max_abs(got, g[f"basis{n}"]) <= TOL64
    f32 = c.execute(precision=q.Precision.F32, fuse=fuse).amplitudes
    assert f32.dtype == np.complex64 and max_abs(f32, g[f"f32_{n}"]) <= TOL32


@pytest.mark.parametrize("n", [18, 22])
def test_qft_analytic_dft_column(cuda, n, mode):
    import paper_2009_01845_b200 as q

    k = int(np.random.default_rng(n).integers(1 << n))
    got = q.qft_circuit(n).execute(q.basis_state(n, k)).amplitudes
    j = np.arange(1 << n, dtype=np.float64)
    want = np.exp(2j * np.pi * ((j * k) % (1 << n)) / (1 << n)) / np.sqrt(1 << n)
    assert max_abs(got, want) <= 1e-12


@pytest.mark.parametrize("n", [10, 14])
@pytest.mark.parametrize("fused_layers", [False, True])
@pytest.mark.parametrize("fuse", [False, True])
def test_variational_golden(cuda, n, fused_layers, fuse, mode):
    import paper_2009_01845_b200 as q

    g = golden("variational")
    c = q.variational_circuit(n, 3, g[f"params{n}"], fused=fused_layers)
    assert max_abs(c.execute(fuse=fuse).amplitudes, g[f"f64_{n}_{int(fused_layers)}"]) <= TOL64
    got32 = c.execute(precision=q.Precision.F32, fuse=fuse).amplitudes
    assert max_abs(got32, g[f"f32_{n}_{int(fused_layers)}"]) <= TOL32


def test_grid_supremacy_golden(cuda, mode):
    g = golden("grid15")
    c = circuit_from_json(g["circuit"])
    for fuse in (False, True):
        assert max_abs(c.execute(fuse=fuse).amplitudes, g["out"]) <= TOL64


def test_callbacks_split_execution(cuda):
    import paper_2009_01845_b200 as q

    class Counter(q.Callback):
        def _compute(self, state, t, hamiltonian):
            return float(np.abs(state.amplitudes[0]))

    c = q.Circuit(2).add([q.H(0), q.H(1), q.X(0)])
    cb = Counter()
    c.execute(callbacks=[(cb, (0, 2))])
    assert len(cb.records) == 2
    assert abs(cb.records[0] - 1 / math.sqrt(2)) < 1e-12 and abs(cb.records[1] - 0.5) < 1e-12


def test_execute_copies_initial(cuda, mode):
    import paper_2009_01845_b200 as q

    init = _sv(np.random.default_rng(5).standard_normal(1 << 14) + 0j)
    keep = init.amplitudes
    q.qft_circuit(14).execute(init)
    assert np.array_equal(init.amplitudes, keep)


# ---------------------------------------------------------------- Trotter / adiabatic
def test_adiabatic_golden(cuda):
    import paper_2009_01845_b200 as q

    g = golden("adiabatic")
    for n in (8, 13, 14):
        dt, T = g[f"cfg{n}"]
        st = q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 1.0), q.Schedule.linear(),
                                q.EvolutionConfig(q.Solver.TROTTER, float(dt), float(T)))
        assert max_abs(st.amplitudes, g[f"n{n}"]) <= TOL64


def test_trotter_expectation_matches_oracle(cuda):
    import paper_2009_01845_b200 as q

    n = 10
    rng = np.random.default_rng(3)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    h = q.build_tfim(n, 0.7)
    want = 0.0
    for qs, m in h.terms:
        t = psi.copy()
        ov.apply_matrix(t, n, qs, m)
        want += np.vdot(psi, t).real
    assert abs(q.expectation(h, _sv(psi)) - want) <= 1e-12


# ---------------------------------------------------------------- measurement
def test_marginals_and_samples_bitwise(cuda):
    import paper_2009_01845_b200 as q

    g = golden("sampling")
    st = _sv(g["state"])
    for i, text in enumerate(g["subsets"]):
        qs = tuple(json.loads(str(text)))
        assert np.array_equal(q.marginal_probabilities(st, qs), g[f"marg{i}"]), qs
        assert np.array_equal(q.sample(st, qs, 2000, seed=100 + i).samples, g[f"samp{i}"]), qs
    f32 = q.StateVector(12, g["state"].astype(np.complex64), q.Precision.F32)
    assert np.array_equal(q.marginal_probabilities(f32, (0, 3, 5)), g["marg_f32"])
    assert np.array_equal(q.sample(f32, (0, 3, 5), 1000, seed=9).samples, g["samp_f32"])


@pytest.mark.parametrize("nq,shots,seed", [(3, 500, 7), (20, 100000, 42)])
def test_cli_shots_digest(cuda, nq, shots, seed):
    import paper_2009_01845_b200 as q

    g = golden("sampling")
    st = q.Circuit(nq).add([q.H(k) for k in range(nq)]).execute()
    res = q.sample(st, range(nq), shots, seed)
    assert hashlib.sha256(res.samples.tobytes()).hexdigest() == str(g[f"digest_{nq}_{shots}_{seed}"])


@pytest.mark.parametrize("n,kind", [(16, "random"), (20, "random"), (20, "qft"), (22, "sparse"), (21, "tiny"),
                                    (24, "uniform"), (24, "near_uniform"), (25, "random")])
def test_exact_parallel_cumsum_equals_sequential(cuda, n, kind):
    import torch

    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import _native as nat
    from paper_2009_01845_b200.measurement import device_cdf

    rng = np.random.default_rng(n)
    if kind == "random":
        p = rng.random(1 << n) ** 3
    elif kind == "qft":
        st = q.qft_circuit(n).execute(q.basis_state(n, 12345))
        p = np.abs(st.amplitudes) ** 2
    elif kind == "sparse":
        p = rng.random(1 << n) * (rng.random(1 << n) < 0.01)
        p[:1000] = 0.0
    elif kind == "uniform":  # prefixes hit powers of two exactly
        p = np.full(1 << n, 2.0 ** -n)
    elif kind == "near_uniform":  # prefixes graze powers of two
        p = (1.0 + 1e-13 * rng.standard_normal(1 << n)) * 2.0 ** -n
    else:
        p = rng.random(1 << n) * 10.0 ** rng.integers(-300, 1, 1 << n)
    want = np.cumsum(p)
    want /= want[-1]
    dp = torch.from_numpy(p).cuda()
    got = device_cdf(dp).cpu().numpy()
    assert np.array_equal(got, want)
    ser = torch.empty_like(dp)
    nat.check(nat.lib().qsb_cumsum_serial(dp.data_ptr(), dp.numel(), ser.data_ptr(), nat.stream_ptr()))
    assert np.array_equal(ser.cpu().numpy(), np.cumsum(p))


def test_large_sample_converges(cuda):
    import paper_2009_01845_b200 as q

    st = q.Circuit(3).add([q.H(k) for k in range(3)]).execute()
    res = q.sample(st, (0, 1, 2), 1_000_000, seed=13)
    freq = q.frequencies(res)
    sigma = math.sqrt(1e6 * 0.125 * 0.875)
    for o in range(8):
        assert abs(freq.get(o, 0) - 125000) <= 6 * sigma


# ---------------------------------------------------------------- size-independent properties
@pytest.mark.parametrize("n", [24, 26])
def test_qft_inverse_round_trip_and_norm(cuda, n, mode):
    import paper_2009_01845_b200 as q

    rng = np.random.default_rng(n)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    st = _sv(psi)
    nrm0 = q.norm(st)
    c = q.qft_circuit(n)
    fwd = c.execute(st)
    assert abs(q.norm(fwd) - nrm0) <= 1e-10
    back = c.inverse().execute(fwd)
    assert max_abs(back.amplitudes, psi) <= 1e-12


def test_fused_equals_unfused_random_large(cuda, mode):
    import paper_2009_01845_b200 as q

    n = 20
    rng = np.random.default_rng(77)
    specs = []
    for _ in range(200):
        spec = _random_spec(q, n, rng)
        specs.append(spec)
    c = q.Circuit(n).add(specs)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    a = c.execute(_sv(psi), fuse=True).amplitudes
    b = c.execute(_sv(psi), fuse=False).amplitudes
    want = ov.run([ov.gate("Unitary", s.targets, s.controls, (), q.gate_matrix(s)) for s in specs], n, psi)
    assert max_abs(a, want) <= TOL64 and max_abs(b, want) <= TOL64


def _random_spec(q, n, rng):
    kinds = ["H", "RX", "RZ", "CZPow", "CNOT", "CZ", "SWAP", "U1", "U2", "Y"]
    k = kinds[rng.integers(len(kinds))]
    order = rng.permutation(n)
    two = k in ("CZPow", "CNOT", "CZ", "SWAP", "U2")
    tg = tuple(int(x) for x in order[: 2 if two else 1])
    ct = tuple(int(x) for x in order[len(tg): len(tg) + int(rng.integers(0, 3))])
    th = float(rng.uniform(0, 2 * math.pi))
    if k == "U1":
        m, _ = np.linalg.qr(rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2)))
        return q.Unitary(m, *tg, controls=ct)
    if k == "U2":
        m, _ = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
        return q.Unitary(m, *tg, controls=ct)
    if k in ("RX", "RZ"):
        return getattr(q, k)(tg[0], th, controls=ct)
    if k == "CZPow":
        return q.CZPow(tg[0], tg[1], th, controls=ct)
    if k in ("H", "Y"):
        return getattr(q, k)(tg[0], controls=ct)
    return getattr(q, k)(tg[0], tg[1], controls=ct)


@pytest.mark.parametrize("n,qubits,prec", [(12, (3,), "f64"), (14, (0, 5, 13), "f64"), (16, (2, 9), "f32")])
def test_collapse_and_measure(cuda, n, qubits, prec):
    """Projective collapse against a numpy projection (extension: no reference semantics)."""
    import paper_2009_01845_b200 as q

    rng = np.random.default_rng(n)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    P = q.Precision.F64 if prec == "f64" else q.Precision.F32
    tol = 1e-12 if prec == "f64" else 1e-5
    st = q.from_amplitudes(psi, precision=P)
    k = len(qubits)
    outcome = (1 << k) - 2 if k > 1 else 1
    p = q.collapse(st, qubits, outcome)
    idx = np.arange(1 << n)
    keep = np.ones(1 << n, dtype=bool)
    for j, qb in enumerate(qubits):
        keep &= ((idx >> (n - 1 - qb)) & 1) == ((outcome >> (k - 1 - j)) & 1)
    want = np.where(keep, psi, 0) / np.sqrt(np.sum(np.abs(psi[keep]) ** 2))
    assert abs(p - np.sum(np.abs(psi[keep]) ** 2)) <= 1e-6
    assert max_abs(st.amplitudes, want) <= tol
    # measure = one draw of sample() + collapse; a second measurement repeats the outcome
    st2 = q.from_amplitudes(psi, precision=P)
    o = q.measure(st2, qubits, seed=3)
    assert o == int(q.sample(q.from_amplitudes(psi, precision=P), qubits, 1, 3).samples[0])
    assert q.measure(st2, qubits, seed=11) == o
    assert abs(q.norm(st2) - 1.0) <= (1e-12 if prec == "f64" else 1e-5)


def test_interpreted_pass_kernel_without_nvrtc(cuda, monkeypatch):
    """With NVRTC unavailable the same plans run on the interpreted pass kernel (csrc/pass.cu,
    its own 512-thread geometry) -- still the CUDA path, still parity-exact."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import jit

    monkeypatch.setattr(jit, "_disabled", True)
    monkeypatch.setattr(jit, "_avail", None)
    assert not jit.available()
    g = golden("qft")
    n = 14
    c = q.qft_circuit(n)
    assert c.plan().n_passes >= 1
    assert max_abs(c.execute(_sv(g[f"rin{n}"])).amplitudes, g[f"rout{n}"]) <= TOL64
    gv = golden("variational")
    vc = q.variational_circuit(14, 3, gv["params14"], fused=True)
    assert max_abs(vc.execute().amplitudes, gv["f64_14_1"]) <= TOL64
    assert max_abs(vc.execute(precision=q.Precision.F32).amplitudes, gv["f32_14_1"]) <= TOL32
    g15 = golden("grid15")
    assert max_abs(circuit_from_json(g15["circuit"]).execute().amplitudes, g15["out"]) <= TOL64


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_expectation_fused_terms(cuda, prec):
    """qsb_expect_terms: mixed 1-/2-qubit terms, reversed target order, > 64 terms (chunked),
    complex64 states read in float64 exactly as the reference's astype(complex128)."""
    import paper_2009_01845_b200 as q

    n = 14
    rng = np.random.default_rng(11)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    P = q.Precision.F64 if prec == "f64" else q.Precision.F32
    st = q.from_amplitudes(psi, precision=P)
    base = st.amplitudes.astype(np.complex128)
    terms = []
    for i in range(n):
        a = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
        terms.append(((i,), a + a.conj().T))
    for i in range(n):
        for j in ((i + 3) % n, (i + 5) % n, (i + 1) % n, (i + 7) % n):
            b = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
            terms.append(((j, i), b + b.conj().T))
    h = q.TrotterHamiltonian(n, terms)
    want = 0.0
    for qs, m in h.terms:
        t = base.copy()
        ov.apply_matrix(t, n, qs, m)
        want += np.vdot(base, t).real
    assert len(h.terms) > 64
    assert abs(q.expectation(h, st) - want) <= 1e-10 * max(1.0, abs(want))


@pytest.mark.parametrize("nq,shots,seed", [(3, 500, 7), (20, 100000, 42)])
def test_cli_shots_record_digest(cuda, capsys, nq, shots, seed):
    """`python -m paper_2009_01845_b200.cli shots` prints the reference's record with the
    reference CLI's sample digest (SURVEY.md 8(c) golden values)."""
    from paper_2009_01845_b200 import cli

    g = golden("sampling")
    assert cli.main(["shots", "--nqubits", str(nq), "--nshots", str(shots), "--seed", str(seed)]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["benchmark"] == "shots" and rec["n_shots"] == shots
    assert rec["sample_digest"] == str(g[f"digest_{nq}_{shots}_{seed}"])


def test_cli_qft_verify_and_evolve(cuda, capsys):
    from paper_2009_01845_b200 import cli

    assert cli.main(["qft", "--nqubits", "16", "--verify"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["verify_max_abs_diff"] <= 1e-12 and rec["passes"] >= 1
    assert cli.main(["evolve", "--nqubits", "8", "--dt", "0.1", "--T", "0.5"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["solver"] == "trotter" and np.isfinite(rec["final_energy"])


@pytest.mark.parametrize("partition", [(0,), (3, 1), (0, 2, 4, 6), (1, 2, 3, 5, 7, 8, 9)])
def test_entanglement_entropy_matches_svd(cuda, partition):
    """Device entropy (reduced-density kernel + eigvalsh on the smaller side) against the
    reference's numpy SVD."""
    import paper_2009_01845_b200 as q

    n = 10
    rng = np.random.default_rng(len(partition))
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    t = np.moveaxis(psi.reshape([2] * n), partition, range(len(partition)))
    sv = np.linalg.svd(t.reshape(1 << len(partition), -1), compute_uv=False)
    p = sv ** 2
    p = p[p > 1e-15]
    want = float(-(p * np.log2(p)).sum())
    assert abs(q.entanglement_entropy(_sv(psi), partition) - want) <= 1e-10
    # a product state has zero entropy; a Bell pair across the cut has one bit
    bell = q.Circuit(n).add([q.H(0), q.CNOT(0, 5)]).execute()
    assert abs(q.entanglement_entropy(bell, (0,)) - 1.0) <= 1e-12
    assert abs(q.entanglement_entropy(q.zero_state(n), (0, 1))) <= 1e-12


@pytest.mark.parametrize("n", [14, 20])
def test_expectation_fused_passes_match_per_term(cuda, n):
    """Fused read-only expectation passes (JIT) = the per-term kernel = numpy, for TFIM + X and
    random dense terms on far-apart qubits."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import hamiltonians as hm

    rng = np.random.default_rng(n)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    st = _sv(psi)
    terms = list(q.combine(q.build_x(n), 0.4, q.build_tfim(n, 1.0), 0.6).terms)
    for i in range(6):
        a = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
        terms.append(((i, n - 1 - i), a + a.conj().T))
    h = q.TrotterHamiltonian(n, terms)
    want = 0.0
    for qs, m in h.terms:
        t = psi.copy()
        ov.apply_matrix(t, n, qs, m)
        want += np.vdot(psi, t).real
    fused = hm._expectation_passes([(tuple(n - 1 - x for x in qs), m) for qs, m in hm._fold_single_terms(h.terms)], st)
    assert fused is not None
    assert abs(fused - want) <= 1e-10 * max(1.0, abs(want))
    assert abs(q.expectation(h, st) - want) <= 1e-10 * max(1.0, abs(want))


@pytest.mark.parametrize("n,prec", [(4, "f64"), (9, "f32"), (12, "f64"), (13, "f64"), (14, "f32"), (14, "f64"),
                                    (17, "f32"), (18, "f64"), (21, "f64"), (22, "f32"), (24, "f64")])
def test_gate_batch_equals_per_gate_kernels(cuda, n, prec):
    """qsb_apply_batch -- state in one CTA's shared memory up to 128 KB, a grid-synchronised
    walk of the state beyond that -- against the per-gate kernels (same bits) and
    the oracle; 150 gates cross the 64-gate launch boundary."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import _native as nat
    from paper_2009_01845_b200 import engine
    from paper_2009_01845_b200.fusion import normalize

    rng = np.random.default_rng(1000 + n)
    specs = [_random_spec(q, n, rng) for _ in range(150)]
    ngates = [g for g in (normalize(s, n, i) for i, s in enumerate(specs)) if g is not None]
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    precision = q.Precision(prec)
    a = q.from_amplitudes(psi, precision=precision)
    b = q.from_amplitudes(psi, precision=precision)
    dtype = precision.qsb_dtype
    engine._apply_gate_batch(a.data_ptr, n, dtype, engine.pack_gate_batch(ngates), nat.stream_ptr())
    for g in ngates:
        engine._apply_gate_step(b.data_ptr, n, dtype, g, nat.stream_ptr())
    # same bodies, same operand order, contraction spelled out in cmul: the same bits
    assert np.array_equal(a.amplitudes, b.amplitudes)
    if n <= 18:
        want = ov.run([ov.gate("Unitary", s.targets, s.controls, (), q.gate_matrix(s)) for s in specs], n, psi)
        tol = TOL64 if prec == "f64" else TOL32
        assert max_abs(a.amplitudes, want) <= tol


def test_gate_batch_small_states_and_limits(cuda):
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import _native as nat
    from paper_2009_01845_b200 import engine
    from paper_2009_01845_b200.errors import CapacityError, ShapeError
    from paper_2009_01845_b200.fusion import normalize

    # 1 and 2 qubits through Circuit.execute (the small-state path runs every stand-alone run)
    for n, specs in ((1, [q.H(0), q.RX(0, 0.3), q.Y(0), q.RZ(0, 1.1)]),
                     (2, [q.H(0), q.CNOT(0, 1), q.RY(1, 0.7), q.SWAP(0, 1), q.CZPow(0, 1, 0.4)])):
        got = q.Circuit(n).add(specs).execute().amplitudes
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1
        want = ov.run([ov.gate("Unitary", s.targets, s.controls, (), q.gate_matrix(s)) for s in specs], n, psi)
        assert max_abs(got, want) <= TOL64
    big = q.zero_state(27)  # 2 GB complex128: beyond the grid walk's limit
    g = [normalize(q.H(0), 27)]
    with pytest.raises(CapacityError):
        engine._apply_gate_batch(big.data_ptr, 27, nat.QSB_C128, engine.pack_gate_batch(g), nat.stream_ptr())
    del big
    small = q.zero_state(5)
    bad = engine.pack_gate_batch([normalize(q.SWAP(0, 1), 5)])
    bad[1][1] = bad[1][0]  # duplicate target bit: rejected before any launch
    with pytest.raises(ShapeError):
        engine._apply_gate_batch(small.data_ptr, 5, nat.QSB_C128, bad, nat.stream_ptr())
    assert np.array_equal(small.amplitudes, np.eye(1, 32, dtype=np.complex128)[0])


@pytest.mark.parametrize("n", [16, 20, 24])
def test_mid_size_first_run_batched_then_planned(cuda, n):
    """A mid-size circuit runs through the grid-synchronised batch first (run_gates returns no
    plan), then as planned fused passes; both match the analytic DFT column."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import engine

    k = 12345 % (1 << n)
    c = q.qft_circuit(n)
    cache = {}
    outs = []
    for expect_plan in (False, True, True):
        st = q.basis_state(n, k)
        plan = engine.run_gates(st, c.queue, None, {}, cache)
        assert (plan is not None) == expect_plan
        outs.append(st.amplitudes)
    j = np.arange(1 << n, dtype=np.float64)
    want = np.exp(2j * np.pi * ((j * k) % (1 << n)) / (1 << n)) / np.sqrt(1 << n)
    for o in outs:
        assert max_abs(o, want) <= 1e-12
    # a prepared plan is used from the first run
    c2 = q.qft_circuit(n)
    cache2 = {}
    engine.prepare_plan(n, q.Precision.F64, c2.queue, None, cache2)
    assert engine.run_gates(q.basis_state(n, k), c2.queue, None, {}, cache2) is not None


@pytest.mark.parametrize("n", [10, 16])
def test_execution_is_cuda_graph_capturable(cuda, n):
    """Gate tables and pass coefficients travel as kernel parameters (no host staging in the
    launch path), so a planned circuit -- shared-memory batch (n = 10) or fused specialised
    passes (n = 16) -- can be captured once in a CUDA graph and replayed on new inputs."""
    import torch

    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import engine

    c = q.variational_circuit(n, 3, np.random.default_rng(n).uniform(0, 6, n * 7), fused=True)
    cache = {}
    if n > 13:
        engine.prepare_plan(n, q.Precision.F64, c.queue, None, cache)
    st = q.zero_state(n)
    engine.run_gates(st, c.queue, None, {}, cache)  # warm: packing / module loads outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    src = st.tensor  # out-of-place passes may leave the result in the captured scratch buffer
    with torch.cuda.stream(stream):
        with torch.cuda.graph(graph, stream=stream):
            engine.run_gates(st, c.queue, None, {}, cache)
    dst = st.tensor
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    for _ in range(2):
        psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
        src.copy_(torch.from_numpy(psi).to(src.device))
        graph.replay()
        torch.cuda.synchronize()
        want = c.execute(_sv(psi)).amplitudes
        assert max_abs(dst.cpu().numpy(), want) <= TOL64


@pytest.mark.parametrize("n,prec", [(8, "f64"), (16, "f32"), (20, "f64")])
def test_circuit_graph_replay(cuda, n, prec):
    """Circuit.capture: execute() contract (default |0..0>, initial copied) from a graph replay."""
    import paper_2009_01845_b200 as q

    precision = q.Precision(prec)
    c = q.variational_circuit(n, 2, np.random.default_rng(n).uniform(0, 6, n * 5), fused=False)
    g = c.capture(precision)
    tol = TOL64 if prec == "f64" else TOL32
    assert max_abs(g.execute().amplitudes, c.execute(precision=precision).amplitudes) <= tol
    rng = np.random.default_rng(5)
    for _ in range(2):
        psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
        init = q.from_amplitudes(psi, precision=precision)
        keep = init.amplitudes
        a = g.execute(init)
        b = c.execute(init, precision=precision)
        assert max_abs(a.amplitudes, b.amplitudes) <= tol
        assert np.array_equal(init.amplitudes, keep)
    with pytest.raises(q.ShapeError):
        g.execute(q.zero_state(n + 1, precision))


def _cached_plans(circuit):
    from paper_2009_01845_b200.fusion import Plan

    return [v[0] for v in circuit.__dict__.get("_plan_cache", {}).values() if isinstance(v[0], Plan)]


def _staged_table_bytes(plan):
    from paper_2009_01845_b200.fusion import PassStep

    return sum(-(-8 * len(s.jit[1][1]) // 256) * 256 for s in plan.steps
               if isinstance(s, PassStep) and s.jit is not None)


def test_captured_qft_replays_after_ring_wraps(cuda):
    """A captured QFT (fused passes with pivot tables) replays correctly after more than the
    library's 16 MB host-staging ring has been cycled by other circuits: the graph's passes read
    their tables from device buffers the plan owns, never from a ring slot."""
    import paper_2009_01845_b200 as q

    n = 16
    c = q.qft_circuit(n)
    g = c.capture()
    (plan,) = _cached_plans(c)
    assert _staged_table_bytes(plan) > 0, "QFT passes should carry pivot tables"
    rng = np.random.default_rng(11)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    want = ov.run(ov.qft(n), n, psi)
    assert max_abs(g.execute(_sv(psi)).amplitudes, want) <= TOL64
    other = q.qft_circuit(20)
    st = q.zero_state(20)
    other.execute(st)
    other.execute(st)  # planned from the second run on
    per_run = _staged_table_bytes(_cached_plans(other)[0])
    assert per_run > 0
    for _ in range((40 << 20) // per_run + 1):  # > 2 wraps of the 16 MB ring
        other.execute(st)
    assert max_abs(g.execute(_sv(psi)).amplitudes, want) <= TOL64


def test_concurrent_small_executes_from_threads(cuda):
    """ctypes drops the GIL around library calls: batched small-state executes from several host
    threads (thread-local gate tables, locked setup) give the single-threaded results."""
    import threading

    import paper_2009_01845_b200 as q

    circuits = [q.variational_circuit(n, 3, np.random.default_rng(n + 7 * k).uniform(0, 6, n * 7), fused=k % 2 == 0)
                for k in range(4) for n in (6, 12, 16)]
    want = [c.execute().amplitudes for c in circuits]
    got = [None] * len(circuits)
    errors = []

    def work(idx):
        try:
            for _ in range(5):
                for i in idx:
                    got[i] = q.Circuit(circuits[i].n_qubits).add(list(circuits[i].queue)).execute().amplitudes
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(list(range(t, len(circuits), 3)),)) for t in range(3)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_expectation_fused_passes_complex64(cuda):
    """complex64 states: fused read-only expectation passes (double accumulation) = numpy."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import hamiltonians as hm

    n = 16
    rng = np.random.default_rng(6)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(np.complex64)
    psi /= np.linalg.norm(psi)
    st = q.from_amplitudes(psi)
    h = q.combine(q.build_x(n), 0.4, q.build_tfim(n, 1.0), 0.6)
    p64 = psi.astype(np.complex128)
    want = 0.0
    for qs, m in h.terms:
        t = p64.copy()
        ov.apply_matrix(t, n, qs, m)
        want += np.vdot(p64, t).real
    bits = [(tuple(n - 1 - x for x in qs), m) for qs, m in hm._fold_single_terms(h.terms)]
    fused = hm._expectation_passes(bits, st)
    assert fused is not None
    assert abs(fused - want) <= 1e-9 * max(1.0, abs(want))
    assert abs(q.expectation(h, st) - want) <= 1e-9 * max(1.0, abs(want))


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_marginal_from_amplitudes_equals_probability_path(cuda, prec):
    """qsb_marginal_amps (leaf sums formed from the amplitudes) = qsb_probabilities +
    qsb_marginal, bit for bit, for subsets that leave the 8 lowest bits reduced."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import _native as nat
    from paper_2009_01845_b200 import measurement as ms

    n = 20
    rng = np.random.default_rng(12)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    st = q.from_amplitudes(psi, precision=q.Precision(prec))
    probs = ms.device_probabilities(st)
    for qubits in ((0,), (3, 1), (11, 0, 5), tuple(range(12)), (7, 2, 9, 4)):
        fused = ms.device_marginal(st, qubits).cpu().numpy()
        k = len(qubits)
        kept = np.array([n - 1 - x for x in qubits], dtype=np.int32)
        out = ms._f64(1 << k)
        scratch = ms._f64(int(nat.lib().qsb_marginal_scratch_doubles(n, k)))
        nat.check(nat.lib().qsb_marginal(probs.data_ptr(), n, k, kept.ctypes.data, out.data_ptr(), scratch.data_ptr(),
                                         nat.stream_ptr()))
        assert np.array_equal(fused, out.cpu().numpy()), qubits
        ref = ov.marginal(st.amplitudes, n, qubits) if hasattr(ov, "marginal") else None
        if ref is not None:
            assert np.array_equal(fused, ref), qubits


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,partition", [(12, (0,)), (12, (11, 3)), (14, (13, 12, 11, 10, 9)), (14, (2, 9, 4, 0, 13, 7)),
                                         (16, tuple(range(0, 16, 2))), (17, (16, 1, 15, 2, 14, 3, 13, 4, 12, 5, 11, 6))])
def test_reduced_density_matrix_kernel(cuda, prec, n, partition):
    """qsb_reduced_density against numpy's M M^dagger of the reference's moveaxis/reshape
    (evolution.py:166-169), every tile shape (k = 1..12, partition bits low, high, mixed)."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200.evolution import reduced_density_matrix

    p = q.Precision(prec)
    rng = np.random.default_rng(n + len(partition))
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(p.complex_dtype)
    psi /= np.linalg.norm(psi)
    st = q.from_amplitudes(psi)
    m = np.moveaxis(psi.astype(np.complex128).reshape([2] * n), partition, range(len(partition)))
    m = m.reshape(1 << len(partition), -1)
    want = m @ m.conj().T
    got = reduced_density_matrix(st, partition).cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-14
    assert np.array_equal(got, got.conj().T)


def test_entanglement_entropy_large(cuda):
    """n = 24 states: a GHZ state across the cut (one bit), a product of Bell pairs (one bit per
    pair cut), and a random state's entropy against the reference's SVD."""
    import paper_2009_01845_b200 as q

    n = 24
    ghz = q.Circuit(n).add([q.H(0)] + [q.CNOT(0, k) for k in range(1, n)]).execute()
    assert abs(q.entanglement_entropy(ghz, (3, 17, 20)) - 1.0) <= 1e-12
    pairs = q.Circuit(n).add([g for k in range(0, n, 2) for g in (q.H(k), q.CNOT(k, k + 1))]).execute()
    assert abs(q.entanglement_entropy(pairs, (0, 2, 4, 7, 9)) - 5.0) <= 1e-11
    rng = np.random.default_rng(1)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    part = (1, 5, 8, 13, 22, 23)
    m = np.moveaxis(psi.reshape([2] * n), part, range(len(part))).reshape(1 << len(part), -1)
    sv = np.linalg.svd(m, compute_uv=False) ** 2
    sv = sv[sv > 1e-15]
    assert abs(q.entanglement_entropy(q.from_amplitudes(psi), part) - float(-(sv * np.log2(sv)).sum())) <= 1e-10


def test_cli_gpu_metric_fields(cuda, capsys):
    """CLI records carry the GPU metrics: device, gpus, passes,
    bytes_moved, hbm_gbps, roofline_frac; sharded runs add exchanges and their bandwidth."""
    import json

    from paper_2009_01845_b200 import cli

    assert cli.main(["qft", "--nqubits", "24"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert "B200" in rec["device"] and rec["gpus"] == 1 and rec["passes"] >= 1
    assert rec["bytes_moved"] == rec["passes"] * 2 * (1 << 24) * 16 or rec["bytes_moved"] > 0
    assert 0 < rec["hbm_gbps"] and 0 < rec["roofline_frac"] < 1.2
    assert cli.main(["variational", "--nqubits", "24", "--fuse", "--gpus", "4"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["shards"] == 4 and rec["exchanges"] >= 1 and rec["exchange_bytes"] == rec["exchanges"] * 3 * (1 << 20) * 16 // 1
    assert rec["exchange_gbps"] > 0


@pytest.mark.parametrize("kind", ["random", "sparse", "tiny", "uniform", "near_uniform", "one_hot"])
def test_sample_exact_sparse_cdf_equals_full_cdf(cuda, kind):
    """qsb_sample_exact (only the CDF blocks holding a draw are materialised) draws exactly what
    the full exact CDF + searchsorted draws, for distributions whose prefixes sit on binade
    boundaries, are mostly zero, tiny, or exactly uniform; 1 to 10^6 shots."""
    torch = cuda
    from paper_2009_01845_b200.measurement import device_cdf, device_sample, device_sample_exact

    rng = np.random.default_rng(len(kind))
    for n in (1 << 16, (1 << 20) + 123, 1 << 23):
        if kind == "random":
            p = rng.random(n)
        elif kind == "sparse":
            p = rng.random(n) * (rng.random(n) < 0.01)
        elif kind == "tiny":
            p = rng.random(n) * 1e-300
        elif kind == "uniform":
            p = np.full(n, 1.0 / n)
        elif kind == "near_uniform":
            p = np.full(n, 1.0 / n) * (1 + 1e-9 * rng.standard_normal(n))
        else:
            p = np.zeros(n)
            p[n // 3] = 1.0
        pt = torch.from_numpy(p).cuda()
        cum = device_cdf(pt)
        for shots in (1, 1000, 10 ** 6):
            for seed in (0, 7):
                a = device_sample(cum, shots, seed)
                b = device_sample_exact(pt, shots, seed)
                assert torch.equal(a, b), (kind, n, shots, seed)
