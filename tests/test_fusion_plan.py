"""CPU verification of the pass planner + program encoder (fusion.py) through the numpy
interpreter of the qsb_run_pass program format (tests/pass_emulator.py)."""

import math

import numpy as np
import pytest

from conftest import golden, max_abs
from oracle import statevec as ov
from plan_helpers import emulate_plan, spec_tuples_to_specs
from paper_2009_01845_b200 import _native as nat
from paper_2009_01845_b200.fusion import GEOMETRY, PassStep, plan_circuit

C128, C64 = nat.QSB_C128, nat.QSB_C64


def check(gates, n, psi=None, dtype=C128, tol=1e-12, allow_ext=True, min_fused=0):
    specs = spec_tuples_to_specs(gates)
    plan = plan_circuit(specs, n, dtype, allow_ext_perm=allow_ext)
    npd = np.complex128 if dtype == C128 else np.complex64
    if psi is None:
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1
    got = emulate_plan(plan, psi, npd)
    want = ov.run(gates, n, psi)
    assert max_abs(got, want) <= tol, (plan.n_passes, len(plan.steps))
    # gates not left to stand-alone kernels (folded single-qubit gates count as fused)
    stand_alone = sum(1 for s in plan.steps if not isinstance(s, PassStep))
    assert len(gates) - stand_alone >= min_fused
    return plan


@pytest.mark.parametrize("n", [13, 14, 16])
def test_qft_plan(n):
    rng = np.random.default_rng(n)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    plan = check(ov.qft(n), n, psi)
    # the QFT collapses to a handful of passes
    assert plan.n_passes <= 4


def test_qft_plan_passes_at_30_qubits():
    plan = plan_circuit(spec_tuples_to_specs(ov.qft(30)), 30, C128)
    assert plan.n_passes == 4 and all(isinstance(s, PassStep) for s in plan.steps)
    assert sum(s.n_transposes for s in plan.steps) <= 8


def test_qft_plan_without_external_permutation():
    n = 15
    rng = np.random.default_rng(3)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    plan = check(ov.qft(n), n, psi, allow_ext=False)
    assert not any(s.ext_perm for s in plan.steps if isinstance(s, PassStep))


@pytest.mark.parametrize("fused", [False, True])
def test_variational_plan(fused):
    g = golden("variational")
    n = 14
    gates = ov.variational(n, 3, g[f"params{n}"], fused=fused)
    check(gates, n, min_fused=len(gates) // 2)
    check(gates, n, dtype=C64, tol=2e-6)


def test_random_circuit_plans():
    g = golden("random_circuits")
    for i, (n, text) in enumerate(zip(g["n"], g["circuits"])):
        if n < 13:
            continue
        _, gates = ov.from_json(text)
        check(gates, int(n), g[f"in{i}"])
        check(gates, int(n), g[f"in{i}"], dtype=C64, tol=5e-6)


def test_grid_plan():
    gates = ov.grid_supremacy(3, 5, 8, seed=42)
    plan = check(gates, 15)
    assert plan.n_passes < len(gates) / 5


def test_trotter_step_plan():
    n = 16
    terms = ov.combine(ov.x_terms(n), 0.4, ov.tfim_terms(n, 1.0), 0.6)
    gates = ov.trotter_step(terms, 0.05)
    rng = np.random.default_rng(5)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    plan = check(gates, n, psi)
    assert plan.n_passes <= 6


def test_controlled_and_mixed_gates():
    n = 14
    rng = np.random.default_rng(11)
    gates = []
    for _ in range(80):
        kinds = ["H", "X", "Y", "Z", "RX", "RZ", "CZPow", "CNOT", "CZ", "SWAP", "U1", "U2"]
        k = kinds[rng.integers(len(kinds))]
        order = rng.permutation(n)
        t2 = k in ("CZPow", "CNOT", "CZ", "SWAP", "U2")
        tg = tuple(int(x) for x in order[: 2 if t2 else 1])
        nc = int(rng.integers(0, 3))
        ct = tuple(int(x) for x in order[len(tg): len(tg) + nc])
        th = float(rng.uniform(0, 2 * math.pi))
        if k == "U1":
            q, _ = np.linalg.qr(rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2)))
            gates.append(ov.gate("Unitary", tg, ct, (), q))
        elif k == "U2":
            q, _ = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
            gates.append(ov.gate("Unitary", tg, ct, (), q))
        elif k in ("RX", "RZ", "CZPow"):
            gates.append(ov.gate(k, tg, ct, (th,)))
        else:
            gates.append(ov.gate(k, tg, ct))
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    check(gates, n, psi)


def test_geometry():
    for dt, geo in GEOMETRY.items():
        assert geo.K - geo.nreg == 9 and geo.A == 1 << geo.nreg
        # 2^L amplitudes per contiguous run = 256 bytes
        assert (1 << geo.L) * (16 if dt == C128 else 8) == 256


@pytest.mark.parametrize("dtype,tol", [(C128, 1e-12), (C64, 1e-5)])
def test_single_qubit_folding_trotter_and_grid(dtype, tol):
    """1-qubit gates folded into neighbouring 2-qubit gates (cost model) keep the state."""
    from paper_2009_01845_b200.fusion import GEOMETRY_JIT, merge_single_qubit, normalize

    n = 16
    rng = np.random.default_rng(5)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    npd = np.complex128 if dtype == C128 else np.complex64
    trot = ov.trotter_step(ov.combine(ov.x_terms(n), 0.3, ov.tfim_terms(n, 1.0), 0.7), 0.1)
    for gates in (trot, ov.grid_supremacy(4, 4, 8, 42)):
        specs = spec_tuples_to_specs(gates)
        plan = plan_circuit(specs, n, dtype, geometry=GEOMETRY_JIT[dtype])
        assert max_abs(emulate_plan(plan, psi, npd), ov.run(gates, n, psi)) <= tol
    ng = [g for g in (normalize(s, n, i) for i, s in enumerate(spec_tuples_to_specs(trot))) if g is not None]
    # the X rotation on each ZZ+hX term's first qubit folds into it: 56 -> 40 gates at n = 16
    assert len(merge_single_qubit(ng)) < len(ng)


@pytest.mark.parametrize("dtype,tol", [(C128, 1e-12), (C64, 1e-5)])
def test_unfused_variational_sandwiches_become_dense(dtype, tol):
    """RY RY . CZ . RY RY around each even CZ folds into one dense 4x4 (the VariationalLayer
    form); the QFT's diagonals stay diagonal."""
    from paper_2009_01845_b200 import gate_matrix, qft_circuit, variational_circuit
    from paper_2009_01845_b200.fusion import GEOMETRY_JIT, normalize, sandwich_diagonals

    n = 14
    rng = np.random.default_rng(4)
    params = rng.uniform(0, 6, n * 7)
    c = variational_circuit(n, 3, params, fused=False)
    ng = [g for g in (normalize(s, n, i) for i, s in enumerate(c.queue)) if g is not None]
    folded = sandwich_diagonals(ng)
    assert sum(g.kind == "g2" for g in folded) == 3 * n // 2
    q = qft_circuit(n)
    nq = [g for g in (normalize(s, n, i) for i, s in enumerate(q.queue)) if g is not None]
    assert sum(g.kind == "g2" for g in sandwich_diagonals(nq)) == 0
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    ref = psi.copy()
    for g in c.queue:
        ov.apply_matrix(ref, n, tuple(g.targets), gate_matrix(g), tuple(g.controls))
    plan = plan_circuit(c.queue, n, dtype, geometry=GEOMETRY_JIT[dtype])
    npd = np.complex128 if dtype == C128 else np.complex64
    assert max_abs(emulate_plan(plan, psi, npd), ref) <= tol


def test_pack_gate_batch_layout():
    """qsb_apply_batch host arrays (include/qsb200.h): 2 target bits and 32 doubles per gate,
    control bits back to back, the stand-alone kernel class of each gate kind."""
    from paper_2009_01845_b200 import CNOT, CZ, RX, SWAP, gate_matrix
    from paper_2009_01845_b200.engine import pack_gate_batch
    from paper_2009_01845_b200.fusion import normalize

    n = 6
    specs = [RX(1, 0.3, controls=(4, 2)), CZ(0, 5), SWAP(2, 3), CNOT(0, 1)]
    gates = [normalize(s, n, i) for i, s in enumerate(specs)]
    nt, tb, nc, cb, mats, kc = pack_gate_batch(gates)
    assert list(nt) == [1, 2, 2, 1]  # CNOT is a controlled X on bit 4
    assert list(tb) == [4, 0, 5, 0, 3, 2, 4, 0]
    assert list(nc) == [2, 0, 0, 1] and list(cb) == [1, 3, 5]
    assert list(kc) == [nat.KERNEL_AUTO, nat.KERNEL_DIAGONAL, nat.KERNEL_PERMUTATION, nat.KERNEL_AUTO]
    m = mats.view(np.complex128).reshape(4, 16)
    assert np.array_equal(m[0, :4], gate_matrix(specs[0]).reshape(-1))
    assert np.array_equal(m[1], np.diag([1, 1, 1, -1]).astype(np.complex128).reshape(-1))
    assert mats.dtype == np.float64 and mats.size == 32 * 4


def test_reordered_layouts_keep_the_state_and_cut_transposes():
    """Gates re-ordered inside their dependencies (fusion._reorder_events): same state as the
    oracle on a dependency-dense mix, and far fewer layout changes on the variational ansatz."""
    from paper_2009_01845_b200 import fusion, variational_circuit

    n = 14
    rng = np.random.default_rng(21)
    gates = []
    for _ in range(60):  # chains of overlapping 2-qubit gates, diagonals and controlled gates
        a = int(rng.integers(n - 1))
        k = rng.integers(4)
        if k == 0:
            q, _ = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
            gates.append(ov.gate("Unitary", (a, a + 1), (), (), q))
        elif k == 1:
            gates.append(ov.gate("CZPow", (a, a + 1), (), (float(rng.uniform(0, 6)),)))
        elif k == 2:
            gates.append(ov.gate("RX", (a,), ((a + 5) % n,), (float(rng.uniform(0, 6)),)))
        else:
            gates.append(ov.gate("RZ", (a + 1,), (), (float(rng.uniform(0, 6)),)))
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    check(gates, n, psi)
    c = variational_circuit(30, 5, np.random.default_rng(42).uniform(0, 2 * np.pi, 330), fused=True)
    geo = fusion.GEOMETRY_JIT[C128]
    on = plan_circuit(c.queue, 30, C128, geometry=geo)
    saved = fusion.REORDER_GATES
    try:
        fusion.REORDER_GATES = False
        off = plan_circuit(c.queue, 30, C128, geometry=geo)
    finally:
        fusion.REORDER_GATES = saved
    t_on = sum(s.n_transposes for s in on.steps if isinstance(s, PassStep))
    t_off = sum(s.n_transposes for s in off.steps if isinstance(s, PassStep))
    assert t_on <= 0.6 * t_off, (t_on, t_off)


@pytest.mark.parametrize("dtype,tol", [(C128, 1e-12), (C64, 1e-5)])
def test_consecutive_trotter_steps_merge_two_qubit_runs(dtype, tol):
    """Several Trotter steps planned as one circuit: the trailing half step of each step and the
    leading half step of the next (X layer in between) become one 4x4 per bit pair; also for a
    pair given in the opposite target order."""
    from paper_2009_01845_b200.fusion import GEOMETRY_JIT, merge_2q_runs, normalize

    n = 16
    rng = np.random.default_rng(6)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    npd = np.complex128 if dtype == C128 else np.complex64
    step = ov.trotter_step(ov.combine(ov.x_terms(n), 0.3, ov.tfim_terms(n, 1.0), 0.7), 0.1)
    gates = step * 3
    specs = spec_tuples_to_specs(gates)
    plan = plan_circuit(specs, n, dtype, geometry=GEOMETRY_JIT[dtype])
    assert max_abs(emulate_plan(plan, psi, npd), ov.run(gates, n, psi)) <= tol
    single = plan_circuit(spec_tuples_to_specs(step), n, dtype, geometry=GEOMETRY_JIT[dtype])
    from paper_2009_01845_b200.fusion import matrix_cost

    def fp(p):
        return sum(matrix_cost(g.matrix) for s in p.steps if isinstance(s, PassStep) for g in s.gates
                   if g.kind in ("g1", "g2"))

    assert fp(plan) < 3 * fp(single)  # the step boundaries merge
    # reversed target order on the second gate of a pair
    a, _ = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
    b, _ = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
    pair = [("Unitary", (3, 7), (), (), a), ("Unitary", (7, 3), (), (), b)]
    ng = [normalize(s, n, i) for i, s in enumerate(spec_tuples_to_specs(pair))]
    merged = merge_2q_runs(ng)
    assert len(merged) == 1
    plan = plan_circuit(spec_tuples_to_specs(pair), n, dtype, geometry=GEOMETRY_JIT[dtype])
    assert max_abs(emulate_plan(plan, psi, npd), ov.run(pair, n, psi)) <= tol


@pytest.mark.parametrize("dtype,tol", [(C128, 1e-12), (C64, 1e-5)])
def test_plan_templates_reuse_structure_with_new_coefficients(dtype, tol, monkeypatch):
    """A circuit with the structure of one planned before (time-dependent Trotter steps,
    phase circuits with new angles, variational layers with new parameters) is planned from the
    template -- merged matrices rebuilt, matrix words patched, diagonal passes re-encoded -- and
    the plan still computes the circuit; a template entry that was special (here an exact
    identity gate) but no longer is forces a fresh plan."""
    from paper_2009_01845_b200 import fusion
    from paper_2009_01845_b200.fusion import GEOMETRY_JIT

    monkeypatch.setattr(fusion, "_TEMPLATES", {})
    monkeypatch.setattr(fusion, "PLAN_TEMPLATES", True)
    n = 15
    rng = np.random.default_rng(12)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    npd = np.complex128 if dtype == C128 else np.complex64

    def trotter(s):
        return ov.trotter_step(ov.combine(ov.x_terms(n), 1 - s, ov.tfim_terms(n, 1.0), s), 0.1) * 2

    def phases(seed):
        r = np.random.default_rng(seed)
        out = []
        for q in range(n - 1):
            out.append(ov.gate("H", (q,)))
            out.append(ov.gate("CZPow", (q, q + 1), (), (float(r.uniform(0.1, 0.9)),)))
            out.append(ov.gate("RZ", (q,), (), (float(r.uniform(0.1, 3)),)))
        return out

    def layers(seed):
        r = np.random.default_rng(seed)
        out = []
        for _ in range(3):
            for q in range(n):
                out.append(ov.gate("RY", (q,), (), (float(r.uniform(0, 6)),)))
            for q in range(0, n - 1, 2):
                out.append(ov.gate("CZ", (q, q + 1)))
        return out

    for family, args in ((trotter, (0.3, 0.45, 0.8)), (phases, (1, 2)), (layers, (3, 4))):
        for k, a in enumerate(args):
            gates = family(a)
            before = dict(fusion.TEMPLATE_STATS)
            plan = plan_circuit(spec_tuples_to_specs(gates), n, dtype, geometry=GEOMETRY_JIT[dtype])
            if k > 0:
                assert fusion.TEMPLATE_STATS["hits"] == before["hits"] + 1
            assert max_abs(emulate_plan(plan, psi, npd), ov.run(gates, n, psi)) <= tol
    # s = 0 (the ZZ terms vanish, the term exponentials become exact identities): planned afresh
    before = dict(fusion.TEMPLATE_STATS)
    gates = trotter(0.0)
    plan = plan_circuit(spec_tuples_to_specs(gates), n, dtype, geometry=GEOMETRY_JIT[dtype])
    assert fusion.TEMPLATE_STATS["hits"] == before["hits"]
    assert max_abs(emulate_plan(plan, psi, npd), ov.run(gates, n, psi)) <= tol
    # ... and a template whose rotations were exact identities (dropped) does not serve the same
    # circuit with non-zero angles
    fusion._TEMPLATES.clear()
    zero = [ov.gate(g[0], g[1], g[2], (0.0,) if g[0] == "RY" else g[3]) for g in layers(3)]
    plan_circuit(spec_tuples_to_specs(zero), n, dtype, geometry=GEOMETRY_JIT[dtype])
    before = dict(fusion.TEMPLATE_STATS)
    gates = layers(4)
    plan = plan_circuit(spec_tuples_to_specs(gates), n, dtype, geometry=GEOMETRY_JIT[dtype])
    assert fusion.TEMPLATE_STATS["hits"] == before["hits"]
    assert max_abs(emulate_plan(plan, psi, npd), ov.run(gates, n, psi)) <= tol


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_plan_templates_on_mixed_random_structures(seed, monkeypatch):
    """Random circuits of mixed gate kinds (dense 1- and 2-qubit unitaries, controlled
    rotations, phase gates, SWAPs): the same structure with fresh parameters is planned from
    the template and still equals the oracle."""
    from paper_2009_01845_b200 import fusion
    from paper_2009_01845_b200.fusion import GEOMETRY_JIT

    monkeypatch.setattr(fusion, "_TEMPLATES", {})
    n = 14
    rng = np.random.default_rng(100 + seed)
    layout = []
    for _ in range(70):
        a = int(rng.integers(n - 1))
        layout.append((int(rng.integers(6)), a, int(rng.integers(n))))

    def build(r):
        out = []
        for kind, a, c in layout:
            if kind == 0:
                u, _ = np.linalg.qr(r.standard_normal((4, 4)) + 1j * r.standard_normal((4, 4)))
                out.append(ov.gate("Unitary", (a, a + 1), (), (), u))
            elif kind == 1:
                u, _ = np.linalg.qr(r.standard_normal((2, 2)) + 1j * r.standard_normal((2, 2)))
                out.append(ov.gate("Unitary", (a,), (), (), u))
            elif kind == 2 and c not in (a,):
                out.append(ov.gate("RX", (a,), (c,), (float(r.uniform(0.1, 6)),)))
            elif kind == 3:
                out.append(ov.gate("CZPow", (a, a + 1), (), (float(r.uniform(0.1, 0.9)),)))
            elif kind == 4:
                out.append(ov.gate("SWAP", (a, (a + 3) % n)))
            else:
                out.append(ov.gate("RZ", (a,), (), (float(r.uniform(0.1, 6)),)))
        return out

    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    for k in range(3):
        gates = build(np.random.default_rng(seed * 10 + k))
        before = fusion.TEMPLATE_STATS["hits"]
        plan = plan_circuit(spec_tuples_to_specs(gates), n, C128, geometry=GEOMETRY_JIT[C128])
        if k > 0:
            assert fusion.TEMPLATE_STATS["hits"] == before + 1
        assert max_abs(emulate_plan(plan, psi), ov.run(gates, n, psi)) <= 1e-12
