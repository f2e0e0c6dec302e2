"""Host-side API parity with the reference (no GPU): gate specs, matrices, kernel classes,
expanded matrices, host fusion, builders, JSON, validation errors."""

import json
import math

import numpy as np
import pytest

from oracle import statevec as ov
from paper_2009_01845_b200 import (
    CNOT, CZ, RX, RY, RZ, SWAP, ArityError, Circuit, CZPow, GateKind, GateSpec, H, KernelClass, ParseError,
    ShapeError, Unitary, VariationalLayer, X, Y, Z, CapacityError, circuit_from_dict, circuit_to_dict,
    classify_kernel, expanded_matrix, fuse, gate_matrix, qft_circuit, variational_circuit,
)


@pytest.mark.parametrize("spec,kind,params", [
    (H(0), "H", ()), (X(0), "X", ()), (Y(0), "Y", ()), (Z(0), "Z", ()), (RX(0, 0.7), "RX", (0.7,)),
    (RY(0, -1.3), "RY", (-1.3,)), (RZ(0, 2.1), "RZ", (2.1,)), (CZPow(0, 1, 0.4), "CZPow", (0.4,)),
    (CNOT(0, 1), "CNOT", ()), (CZ(0, 1), "CZ", ()), (SWAP(0, 1), "SWAP", ()),
    (VariationalLayer(0, 1, (0.3, 1.1, -0.7, 2.0)), "VariationalLayer", (0.3, 1.1, -0.7, 2.0)),
])
def test_matrices_bitwise_equal_to_oracle(spec, kind, params):
    assert np.array_equal(gate_matrix(spec), ov.matrix_of(kind, params))


def test_classification():
    assert classify_kernel(gate_matrix(H(0))) is KernelClass.GENERAL
    for s in (Z(0), RZ(0, 0.4), CZ(0, 1), CZPow(0, 1, 0.4)):
        assert classify_kernel(gate_matrix(s)) is KernelClass.DIAGONAL
    for s in (X(0), CNOT(0, 1), SWAP(0, 1), Y(0)):
        assert classify_kernel(gate_matrix(s)) is KernelClass.PERMUTATION
    assert classify_kernel(gate_matrix(RY(0, 1.0))) is KernelClass.GENERAL


def test_spec_validation():
    with pytest.raises(ShapeError):
        GateSpec(GateKind.SWAP, (1, 1))
    with pytest.raises(ShapeError):
        CNOT(0, 1, controls=(1,))
    with pytest.raises(ShapeError):
        H(-1)
    with pytest.raises(ArityError):
        GateSpec(GateKind.RY, (0,), params=())
    with pytest.raises(ArityError):
        GateSpec(GateKind.H, (0,), params=(0.1,))
    with pytest.raises(ValueError):
        GateSpec(GateKind.UNITARY, (0,))
    with pytest.raises(ValueError):
        Unitary(np.array([[1, 0], [0, 2]]), 0)
    with pytest.raises(ShapeError):
        Unitary(np.eye(4), 0)


def test_adjoint_and_rebinding():
    layer = VariationalLayer(0, 1, (0.1, 0.2, 0.3, 0.4))
    assert np.array_equal(layer.with_params((0.5, 0.6, 0.7, 0.8)).matrix,
                          VariationalLayer(0, 1, (0.5, 0.6, 0.7, 0.8)).matrix)
    assert RY(0, 0.3).adjoint().params == (-0.3,)
    u = Unitary(ov.ry(0.9), 2)
    assert np.allclose(gate_matrix(u.adjoint()) @ gate_matrix(u), np.eye(2))


def test_expanded_matrix():
    assert np.allclose(expanded_matrix(H(0), (0, 1)), np.kron(gate_matrix(H(0)), np.eye(2)))
    assert np.allclose(expanded_matrix(H(0), (1, 0)), np.kron(np.eye(2), gate_matrix(H(0))))
    assert np.allclose(expanded_matrix(X(1, controls=(0,)), (0, 1)), gate_matrix(CNOT(0, 1)))


def test_qft_structure():
    kinds = [g.kind for g in qft_circuit(3).queue]
    assert kinds.count(GateKind.H) == 3 and kinds.count(GateKind.CZPOW) == 3 and kinds.count(GateKind.SWAP) == 1
    assert len(qft_circuit(30).queue) == 480
    for mine, ref in zip(qft_circuit(9).queue, ov.qft(9)):
        assert mine.targets == ref[1] and np.array_equal(gate_matrix(mine), ref[4])


def test_variational_structure_and_params():
    params = np.random.default_rng(42).uniform(0, 2 * np.pi, 30 * 11)
    for fused, count in ((False, 480), (True, 180)):
        c = variational_circuit(30, 5, params, fused=fused)
        assert len(c.queue) == count
        for mine, ref in zip(c.queue, ov.variational(30, 5, params, fused=fused)):
            assert mine.targets == ref[1] and np.array_equal(gate_matrix(mine), ref[4])
    with pytest.raises(ShapeError):
        variational_circuit(3, 1, np.zeros(9))
    with pytest.raises(ArityError):
        variational_circuit(4, 5, np.zeros(43))


def test_host_fuse_semantics_match_reference_matrices():
    # fuse() is host matrix algebra; compare the fused matrices with a brute-force product
    c = Circuit(4).add([H(0), RY(1, 0.3), CZ(0, 1), RX(1, 0.2), H(2), CNOT(2, 3), Z(3)])
    f = fuse(c)
    assert len(f.queue) <= len(c.queue)
    psi = np.random.default_rng(1).standard_normal(16) + 0j
    want = ov.run([ov.gate(g.kind.value, g.targets, g.controls, g.params) for g in c.queue], 4, psi)
    got = ov.run([ov.gate("Unitary", g.targets, g.controls, (), gate_matrix(g)) for g in f.queue], 4, psi)
    assert np.max(np.abs(want - got)) <= 1e-12


def test_json_round_trip_and_errors():
    c = Circuit(3).add([H(0), RX(1, 0.3, controls=(0,)), Unitary(ov.rx(0.4), 2), CZPow(0, 2, 0.2)])
    back = circuit_from_dict(json.loads(json.dumps(circuit_to_dict(c))))
    assert back.queue == c.queue
    with pytest.raises(ParseError):
        circuit_from_dict({"nqubits": 2})
    with pytest.raises(ParseError):
        circuit_from_dict({"nqubits": 2, "gates": [{"name": "Nope", "targets": [0]}]})
    with pytest.raises(ParseError):
        circuit_from_dict({"nqubits": 2, "gates": [{"name": "RY", "targets": [0]}]})


def test_circuit_validation_and_cap():
    with pytest.raises(ShapeError):
        Circuit(2).add(H(2))
    with pytest.raises(CapacityError):
        Circuit(35)
    c = Circuit(4).add([RY(0, 0.1), VariationalLayer(1, 2, (0.1, 0.2, 0.3, 0.4))])
    assert c.parameter_count == 5
    c.set_parameters(np.zeros(5))
    with pytest.raises(ArityError):
        c.set_parameters(np.zeros(4))
    inv = c.inverse()
    assert [g.targets for g in inv.queue] == [g.targets for g in reversed(c.queue)]


def test_trotter_step_circuit_structure():
    from paper_2009_01845_b200 import build_tfim, build_x, combine, trotter_step_circuit

    h = combine(build_x(4), 0.5, build_tfim(4, 1.0), 0.5)
    c = trotter_step_circuit(h, 0.1)
    terms = ov.combine(ov.x_terms(4), 0.5, ov.tfim_terms(4, 1.0), 0.5)
    ref = ov.trotter_step(terms, 0.1)
    assert len(c.queue) == len(ref) == 14
    for mine, r in zip(c.queue, ref):
        assert mine.targets == r[1] and np.array_equal(gate_matrix(mine), r[4])
    assert len(trotter_step_circuit(build_tfim(34, 1.0), 0.05).queue) > 0
    assert len(trotter_step_circuit(combine(build_x(34), 0.5, build_tfim(34, 1.0), 0.5), 0.05).queue) == 119


def test_pcg64_jump_model_matches_numpy():
    # the device sampler's PCG64 model: draw k = output(advance(s0, k + 1)) (App. B.4)
    from paper_2009_01845_b200.measurement import pcg64_seed_state

    M = 0x2360ED051FC65DA44385DF649FCCF645
    for seed in (7, 42, 123456789):
        sh, sl, ih, il = pcg64_seed_state(seed)
        s, inc = (sh << 64) | sl, (ih << 64) | il
        want = np.random.default_rng(seed).random(1000)
        for k in range(1000):
            s = (s * M + inc) % (1 << 128)
            hi, lo = s >> 64, s & ((1 << 64) - 1)
            rot = hi >> 58
            x = hi ^ lo
            raw = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
            assert (raw >> 11) * 2.0 ** -53 == want[k]


def test_numpy_abs_formula_on_this_host():
    # the device probability kernel assumes numpy's |z| is M*sqrt(fma(r, r, 1)) (App. B.1)
    rng = np.random.default_rng(0)
    z = (rng.standard_normal(4000) + 1j * rng.standard_normal(4000)) * 10.0 ** rng.integers(-30, 3, 4000)
    z[:10] = 0
    ref = np.abs(z) ** 2
    re, im = np.abs(z.real), np.abs(z.imag)
    big, small = np.maximum(re, im), np.minimum(re, im)
    with np.errstate(invalid="ignore", divide="ignore"):
        r = small / big
    from fractions import Fraction

    # exactly rounded fma(r, r, 1) (math.fma needs Python 3.13)
    fma = np.array([float(Fraction(float(x)) ** 2 + 1) if np.isfinite(x) else np.nan for x in r])
    v = np.where(big == 0, 0.0, big * np.sqrt(fma))
    assert np.array_equal(v * v, ref)


def test_random_grid_builder_matches_oracle_generator():
    """The package's supremacy-style builder emits the oracle generator's gates exactly."""
    import paper_2009_01845_b200 as q
    from oracle import statevec as ov

    for rows, cols, cyc, seed in ((3, 4, 10, 42), (2, 5, 20, 7)):
        c = q.random_grid_circuit(rows, cols, cyc, seed)
        ref = ov.grid_supremacy(rows, cols, cyc, seed)
        assert len(c.queue) == len(ref)
        for g, (_k, tg, _ct, _p, m) in zip(c.queue, ref):
            assert tuple(g.targets) == tuple(tg)
            assert np.array_equal(q.gate_matrix(g), m)


def test_cli_errors_without_gpu(tmp_path, capsys):
    """Parse / form errors exit like the reference CLI (2) before any device work."""
    from paper_2009_01845_b200 import cli

    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["run", "--circuit", str(bad)]) == 2
    assert cli.main(["run", "--circuit", str(tmp_path / "missing.json")]) == 2
    assert cli.main(["evolve", "--nqubits", "4", "--solver", "exp"]) == 2
    assert cli.main(["nosuch"]) == 2
