"""Pin the CPU oracle (oracle/statevec.py) against vectors produced by the real reference
(tests/golden, made by oracle/gen_golden.py).  CPU only."""

import hashlib
import json

import numpy as np
import pytest

from conftest import golden, max_abs
from oracle import statevec as ov


def test_single_gates_match_reference_bitwise_or_tight():
    g = golden("single_gates")
    for text, inp, out in zip(g["circuits"], g["inputs"], g["outputs"]):
        n, gates = ov.from_json(text)
        got = ov.run(gates, n, inp)
        assert max_abs(got, out) <= 1e-15


def test_random_circuits():
    g = golden("random_circuits")
    for i, (n, text) in enumerate(zip(g["n"], g["circuits"])):
        _, gates = ov.from_json(text)
        assert max_abs(ov.run(gates, int(n), g[f"in{i}"]), g[f"out{i}"]) <= 1e-14


@pytest.mark.parametrize("n", [10, 14])
def test_qft(n):
    g = golden("qft")
    gates = ov.qft(n)
    assert max_abs(ov.run(gates, n), g[f"zero{n}"]) <= 1e-15
    assert max_abs(ov.run(gates, n, g[f"rin{n}"]), g[f"rout{n}"]) <= 1e-15
    k = int(g[f"basisk{n}"])
    basis = np.zeros(1 << n, dtype=complex)
    basis[k] = 1
    got = ov.run(gates, n, basis)
    assert max_abs(got, g[f"basis{n}"]) <= 1e-15
    j = np.arange(1 << n)
    dft = np.exp(2j * np.pi * j * k / (1 << n)) / np.sqrt(1 << n)
    assert max_abs(got, dft) <= 1e-10
    assert max_abs(ov.run(gates, n, dtype=np.complex64), g[f"f32_{n}"]) <= 1e-7


@pytest.mark.parametrize("n", [10, 14])
@pytest.mark.parametrize("fused", [False, True])
def test_variational(n, fused):
    g = golden("variational")
    gates = ov.variational(n, 3, g[f"params{n}"], fused=fused)
    assert max_abs(ov.run(gates, n), g[f"f64_{n}_{int(fused)}"]) <= 1e-15
    assert max_abs(ov.run(gates, n, dtype=np.complex64), g[f"f32_{n}_{int(fused)}"]) <= 1e-7


def test_c64_large_fixtures():
    """complex64 at n = 16 (the fixtures the GPU tests run through planned fused passes)."""
    g = golden("c64_large")
    n = 16
    assert max_abs(ov.run(ov.qft(n), n, g["qft_in"], dtype=np.complex64), g["qft_out"]) <= 1e-7
    for fused in (False, True):
        gates = ov.variational(n, 3, g["var_params"], fused=fused)
        assert max_abs(ov.run(gates, n, dtype=np.complex64), g[f"var_{int(fused)}"]) <= 1e-7
    _, gates = ov.from_json(g["grid_circuit"])
    assert max_abs(ov.run(gates, n, dtype=np.complex64), g["grid_out"]) <= 1e-7


def test_grid_supremacy_builder_matches_reference_execution():
    g = golden("grid15")
    gates = ov.grid_supremacy(3, 5, 8, seed=42)
    n, parsed = ov.from_json(g["circuit"])
    assert n == 15 and len(parsed) == len(gates)
    for a, b in zip(gates, parsed):
        assert a[1] == b[1] and np.array_equal(a[4], b[4])
    assert max_abs(ov.run(gates, 15), g["out"]) <= 1e-15


def test_adiabatic():
    g = golden("adiabatic")
    for n in (8, 13, 14):
        dt, T = g[f"cfg{n}"]
        assert max_abs(ov.adiabatic(n, 1.0, float(dt), float(T)), g[f"n{n}"]) <= 1e-15


def test_sampling_bitwise():
    g = golden("sampling")
    state = g["state"]
    for i, text in enumerate(g["subsets"]):
        qs = tuple(json.loads(str(text)))
        assert np.array_equal(ov.marginal(state, 12, qs), g[f"marg{i}"])
        assert np.array_equal(ov.sample(state, 12, qs, 2000, 100 + i), g[f"samp{i}"])
    f32 = state.astype(np.complex64)
    assert np.array_equal(ov.marginal(f32, 12, (0, 3, 5)), g["marg_f32"])
    assert np.array_equal(ov.sample(f32, 12, (0, 3, 5), 1000, 9), g["samp_f32"])


@pytest.mark.parametrize("nq,shots,seed", [(3, 500, 7), (20, 100000, 42)])
def test_cli_shots_digest(nq, shots, seed):
    g = golden("sampling")
    amps = ov.run([ov.gate("H", (q,)) for q in range(nq)], nq)
    s = ov.sample(amps, nq, tuple(range(nq)), shots, seed)
    assert hashlib.sha256(s.tobytes()).hexdigest() == str(g[f"digest_{nq}_{shots}_{seed}"])
