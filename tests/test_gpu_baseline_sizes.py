"""GPU parity at BASELINE sizes (n = 30; BASELINE.json configs 2 and 3) and for the complex64
fused passes.

The kernels bench.py times run here on the states bench.py times them on, against checkers that
work at any size:
* QFT-30 on a basis state |k> against the analytic DFT column (the reference's own check,
  /root/reference/pkg/tests/test_circuit.py:189-201), compared on the device in chunks;
* variational-30 (fused layers), the random grid 3x10 and a Trotter TFIM step at n = 30: the
  fused-pass plan against the per-gate kernels (fuse=False), which the reference's single-gate
  goldens pin bit-for-bit / to 1e-15 (tests/test_gpu_parity.py);
* complex64 at n = 16 (512 KB, above the shared-memory batch limit) against fixtures made by
  the reference itself (tests/golden/c64_large.npz), through the planned fused passes.
Tolerances: 1e-12 per amplitude (complex128), 1e-5 (complex64) -- BASELINE north star."""

import math

import numpy as np
import pytest

from conftest import circuit_from_json, golden, max_abs

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


def _device_max_abs_diff(a, b):
    from paper_2009_01845_b200.verify import max_abs_diff

    return max_abs_diff(a, b)


def dft_column_error(state, k):
    from paper_2009_01845_b200.verify import dft_column_error as err

    return err(state, k)


def _free(*objs):
    import torch

    del objs
    torch.cuda.empty_cache()


@pytest.mark.parametrize("prec,tol", [("f64", TOL64), ("f32", TOL32)])
def test_qft30_basis_state_matches_dft_column(cuda, prec, tol):
    import paper_2009_01845_b200 as q

    n = 30
    precision = q.Precision(prec)
    k = int(np.random.default_rng(30).integers(1 << n))
    c = q.qft_circuit(n)
    plan = c.plan(precision)
    assert plan.n_passes == 4  # the bench's plan: four fused HBM passes, SWAPs folded
    out = c.execute(q.basis_state(n, k, precision), precision=precision)
    err = dft_column_error(out, k)
    assert err <= tol, f"QFT-30 {prec} max |psi - DFT column| = {err:.3e}"
    _free(out)


def _fused_vs_per_gate(circuit, n, precision, tol, initial=None):
    import paper_2009_01845_b200 as q

    start = initial if initial is not None else q.zero_state(n, precision)
    fused = circuit.execute(start, precision=precision)
    plan = circuit.plan(precision)
    assert plan.n_passes >= 1
    ref = circuit.execute(start, precision=precision, fuse=False)
    err = _device_max_abs_diff(fused.tensor, ref.tensor)
    _free(fused, ref)
    assert err <= tol, f"fused vs per-gate max |diff| = {err:.3e}"
    return err


@pytest.mark.parametrize("prec,tol", [("f64", TOL64), ("f32", TOL32)])
def test_variational30_fused_passes_equal_per_gate_kernels(cuda, prec, tol):
    import paper_2009_01845_b200 as q

    n = 30
    params = np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11)
    c = q.variational_circuit(n, 5, params, fused=True)
    _fused_vs_per_gate(c, n, q.Precision(prec), tol)


def test_grid30_fused_passes_equal_per_gate_kernels(cuda):
    import paper_2009_01845_b200 as q

    c = q.random_grid_circuit(3, 10, 20, 42)
    _fused_vs_per_gate(c, 30, q.Precision.F64, TOL64)


def test_trotter_step30_fused_passes_equal_per_gate_kernels(cuda):
    import paper_2009_01845_b200 as q

    n = 30
    h = q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5)
    c = q.trotter_step_circuit(h, 0.05)
    _fused_vs_per_gate(c, n, q.Precision.F64, TOL64, initial=q.uniform_state(n))


@pytest.mark.parametrize("n", [24, 26])
def test_norm_and_overlap_against_numpy_large(cuda, n):
    """state.py:109-122 norm / overlap as device reductions, against numpy on the host copy."""
    import paper_2009_01845_b200 as q

    rng = np.random.default_rng(n)
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    b = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    sa, sb = q.from_amplitudes(a), q.from_amplitudes(b)
    assert abs(q.norm(sa) - np.linalg.norm(a)) <= 1e-12 * np.linalg.norm(a)
    want = np.vdot(a, b)
    assert abs(q.overlap(sa, sb) - want) <= 1e-12 * abs(want) + 1e-9
    a32, b32 = a.astype(np.complex64), b.astype(np.complex64)
    s32a, s32b = q.from_amplitudes(a32), q.from_amplitudes(b32)
    assert abs(q.norm(s32a) - np.linalg.norm(a32.astype(np.complex128))) <= 1e-9 * np.linalg.norm(a)
    want32 = np.vdot(a32.astype(np.complex128), b32.astype(np.complex128))
    assert abs(q.overlap(s32a, s32b) - want32) <= 1e-9 * abs(want32) + 1e-6


# ---------------------------------------------------------------- complex64 fused passes
def test_c64_large_fixtures_through_planned_passes(cuda, mode):
    """complex64 at n = 16 against the reference (c64_large.npz): in `planned` mode every circuit
    runs as fused passes with the packed FP32-pair gate code; in `batched` mode the first run is
    the grid-synchronised batch and the second run of the same circuit is planned."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200.fusion import PassStep

    g = golden("c64_large")
    n = 16
    f32 = q.Precision.F32
    cases = [(q.qft_circuit(n), q.from_amplitudes(g["qft_in"]), g["qft_out"])]
    for fused in (False, True):
        cases.append((q.variational_circuit(n, 3, g["var_params"], fused=fused), None, g[f"var_{int(fused)}"]))
    cases.append((circuit_from_json(g["grid_circuit"]), None, g["grid_out"]))
    for c, init, want in cases:
        for _ in range(2):  # second run: planned in both modes
            got = c.execute(init, precision=f32).amplitudes
            assert got.dtype == np.complex64
            assert max_abs(got, want) <= TOL32
        plan = c.plan(f32)
        assert any(isinstance(s, PassStep) for s in plan.steps)


def test_evolve_step_windows_equal_single_steps(cuda, monkeypatch):
    """evolve() without callbacks runs consecutive Trotter steps as one circuit
    (evolution.STEP_WINDOW); planned fused passes then cross the step boundaries.  The result
    equals stepping one circuit at a time (the reference's loop, evolution.py:339-347) to 1e-12,
    for a time-independent H and for the time-dependent adiabatic schedule (with its remainder
    step)."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import engine, evolution

    monkeypatch.setattr(engine, "FIRST_RUN_BATCH", False)
    n = 22
    h = q.combine(q.build_x(n), 0.4, q.build_tfim(n, 1.0), 0.6)
    cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.05, 0.33)  # 6 full steps + a remainder
    psi0 = q.uniform_state(n)
    outs = {}
    for w in (1, 4):
        monkeypatch.setattr(evolution, "STEP_WINDOW", w)
        outs[w] = (q.evolve(h, psi0, cfg).tensor,
                   q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 1.0), q.Schedule.linear(), cfg).tensor)
    assert _device_max_abs_diff(outs[1][0], outs[4][0]) <= TOL64
    assert _device_max_abs_diff(outs[1][1], outs[4][1]) <= TOL64


@pytest.mark.parametrize("prec,tol", [("f64", TOL64), ("f32", TOL32)])
def test_template_and_recipe_plans_equal_per_gate_kernels(cuda, prec, tol, monkeypatch):
    """Circuits of one structure with fresh angles (phase-heavy: H, CZPow, RZ, controlled RX, so
    the passes hold pivots and diagonal terms, re-encoded from the template; and dense layers,
    whose matrix words are patched) run on plans from the template with kernels reused through
    coefficient recipes -- and still equal the per-gate kernels at n = 24."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import engine, fusion, jit

    monkeypatch.setattr(engine, "FIRST_RUN_BATCH", False)  # planned passes from the first run
    n = 24
    precision = q.Precision(prec)

    def build(seed):
        r = np.random.default_rng(seed)
        c = q.Circuit(n)
        for layer in range(3):
            for k in range(n):
                c.add(q.H(k))
                c.add(q.RZ(k, float(r.uniform(0.1, 3))))
            for k in range(n - 1):
                c.add(q.CZPow(k, k + 1, float(r.uniform(0.1, 0.9))))
            for k in range(0, n - 2, 3):
                c.add(q.RX(k + 2, float(r.uniform(0.1, 3)), controls=(k,)))
        return c

    hits0, rec0 = fusion.TEMPLATE_STATS["hits"], jit.RECIPE_STATS["hits"]
    start = q.uniform_state(n, precision)
    for seed in (1, 2, 3):
        _fused_vs_per_gate(build(seed), n, precision, tol, initial=start)
    assert fusion.TEMPLATE_STATS["hits"] >= hits0 + 2
    assert jit.RECIPE_STATS["hits"] > rec0
