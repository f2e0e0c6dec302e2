"""CPU check of the pass specialiser: generated sources compile for sm_100a with nvcc, and
structurally identical passes (same bits, different angles) share one kernel source."""

import shutil
import subprocess

import numpy as np
import pytest

from oracle import statevec as ov
from plan_helpers import spec_tuples_to_specs
from paper_2009_01845_b200 import _native as nat, jit, qft_circuit, variational_circuit
from paper_2009_01845_b200.fusion import GEOMETRY_JIT, PassStep, plan_circuit


def _compile(src, tmp_path):
    f = tmp_path / "k.cu"
    f.write_text(src)
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-c", str(f),
                        "-o", str(tmp_path / "k.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
@pytest.mark.parametrize("dtype", [nat.QSB_C128, nat.QSB_C64])
def test_generated_sources_compile(tmp_path, dtype):
    n = 16
    rng = np.random.default_rng(3)
    circuits = [qft_circuit(n).queue,
                variational_circuit(n, 2, rng.uniform(0, 6, n * 5), fused=True).queue,
                spec_tuples_to_specs(ov.trotter_step(ov.combine(ov.x_terms(n), 0.3, ov.tfim_terms(n, 1.0), 0.7), 0.1))]
    seen = 0
    for queue in circuits:
        plan = plan_circuit(queue, n, dtype)
        for s in plan.steps:
            if isinstance(s, PassStep) and seen < 3:
                src, name, cf = jit.generate(s.words, dtype)
                assert name in src and np.all(np.isfinite(cf))
                _compile(src, tmp_path)
                seen += 1
    assert seen == 3


def test_structure_sharing_across_angles():
    n = 18
    terms1 = ov.combine(ov.x_terms(n), 0.3, ov.tfim_terms(n, 1.0), 0.7)
    terms2 = ov.combine(ov.x_terms(n), 0.6, ov.tfim_terms(n, 1.0), 0.4)
    p1 = plan_circuit(spec_tuples_to_specs(ov.trotter_step(terms1, 0.05)), n, nat.QSB_C128)
    p2 = plan_circuit(spec_tuples_to_specs(ov.trotter_step(terms2, 0.05)), n, nat.QSB_C128)
    for a, b in zip(p1.steps, p2.steps):
        sa, _, ca = jit.generate(a.words, nat.QSB_C128)
        sb, _, cb = jit.generate(b.words, nat.QSB_C128)
        assert sa == sb and not np.array_equal(ca, cb)


def test_parity_sign_word_equals_quadratic_form():
    """The jit's per-thread sign word for -1-phase diagonal batches (jit.parity_sign_plan) gives
    every slot the sign Q(x | goff[s]) of the direct per-amplitude quadratic form."""
    rng = np.random.default_rng(11)
    for trial in range(200):
        n = int(rng.integers(8, 34))
        nreg = int(rng.integers(2, 6))
        pos = rng.permutation(n)
        regs = sorted(int(p) for p in pos[:nreg])
        rest = [int(p) for p in pos[nreg:]]
        goff = [sum(1 << regs[i] for i in range(nreg) if (sl >> i) & 1) for sl in range(1 << nreg)]
        s1 = int(sum(1 << int(b) for b in rng.choice(n, size=int(rng.integers(0, 4)), replace=False)))
        pairs = []
        for d in sorted(set(int(x) for x in rng.integers(1, n, size=int(rng.integers(0, 4))))):
            m = int(sum(1 << int(b) for b in range(n - d) if rng.random() < 0.3))
            if m:
                pairs.append((d, m))
        C, cross = jit.parity_sign_plan(s1, pairs, goff, nreg)
        for _ in range(8):
            x = sum(1 << p for p in rest if rng.random() < 0.5)
            W = C ^ (((1 << (1 << nreg)) - 1) if jit.parity_quadratic(x, s1, pairs) else 0)
            for K, M in cross:
                if bin(x & K).count("1") & 1:
                    W ^= M
            for sl in range(1 << nreg):
                assert (W >> sl) & 1 == jit.parity_quadratic(x | goff[sl], s1, pairs), (trial, sl)


def test_structure_key_determines_source():
    """jit.coefficients_only: programs with equal structure keys generate identical kernel
    sources, and the coefficient-only pass yields exactly the full generator's coefficients --
    so compile_words may reuse a compiled kernel by key (time-dependent Trotter steps)."""
    from paper_2009_01845_b200 import build_tfim, build_x, combine, random_grid_circuit, trotter_step_circuit

    n = 18
    seen = {}
    progs = []
    for s in (0.2, 0.5, 0.9):
        h = combine(build_x(n), 1 - s, build_tfim(n, 1.0), s)
        progs.append(trotter_step_circuit(h, 0.05).queue)
    rng = np.random.default_rng(4)
    for seed in (1, 2):
        progs.append(random_grid_circuit(3, 6, 4, seed).queue)
        progs.append(variational_circuit(n, 2, rng.uniform(0, 6, n * 5), fused=True).queue)
    progs.append(qft_circuit(n).queue)
    for dtype in (nat.QSB_C128, nat.QSB_C64):
        for queue in progs:
            plan = plan_circuit(queue, n, dtype, geometry=GEOMETRY_JIT[dtype])
            for st in plan.steps:
                if not isinstance(st, PassStep):
                    continue
                src, _name, cf, tab, _tp, key = jit._generate(st.words, dtype)
                k2, cf2, tab2 = jit.coefficients_only(st.words, dtype)
                assert k2 == key and np.array_equal(cf, cf2) and np.array_equal(tab, tab2)
                if key in seen:
                    assert seen[key] == src
                seen[key] = src
    # the Trotter steps at different field ratios share their kernels
    assert len(seen) < sum(1 for q_ in progs for _ in q_)


def test_coefficient_recipes_equal_the_generator(monkeypatch):
    """jit coefficient recipes: after one program of a structure has been recorded, another
    program of that structure (new coefficients) gets exactly the coefficient-only generator's
    structure key, parameters and tables by plain word reads -- for dense-gate passes
    (Trotter, grid, variational) and diagonal / pivot passes (QFT, random phases)."""
    from paper_2009_01845_b200 import build_tfim, build_x, combine, random_grid_circuit, trotter_step_circuit
    from paper_2009_01845_b200 import gates as G

    monkeypatch.setattr(jit, "_RECIPES", {})
    monkeypatch.setattr(jit, "RECIPES", True)
    n = 18
    rng = np.random.default_rng(9)

    def phases(seed):
        r = np.random.default_rng(seed)
        out = []
        for q in range(n - 1):
            out.append(G.GateSpec(G.GateKind.H, (q,), (), ()))
            out.append(G.GateSpec(G.GateKind.CZPOW, (q, q + 1), (), (float(r.uniform(0.1, 0.9)),)))
            out.append(G.GateSpec(G.GateKind.RZ, (q,), (), (float(r.uniform(0.1, 3)),)))
        return out

    families = [
        [combine(build_x(n), 1 - s, build_tfim(n, 1.0), s) for s in (0.2, 0.3, 0.7)],
        [3, 4],
        [rng.uniform(0, 6, n * 5) for _ in range(2)],
        [5, 6],
    ]
    checked = 0
    for dtype in (nat.QSB_C128, nat.QSB_C64):
        for fam, members in enumerate(families):
            first = True
            for mbr in members:
                if fam == 0:
                    queue = trotter_step_circuit(mbr, 0.05).queue
                elif fam == 1:
                    queue = random_grid_circuit(3, 6, 4, mbr).queue
                elif fam == 2:
                    queue = variational_circuit(n, 2, mbr, fused=True).queue
                else:
                    queue = phases(mbr)
                plan = plan_circuit(queue, n, dtype, geometry=GEOMETRY_JIT[dtype])
                for st in plan.steps:
                    if not isinstance(st, PassStep):
                        continue
                    ref = jit.coefficients_only(st.words, dtype)
                    if first:
                        jit._recipe_build(st.words, dtype)
                        continue
                    w = np.asarray(st.words, dtype=np.int64)
                    r = jit._recipe_lookup(w, dtype)
                    if r is None:
                        continue  # another structure (e.g. a grid cycle with other gates)
                    key, p, t = jit.fast_coefficients(st.words, dtype)
                    assert key == ref[0] and np.array_equal(p, ref[1]) and np.array_equal(t, ref[2])
                    checked += 1
                first = False
    assert checked >= 10
    assert jit.RECIPE_STATS["refused"] == 0 or jit.RECIPE_STATS["built"] > 0
