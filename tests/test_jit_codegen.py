"""CPU check of the pass specialiser: generated sources compile for sm_100a with nvcc, and
structurally identical passes (same bits, different angles) share one kernel source."""

import shutil
import subprocess

import numpy as np
import pytest

from oracle import statevec as ov
from plan_helpers import spec_tuples_to_specs
from paper_2009_01845_b200 import _native as nat, jit, qft_circuit, variational_circuit
from paper_2009_01845_b200.fusion import PassStep, plan_circuit


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
