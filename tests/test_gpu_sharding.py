"""GPU parity of the sharded executor with in-process shards (the single-GPU placement of the
distributed runner): against the oracle and against the unsharded engine."""

import math

import numpy as np
import pytest

from conftest import golden, max_abs
from oracle import statevec as ov

pytestmark = pytest.mark.gpu


def _sv(a):
    import paper_2009_01845_b200 as q

    return q.from_amplitudes(np.asarray(a))


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_sharded_random_circuits_golden(cuda, shards, mode):
    from conftest import circuit_from_json
    import paper_2009_01845_b200 as q

    g = golden("random_circuits")
    for i, text in enumerate(g["circuits"]):
        c = circuit_from_json(text)
        got = q.execute_sharded(c, shards, initial=_sv(g[f"in{i}"])).amplitudes
        assert max_abs(got, g[f"out{i}"]) <= 1e-12


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_sharded_qft_variational(cuda, shards, mode):
    import paper_2009_01845_b200 as q

    gq = golden("qft")
    assert max_abs(q.execute_sharded(q.qft_circuit(14), shards).amplitudes, gq["zero14"]) <= 1e-12
    assert max_abs(q.execute_sharded(q.qft_circuit(14), shards, initial=_sv(gq["rin14"])).amplitudes,
                   gq["rout14"]) <= 1e-12
    gv = golden("variational")
    c = q.variational_circuit(14, 3, gv["params14"], fused=True)
    assert max_abs(q.execute_sharded(c, shards).amplitudes, gv["f64_14_1"]) <= 1e-12


def test_sharded_equals_unsharded_large(cuda, mode):
    import paper_2009_01845_b200 as q

    n = 22
    rng = np.random.default_rng(8)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    c = q.qft_circuit(n)
    a = c.execute(_sv(psi)).amplitudes
    for shards in (2, 8):
        b = q.execute_sharded(c, shards, initial=_sv(psi)).amplitudes
        assert max_abs(a, b) <= 1e-12


def test_sharded_trotter_step(cuda, mode):
    import paper_2009_01845_b200 as q

    g = golden("adiabatic")
    dt, T = g["cfg14"]
    st = q.adiabatic_evolve(q.build_x(14), q.build_tfim(14, 1.0), q.Schedule.linear(),
                            q.EvolutionConfig(q.Solver.TROTTER, float(dt), float(T)), n_shards=4)
    assert max_abs(st.amplitudes, g["n14"]) <= 1e-12


def test_sharded_preserves_initial(cuda):
    import paper_2009_01845_b200 as q

    init = _sv(np.random.default_rng(1).standard_normal(16) + 0j)
    keep = init.amplitudes
    q.execute_sharded(q.qft_circuit(4), 2, initial=init)
    assert np.array_equal(init.amplitudes, keep)


@pytest.mark.parametrize("n,shards,glob", [(12, 2, None), (14, 4, None), (13, 8, (5, 0, 11)), (16, 4, (3, 9))])
def test_sharded_sampling_bitwise(cuda, n, shards, glob):
    """sample_sharded (chained exact cumsum, per-shard unclipped counts) draws the same samples
    as sampling the gathered state, including non-canonical global qubit sets."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import sharding as sd

    rng = np.random.default_rng(n * shards)
    c = q.random_grid_circuit(2, n // 2, 4, int(rng.integers(1000))) if n % 2 == 0 else q.qft_circuit(n)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    sh = sd.run_sharded(c, shards, _sv(psi), global_qubits=glob)
    full = sd.gather(sh)
    for seed, shots in ((3, 5000), (11, 20000)):
        want = q.sample(full, range(n), shots, seed).samples
        got = sd.sample_sharded(sh, shots, seed)
        assert np.array_equal(got.samples, want)
        assert got.qubits == tuple(range(n))
    # still the same state after canonicalisation
    assert max_abs(sd.gather(sh).amplitudes, full.amplitudes) == 0


def test_chained_cumsum_equals_serial(cuda):
    """The exact cumsum chained over pieces (previous last value prepended) equals one sequential
    cumsum over the whole vector, bit for bit (including a heavy-tailed distribution)."""
    import torch

    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import _native as nat
    from paper_2009_01845_b200.measurement import device_cdf

    rng = np.random.default_rng(4)
    n = 1 << 18
    for p in (rng.random(n) / n, np.exp(rng.standard_normal(n) * 6) / n):
        pt = torch.from_numpy(p).cuda()
        serial = torch.empty_like(pt)
        nat.check(nat.lib().qsb_cumsum_serial(pt.data_ptr(), n, serial.data_ptr(), nat.stream_ptr()))
        pieces, carry = [], None
        for chunk in torch.chunk(pt, 8):
            if carry is None:
                cum = device_cdf(chunk.contiguous(), normalize=False)
            else:
                cum = device_cdf(torch.cat([carry, chunk]), normalize=False)[1:]
            carry = cum[-1:].clone()
            pieces.append(cum)
        assert torch.equal(torch.cat(pieces), serial)
        assert np.array_equal(torch.cat(pieces).cpu().numpy(), np.cumsum(p))


@pytest.mark.parametrize("n,shards", [(10, 2), (12, 4), (13, 8)])
def test_resident_sharded_adiabatic_evolution(cuda, n, shards):
    """adiabatic_evolve_sharded keeps the state in shards for all steps (no gather per step): the
    gathered result, its energy (expectation_sharded, no gather) and its samples match the
    1-GPU evolution."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import sharding as sd

    h0, h1 = q.build_x(n), q.build_tfim(n, 1.0)
    cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.1, 1.0)
    want = q.adiabatic_evolve(h0, h1, q.Schedule.linear(), cfg)
    sh = q.adiabatic_evolve_sharded(h0, h1, q.Schedule.linear(), cfg, n_shards=shards)
    e = sd.expectation_sharded(h1, sh)
    assert abs(e - q.expectation(h1, want)) <= 1e-10
    assert abs(sd.expectation_sharded(h0, sh) - q.expectation(h0, want)) <= 1e-10
    got = sd.gather(sh)
    assert max_abs(got.amplitudes, want.amplitudes) <= 1e-12
    # evolving a given state (partitioned once) and a resident ShardedState in place
    init = q.from_amplitudes(want.amplitudes)
    a = sd.gather(q.evolve_sharded(h1, cfg, n_shards=shards, initial=init)).amplitudes
    b = q.evolve(h1, init, cfg).amplitudes
    assert max_abs(a, b) <= 1e-12


def test_cli_evolve_sharded_energy(cuda, capsys):
    import json

    from paper_2009_01845_b200 import cli

    assert cli.main(["evolve", "--nqubits", "10", "--dt", "0.1", "--T", "1.0"]) == 0
    one = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert cli.main(["evolve", "--nqubits", "10", "--dt", "0.1", "--T", "1.0", "--shards", "4"]) == 0
    four = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert abs(one["final_energy"] - four["final_energy"]) <= 1e-10


@pytest.mark.parametrize("window", [1, 3, None])
def test_resident_evolution_callbacks_and_windows(cuda, window):
    """Callbacks during a resident sharded evolution (evaluated at t = 0 and after every step
    without a gather, as evolution.py:339-347 does on the full state) and windows of several
    Trotter steps scheduled together: the state, the energies and the overlaps equal the 1-GPU
    evolution's."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import sharding as sd

    n, shards = 12, 8
    h0, h1 = q.build_x(n), q.build_tfim(n, 1.0)
    cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.1, 0.75)  # 7 full steps + a remainder step
    target = q.uniform_state(n)
    cb1 = [q.EnergyCallback(h1), q.OverlapCallback(target)]
    want = q.adiabatic_evolve(h0, h1, q.Schedule.linear(), cfg, callbacks=cb1)
    if window == 1:
        cb2 = [q.EnergyCallback(h1), q.OverlapCallback(target)]
        sh = q.adiabatic_evolve_sharded(h0, h1, q.Schedule.linear(), cfg, n_shards=shards, callbacks=cb2)
        for a, b in zip(cb1, cb2):
            assert len(a.records) == len(b.records) == 9
            assert np.max(np.abs(np.array(a.records) - np.array(b.records))) <= 1e-10
    else:
        sh = q.adiabatic_evolve_sharded(h0, h1, q.Schedule.linear(), cfg, n_shards=shards, window=window)
    assert abs(sd.norm_sharded(sh) - 1.0) <= 1e-12
    assert abs(sd.overlap_sharded(target, sh) - q.overlap(target, want)) <= 1e-12
    assert max_abs(sd.gather(sh).amplitudes, want.amplitudes) <= 1e-12


def test_sharded_equals_one_gpu_at_config4_size(cuda):
    """SURVEY.md section 8(e) at BASELINE config 4's size: the 33-qubit random grid circuit
    sharded over 8 shards (batched all-to-all schedule) against the whole 137 GB state on one
    B200, compared through per-chunk fingerprints and 2^20 sampled amplitudes
    (tools/sharded33_check.py; each state is freed before the other is built)."""
    import os
    import subprocess
    import sys

    cuda.cuda.synchronize()
    cuda.cuda.empty_cache()
    free, _ = cuda.cuda.mem_get_info()
    if free < (165 << 30):
        pytest.skip(f"needs ~160 GB of free device memory, {free / 2**30:.0f} GiB free")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sharded33_check.py"), "33", "8", "20"],
                       capture_output=True, text=True, timeout=900, cwd=root)
    assert "CHECK_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_sharded_bit_identical_with_per_gate_kernels(cuda, shards, monkeypatch):
    """SURVEY.md section 8(e)'s invariant, bit for bit, in the reference's own terms: every gate
    its own kernel (QSB_FUSION=0) and the reference's in-order reshuffle schedule
    (QSB_SHARD_PLANNER=reference) -- partition, per-shard gates, global-qubit gates as per-shard
    phases, pairwise exchanges, gather -- give exactly the 1-GPU result.  The default batched
    schedule moves commuting gates across each other (exact in real arithmetic, a different
    summation order in floating point) and fused passes group and merge gates differently, so
    those agree to rounding (<= 1e-12), as the other tests check."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import engine
    from paper_2009_01845_b200 import sharding as sd

    monkeypatch.setattr(engine, "FUSION_DEFAULT", False)
    monkeypatch.setattr(sd, "SHARD_PLANNER", "reference")
    n = 20
    rng = np.random.default_rng(31)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    circuits = [q.qft_circuit(n), q.variational_circuit(n, 2, rng.uniform(0, 6, n * 5), fused=True),
                q.random_grid_circuit(4, 5, 6, 3)]
    for c in circuits:
        a = c.execute(_sv(psi)).amplitudes
        b = q.execute_sharded(c, shards, initial=_sv(psi)).amplitudes
        assert np.array_equal(a, b), (c, shards, float(np.max(np.abs(a - b))))
