"""Sharded executor on CPU: planner parity with the reference, and the full runner (shard
filters, local diagonals, whole-shard phases, exchanges, relabels, gather) executed with a
CPU stand-in backend -- in-process shards and world_size 2/4 over gloo."""

import json
import math
import os
import socket

import numpy as np
import pytest
import torch

from conftest import golden, max_abs
from cpu_backend import CpuBackend
from oracle import statevec as ov
from plan_helpers import spec_tuples_to_specs
from paper_2009_01845_b200 import CNOT, CZ, H, RY, SWAP, X, Circuit, CZPow, Precision, qft_circuit
from paper_2009_01845_b200 import sharding as sd
from paper_2009_01845_b200.errors import CapacityError, ShapeError


class FakeState:
    def __init__(self, amps, prec=Precision.F64):
        self.tensor = torch.from_numpy(np.array(amps, dtype=prec.complex_dtype))
        self.n_qubits = int(np.log2(len(amps)))
        self.precision = prec


def run_cpu(circuit, n_shards, psi=None, comm=None, global_qubits=None):
    init = FakeState(psi) if psi is not None else None
    sh = sd.run_sharded(circuit, n_shards, init, Precision.F64, global_qubits, comm or sd.LocalComm(),
                        CpuBackend(Precision.F64))
    return sd.gather_tensor(sh).numpy()


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return a / np.linalg.norm(a)


def oracle_of(circuit, psi=None):
    gates = [ov.gate("Unitary", g.targets, g.controls, (), _m(g)) for g in circuit.queue]
    return ov.run(gates, circuit.n_qubits, psi)


def _m(g):
    from paper_2009_01845_b200 import gate_matrix

    return gate_matrix(g)


def random_circuit(n, depth, seed, max_controls=2):
    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(depth):
        kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CZPow", "CNOT", "CZ", "SWAP", "U2", "VL"]
        k = kinds[rng.integers(len(kinds))]
        order = rng.permutation(n)
        two = k in ("CZPow", "CNOT", "CZ", "SWAP", "U2", "VL")
        tg = tuple(int(x) for x in order[: 2 if two else 1])
        ct = tuple(int(x) for x in order[len(tg): len(tg) + int(rng.integers(0, max_controls + 1))])
        th = float(rng.uniform(0, 2 * math.pi))
        if k == "U2":
            q, _ = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
            gates.append(ov.gate("Unitary", tg, ct, (), q))
        elif k == "VL":
            gates.append(ov.gate("VariationalLayer", tg, (), tuple(rng.uniform(0, 6, 4))))
        elif k in ("RX", "RY", "RZ", "CZPow"):
            gates.append(ov.gate(k, tg, ct, (th,)))
        else:
            gates.append(ov.gate(k, tg, ct))
    return Circuit(n).add(spec_tuples_to_specs(gates))


# ------------------------------------------------------------------ planner (reference parity)
def test_plan_matches_reference_for_qft14():
    g = golden("sharding")
    for shards in (2, 4, 8):
        p = sd.plan(qft_circuit(14), shards)
        assert p.n_reshuffles == int(g[f"qft14_reshuffles_{shards}"])
        assert p.global_qubits == tuple(int(x) for x in g[f"qft14_globals_{shards}"])


def test_plan_rules():
    c = Circuit(3).add(H(0))
    for bad in (0, 1, 3, 6):
        with pytest.raises(ShapeError):
            sd.plan(c, bad)
    with pytest.raises(CapacityError):
        sd.plan(c, 8)
    assert sd.plan(Circuit(4).add([X(3, controls=(0,)), H(1), H(2), H(3)]), 2).global_qubits == (0,)
    assert sd.plan(Circuit(3).add([CZ(0, 1), CZPow(1, 2, 0.5), CZ(0, 2)]), 4).n_reshuffles == 0
    p = sd.plan(Circuit(4).add([H(0), H(1), H(2), H(3), H(1)]), 2)
    moves = [s for s in p.steps if isinstance(s, sd.Reshuffle)]
    assert p.global_qubits == (3,) and len(moves) == 1
    assert (moves[0].global_qubit, moves[0].local_qubit) == (3, 2)


def _trotter(n, steps):
    from paper_2009_01845_b200 import build_tfim, build_x, combine
    from paper_2009_01845_b200.evolution import trotter_step_circuit

    c = Circuit(n)
    for k in range(steps):
        s = (k + 0.5) / steps
        c.add(list(trotter_step_circuit(combine(build_x(n), 1 - s, build_tfim(n, 1.0), s), 0.05).queue))
    return c


def _check_batched_plan(c, shards):
    """Replay a batched plan: every gate runs exactly once, after its DAG predecessors, with its
    required qubits local; exchanges pair current globals with current locals."""
    p = sd.plan_batched(c, shards)
    g = shards.bit_length() - 1
    glob, loc = list(p.global_qubits), [q for q in range(c.n_qubits) if q not in p.global_qubits]
    preds = sd._gate_dag(c.queue)
    seen = set()
    for st in p.steps:
        if isinstance(st, sd.Exchange):
            assert 1 <= st.k <= g
            for a, b in st.pairs:
                assert a in glob and b in loc
                glob[glob.index(a)], loc[loc.index(b)] = b, a
            continue
        for pos in st.positions:
            assert pos not in seen and preds[pos] <= seen
            assert not set(sd._required_local_batched(c.queue[pos])) & set(glob)
            spec = c.queue[pos]
            if sd._is_free_swap(spec):
                a, b = spec.targets
                for lst in (glob, loc):
                    for i, x in enumerate(lst):
                        lst[i] = b if x == a else a if x == b else x
            seen.add(pos)
    assert seen == set(range(len(c.queue)))
    return p


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_batched_plan_valid_and_fewer_exchanges(shards):
    """The all-to-all schedule never needs more data-moving steps (or bytes) than the
    reference's one-qubit Belady plan, and at 8 shards a TFIM Trotter step needs one exchange
    where the reference needs 15 ('Communication vs compute')."""
    from paper_2009_01845_b200 import random_grid_circuit, variational_circuit

    rng = np.random.default_rng(5)
    cases = [qft_circuit(12), random_grid_circuit(3, 4, 8, 42), _trotter(12, 2),
             variational_circuit(12, 3, rng.uniform(0, 6, 12 * 7), fused=True), random_circuit(10, 60, 9)]
    for c in cases:
        bat = _check_batched_plan(c, shards)
        ref = sd.plan(c, shards)
        assert bat.n_exchanges <= ref.n_reshuffles
        assert bat.shard_fraction_moved() <= ref.shard_fraction_moved() + 1e-12
    if shards == 8:
        one = _trotter(34, 1)
        assert sd.plan(one, 8).n_reshuffles == 15
        assert _check_batched_plan(one, 8).n_exchanges == 1


# ------------------------------------------------------------------ in-process runner on CPU
@pytest.fixture(params=["batched", "reference"])
def planner(request, monkeypatch):
    monkeypatch.setattr(sd, "SHARD_PLANNER", request.param)
    return request.param


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_local_runner_qft_and_random(shards, planner):
    n = 8
    assert max_abs(run_cpu(qft_circuit(n), shards), oracle_of(qft_circuit(n))) <= 1e-12
    for seed in range(6):
        c = random_circuit(n, 30, seed)
        psi = rand_state(n, 100 + seed)
        assert max_abs(run_cpu(c, shards, psi), oracle_of(c, psi)) <= 1e-12


def test_local_runner_special_cases(planner):
    n = 5
    psi = rand_state(n, 3)
    cases = [
        (Circuit(n).add(SWAP(0, 3)), (0,)),          # one global qubit: half exchange
        (Circuit(n).add(SWAP(0, 1)), (0, 1)),        # both global: relabel
        (Circuit(n).add([CNOT(0, 2), CNOT(0, 3)]), (0,)),   # control stays global
        (Circuit(n).add([X(2, controls=(0, 1)), RY(3, 0.7, controls=(1,))]), (0, 1)),
        (Circuit(n).add([CZ(0, 1), CZPow(0, 1, 1.3, controls=(2,))]), (0, 1)),  # all-global phases
        (Circuit(n).add([H(0), H(1), H(2), H(0), H(1), H(2)]), (0,)),  # forced reshuffles
        (Circuit(n).add([H(0), H(1), H(2), H(3), H(4), H(0), H(1)]), (0, 1, 2)),  # 3-qubit exchanges
        (Circuit(n).add([SWAP(0, 4), H(0), SWAP(1, 3), RY(1, 0.3), SWAP(0, 1), H(4)]), (0, 1)),  # relabels
    ]
    for c, globs in cases:
        shards = 1 << len(globs)
        assert max_abs(run_cpu(c, shards, psi, global_qubits=globs), oracle_of(c, psi)) <= 1e-12


# ------------------------------------------------------------------ distributed (gloo, CPU)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, planner="batched"):
    import torch.distributed as dist

    sd.SHARD_PLANNER = planner
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 8
        results = {}
        comm = sd.TorchComm()
        comm.CHUNK_BYTES = 16 * 7  # force several exchange chunks (odd size on purpose)
        for name, c, psi in [("qft", qft_circuit(n), None),
                             ("rand0", random_circuit(n, 40, 11), rand_state(n, 1)),
                             ("rand1", random_circuit(n, 40, 12, max_controls=3), rand_state(n, 2)),
                             ("swaps", Circuit(n).add([H(0), SWAP(0, 1), SWAP(7, 0), CNOT(1, 6), SWAP(2, 5)]),
                              rand_state(n, 3))]:
            init = FakeState(psi) if psi is not None else None
            sh = sd.run_sharded(c, world, init, Precision.F64, None, comm, CpuBackend(Precision.F64))
            got = sd.gather_tensor(sh).numpy()
            results[name] = float(np.max(np.abs(got - oracle_of(c, psi))))
        # a state resident in the ranks' shards across several circuits (apply_sharded: each
        # planned from the current global qubits), then brought to the canonical layout
        c1, c2, c3 = random_circuit(n, 25, 21), qft_circuit(n), random_circuit(n, 25, 22)
        psi = rand_state(n, 4)
        sh = sd.run_sharded(c1, world, FakeState(psi), Precision.F64, None, comm, CpuBackend(Precision.F64))
        sd.apply_sharded(sh, c2)
        sd.apply_sharded(sh, c3)
        want = oracle_of(c3, oracle_of(c2, oracle_of(c1, psi)))
        results["resident"] = float(np.max(np.abs(sd.gather_tensor(sh).numpy() - want)))
        sd.canonicalize(sh)
        assert set(sh.global_qubits) == set(range(world.bit_length() - 1))
        assert list(sh.local_qubits) == sorted(sh.local_qubits)
        results["canonical"] = float(np.max(np.abs(sd.gather_tensor(sh).numpy() - want)))
        with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
            json.dump(results, f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,planner", [(2, "batched"), (4, "batched"), (4, "reference")])
def test_distributed_gloo(world, planner, tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), planner), nprocs=world, join=True)
    for r in range(world):
        res = json.load(open(tmp_path / f"r{r}.json"))
        for name, err in res.items():
            assert err <= 1e-12, (world, r, name, err)


def test_bench_distributed_summary():
    """bench.py's sharded-step roofline/launch accounting: sweeps from the runner's plan cache,
    exchange time subtracted, pack+unpack per chunk per reshuffle."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2009_01845_b200 import _native as nat
    from paper_2009_01845_b200 import qft_circuit
    from paper_2009_01845_b200.fusion import plan_circuit

    p = plan_circuit(qft_circuit(14).queue, 14, nat.QSB_C128)
    shard = (1 << 14) * 16
    roof, launches = bench._dist_summary({"k": p, "other": object()}, 2, 1e-3, 1e-4, shard, 16, 1 << 16)
    assert roof["sweeps_per_step"] == p.state_sweeps()
    assert abs(roof["achieved"] - p.state_sweeps() * 2 * shard / 8e-4 / 1e9) < 1e-9
    assert launches == len(p.steps) + 2 * 2 * ((shard // 32) // 4096) + 1
    # 3-qubit exchanges: 7 peers, each part 2^11 amplitudes in chunks of (2^16 / 16) // 7 = 585
    roof, launches = bench._dist_summary({"k": p}, 1, 1e-3, 1e-4, shard, 16, 1 << 16, 3)
    assert launches == len(p.steps) + 2 * 7 * -(-(1 << 11) // 585) + 1
