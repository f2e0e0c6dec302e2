"""Batched global<->local exchange on the GPU: the k-qubit part kernels against the index math
of the CPU stand-in, the in-process all-to-all against execute(), and the stream-ordered
(NCCL-semantics) exchange pipeline with ranks as threads on one GPU (tests/thread_comm.py)."""

import math

import numpy as np
import pytest

from conftest import max_abs
from cpu_backend import CpuBackend

pytestmark = pytest.mark.gpu


def _rand(n, seed, torch, dtype):
    rng = np.random.default_rng(seed)
    a = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(dtype)
    return torch.from_numpy(a)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_part_kernels_match_index_math(cuda, prec):
    torch = cuda
    from paper_2009_01845_b200 import Precision
    from paper_2009_01845_b200.sharding import CudaBackend, _part_bits

    p = Precision(prec)
    dev, cpu = CudaBackend(p), CpuBackend(p)
    nl = 12
    for bits in ([11], [0], [3, 7], [10, 2, 6], [0, 1, 2]):
        k = len(bits)
        for v in range(1 << k):
            pb = _part_bits(v, bits)
            src = _rand(nl, 10 + v, torch, p.complex_dtype)
            count, first = (1 << (nl - k)) - 5, 3
            st_d, st_c = dev.empty(1 << (nl - k)), cpu.empty(1 << (nl - k))
            dev.pack_part(src.cuda(), nl, bits, pb, first, count, st_d)
            cpu.pack_part(src, nl, bits, pb, first, count, st_c)
            assert torch.equal(st_d[:count].cpu(), st_c[:count])
            a_d, a_c = src.cuda(), src.clone()
            new = _rand(nl - k, 99, torch, p.complex_dtype)
            dev.unpack_part(a_d, nl, bits, pb, first, count, new.cuda())
            cpu.unpack_part(a_c, nl, bits, pb, first, count, new)
            assert torch.equal(a_d.cpu(), a_c)
            b = _rand(nl, 50 + v, torch, p.complex_dtype)
            a_d, b_d, a_c, b_c = src.cuda(), b.cuda(), src.clone(), b.clone()
            other = _part_bits((v + 1) % (1 << k), bits)
            dev.exchange_parts(a_d, b_d, nl, bits, pb, other)
            cpu.exchange_parts(a_c, b_c, nl, bits, pb, other)
            assert torch.equal(a_d.cpu(), a_c) and torch.equal(b_d.cpu(), b_c)


def test_part_kernels_reject_bad_args(cuda):
    torch = cuda
    from paper_2009_01845_b200 import Precision
    from paper_2009_01845_b200.errors import ShapeError
    from paper_2009_01845_b200.sharding import CudaBackend

    dev = CudaBackend(Precision.F64)
    a = dev.empty(1 << 8)
    st = dev.empty(1 << 8)
    for bits, pb in (([8], 0), ([2, 2], 0), ([3], 1 << 4)):
        with pytest.raises(ShapeError):
            dev.pack_part(a, 8, bits, pb, 0, 1, st)
    with pytest.raises(ShapeError):
        dev.pack_part(a, 8, [3], 0, 100, 100, st)


@pytest.mark.parametrize("shards", [4, 8])
def test_in_process_exchanges_equal_execute(cuda, shards):
    """Circuits whose batched plans need k = log2(shards) qubit exchanges, in-process shards."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import sharding as sd

    n = 16
    rng = np.random.default_rng(3)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    for c in (q.random_grid_circuit(4, 4, 12, 42), q.qft_circuit(n),
              q.variational_circuit(n, 3, rng.uniform(0, 6, n * 7), fused=True)):
        p = sd.plan_batched(c, shards)
        assert any(isinstance(s, sd.Exchange) and s.k > 1 for s in p.steps) or p.n_exchanges <= 1
        want = c.execute(q.from_amplitudes(psi)).amplitudes
        got = q.execute_sharded(c, shards, initial=q.from_amplitudes(psi)).amplitudes
        assert max_abs(got, want) <= 1e-12


@pytest.mark.parametrize("world", [2, 4])
def test_stream_ordered_exchange_threads(cuda, world):
    """The NCCL branch of the exchange (stream_ordered: no host sync between pack, transfer and
    unpack; many chunks in flight) with every rank a thread on its own stream."""
    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import sharding as sd
    from thread_comm import run_ranks

    n = 16
    rng = np.random.default_rng(5)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / math.sqrt(2 << n)
    circuits = [q.random_grid_circuit(4, 4, 12, 7), q.qft_circuit(n)]
    wants = [c.execute(q.from_amplitudes(psi)).amplitudes for c in circuits]
    for planner in ("batched", "reference"):
        sd.SHARD_PLANNER = planner
        try:
            def fn(comm):
                outs = []
                for c in circuits:
                    sh = sd.run_sharded(c, world, q.from_amplitudes(psi), comm=comm)
                    outs.append(sd.gather_tensor(sh).cpu().numpy())
                return outs
            res = run_ranks(world, fn)
        finally:
            sd.SHARD_PLANNER = "batched"
        for r in range(world):
            for got, want in zip(res[r], wants):
                assert max_abs(got, want) <= 1e-12, (planner, r)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_permute_qubits_tiled_and_plain(cuda, prec):
    """qsb_permute_qubits (tiled through shared memory when the permutation leaves room for a
    2^10-element tile, plain otherwise) against numpy's bit permutation, random and reversal
    permutations, n = 6 .. 21."""
    torch = cuda
    from paper_2009_01845_b200 import Precision
    from paper_2009_01845_b200.sharding import CudaBackend

    p = Precision(prec)
    dev, cpu = CudaBackend(p), CpuBackend(p)
    rng = np.random.default_rng(17)
    for n in (6, 11, 14, 21):
        a = _rand(n, n, torch, p.complex_dtype)
        for perm in (list(range(n))[::-1], [int(x) for x in rng.permutation(n)], list(range(n))):
            got = dev.permute(a.cuda(), n, perm).cpu()
            want = cpu.permute(a, n, perm)
            assert torch.equal(got, want), (n, perm)
