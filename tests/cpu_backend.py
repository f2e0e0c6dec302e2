"""Test-only CPU stand-in for sharding.CudaBackend: the same methods on CPU torch tensors,
gates applied with the numpy oracle.  Lets the distributed runner (plans, exchanges, relabels,
shard filters, gather) run under gloo with world_size > 1 on a machine without GPUs."""

import numpy as np
import torch

from oracle import statevec as ov


class CpuBackend:
    def __init__(self, precision):
        self.precision = precision
        self.np_dtype = precision.complex_dtype
        self.t_dtype = torch.complex128 if self.np_dtype == np.complex128 else torch.complex64

    def empty(self, n):
        return torch.empty(n, dtype=self.t_dtype)

    def zeros(self, n):
        return torch.zeros(n, dtype=self.t_dtype)

    def run_local(self, shard, n_local, ngates, cache):
        a = shard.numpy()
        for g in ngates:
            tq = tuple(n_local - 1 - b for b in g.targets)
            cq = tuple(n_local - 1 - b for b in g.controls)
            if g.kind == "diag":
                m = np.diag(g.matrix)
            elif g.kind == "swap":
                m = ov.FIXED["SWAP"]
            else:
                m = g.matrix
            ov.apply_matrix(a, n_local, tq, m, cq)
        return shard

    def scale(self, shard, phase):
        shard.mul_(complex(phase))

    @staticmethod
    def _half_index(n_local, bit, half):
        e = np.arange(1 << (n_local - 1), dtype=np.int64)
        low = e & ((1 << bit) - 1)
        return ((e >> bit) << (bit + 1)) | (half << bit) | low

    def exchange_local(self, a, b, n_local, bit):
        i1 = torch.from_numpy(self._half_index(n_local, bit, 1))
        i0 = torch.from_numpy(self._half_index(n_local, bit, 0))
        tmp = a[i1].clone()
        a[i1] = b[i0]
        b[i0] = tmp

    def pack(self, shard, n_local, bit, half, first, count, staging):
        idx = torch.from_numpy(self._half_index(n_local, bit, half)[first:first + count])
        staging[:count] = shard[idx]

    def unpack(self, shard, n_local, bit, half, first, count, staging):
        idx = torch.from_numpy(self._half_index(n_local, bit, half)[first:first + count])
        shard[idx] = staging[:count]

    @staticmethod
    def _part_index(n_local, bits, part_bits):
        occ = sorted(bits)
        e = np.arange(1 << (n_local - len(bits)), dtype=np.int64)
        for p in occ:  # open a zero bit at each position, ascending (gates.py:355-360)
            low = e & ((1 << p) - 1)
            e = ((e ^ low) << 1) | low
        return e | part_bits

    def exchange_parts(self, a, b, n_local, bits, a_bits, b_bits):
        ia = torch.from_numpy(self._part_index(n_local, bits, a_bits))
        ib = torch.from_numpy(self._part_index(n_local, bits, b_bits))
        tmp = a[ia].clone()
        a[ia] = b[ib]
        b[ib] = tmp

    def pack_part(self, shard, n_local, bits, part_bits, first, count, staging):
        idx = torch.from_numpy(self._part_index(n_local, bits, part_bits)[first:first + count])
        staging[:count] = shard[idx]

    def unpack_part(self, shard, n_local, bits, part_bits, first, count, staging):
        idx = torch.from_numpy(self._part_index(n_local, bits, part_bits)[first:first + count])
        shard[idx] = staging[:count]

    def permute(self, src, n_bits, dst_bit):
        i = np.arange(1 << n_bits, dtype=np.int64)
        j = np.zeros_like(i)
        for b, d in enumerate(dst_bit):
            j |= ((i >> b) & 1) << d
        out = torch.empty_like(src)
        out[torch.from_numpy(j)] = src
        return out
