"""Distributed sharded path on the GPU: 2 ranks (torchrun, gloo with host-staged transfers, both
ranks on cuda:0) run CUDA shards, the pack/unpack kernels and the double-buffered exchange
pipeline; the gathered state must equal the single-GPU execute() result (tools/dist_check.py).
NCCL itself needs two GPUs (gpurun provides one)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_ranks_on_one_gpu(cuda, world):
    env = dict(os.environ, QSB_EXCHANGE_CHUNK_BYTES=str(1 << 15))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
                        f"--nproc-per-node={world}", os.path.join(ROOT, "tools", "dist_check.py"), "16"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert "DIST_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
