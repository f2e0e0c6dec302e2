"""Multi-rank check on ONE GPU: torchrun --nproc-per-node W with the gloo backend and every
rank on cuda:0 runs the distributed sharded path (CUDA shards, pack/unpack kernels, the
double-buffered exchange with host syncs) and compares the gathered state with execute()."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import sharding as sd

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
os.environ.setdefault("QSB_EXCHANGE_CHUNK_BYTES", str(1 << 16))
sd.TorchComm.CHUNK_BYTES = int(os.environ["QSB_EXCHANGE_CHUNK_BYTES"])


HostStagedComm = sd.HostStagedComm


n = int(sys.argv[1]) if len(sys.argv) > 1 else 18
worst = 0.0
for name, c in [("qft", q.qft_circuit(n)),
                ("var", q.variational_circuit(n, 2, np.random.default_rng(1).uniform(0, 6, n * 5), fused=True)),
                ("grid", q.random_grid_circuit(2, n // 2, 6, 3))]:
    sh = sd.execute_distributed(c, q.Precision.F64, comm=HostStagedComm())
    got = sd.gather(sh).amplitudes
    want = c.execute().amplitudes
    err = float(np.max(np.abs(got - want)))
    worst = max(worst, err)
    if rank == 0:
        print(f"world {world} {name}-{n}: reshuffles {sd.plan(c, world).n_reshuffles}, max|diff| {err:.2e}", flush=True)
dist.barrier()
# sharded sampling across ranks (chained cumsum over all_gather, counts all-reduced)
c = q.variational_circuit(n, 2, np.random.default_rng(5).uniform(0, 6, n * 5), fused=True)
sh = sd.execute_distributed(c, q.Precision.F64, comm=HostStagedComm())
got = sd.sample_sharded(sh, 4000, 9).samples
want = q.sample(c.execute(), range(n), 4000, 9).samples
ok = bool(np.array_equal(got, want))
if rank == 0:
    print(f"world {world} sharded sampling bit-exact: {ok}", flush=True)
worst = worst if ok else 1.0
dist.barrier()
# adiabatic evolution resident in the ranks' shards + sharded energy
cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.1, 1.0)
h0, h1 = q.build_x(n), q.build_tfim(n, 1.0)
sh = q.adiabatic_evolve_sharded(h0, h1, q.Schedule.linear(), cfg, comm=HostStagedComm())
e = sd.expectation_sharded(h1, sh)
ref = q.adiabatic_evolve(h0, h1, q.Schedule.linear(), cfg)
err = float(np.max(np.abs(sd.gather(sh).amplitudes - ref.amplitudes)))
de = abs(e - q.expectation(h1, ref))
if rank == 0:
    print(f"world {world} resident adiabatic evolution: max|diff| {err:.2e}, energy diff {de:.2e}", flush=True)
worst = max(worst, err, de / 100)
dist.barrier()
# the bench's isolated-exchange timing through the same runner pipeline (numbers meaningless here:
# every rank shares one GPU and chunks are staged through the host)
import bench  # noqa: E402

c = q.qft_circuit(n)
ep = sd.plan(c, world)
nv, _ = bench._time_exchanges(sd, HostStagedComm(), sd.CudaBackend(q.Precision.F64), q.Precision.F64, n, ep,
                              (1 << (n - (world.bit_length() - 1))) * 16, reps=2)
wl = bench._dist_adiabatic(q, sd, HostStagedComm(), n, world, steps=2)
wg = bench._dist_grid(q, sd, HostStagedComm(), n, world, q.Precision.F64, cycles=4)
if rank == 0:
    print("grid workload:", wg, flush=True)
    worst = worst if "value" in wg else 1.0
if rank == 0:
    print("exchange timing:", nv, flush=True)
    print("adiabatic step workload:", wl, flush=True)
    worst = worst if "value" in wl else 1.0
    worst = worst if "achieved" in nv else 1.0
if rank == 0:
    print("DIST_OK" if worst <= 1e-12 else "DIST_FAIL", flush=True)
dist.destroy_process_group()
