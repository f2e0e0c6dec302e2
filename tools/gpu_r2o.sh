set -x
export QSB_BENCH_DIST_BACKEND=gloo QSB_EXCHANGE_CHUNK_BYTES=$((1<<22))
timeout 900 python -m torch.distributed.run --standalone --nnodes=1 --nproc-per-node 2 bench.py --gpus 2 --steps 2 --warmup 3 --qubits 22 > gpurun_out/r2o_dist2.log 2>&1; echo "rc=$?"; tail -c 3000 gpurun_out/r2o_dist2.log
timeout 900 python -m torch.distributed.run --standalone --nnodes=1 --nproc-per-node 4 bench.py --gpus 4 --steps 2 --warmup 3 --qubits 20 > gpurun_out/r2o_dist4.log 2>&1; echo "rc=$?"; tail -c 3000 gpurun_out/r2o_dist4.log
unset QSB_BENCH_DIST_BACKEND
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q -p no:cacheprovider 2>&1 | tail -2
