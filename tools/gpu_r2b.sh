set -x
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_distributed.py tests/test_gpu_sharding.py -x -q -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_tests.log
tail -15 gpurun_out/r2b_tests.log
for tpc in 8 32; do
  echo "=== QSB_TILES_PER_CTA=$tpc"
  QSB_TILES_PER_CTA=$tpc QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30
  QSB_TILES_PER_CTA=$tpc timeout 600 python tools/workloads.py 30 2>&1 | grep -v "per pass"
done
