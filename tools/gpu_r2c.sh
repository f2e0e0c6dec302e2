set -x
timeout 1200 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py tests/test_gpu_sharding.py -x -q -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
tail -5 gpurun_out/r2c_tests.log
for ch in 1 2 4; do
  echo "=== dynamic chunk=$ch"
  QSB_DYN_CHUNK=$ch QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30
  QSB_DYN_CHUNK=$ch timeout 600 python tools/workloads.py 30 2>&1 | grep -v "per pass" | head -7
done
