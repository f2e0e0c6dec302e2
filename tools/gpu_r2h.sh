set -x
for ts in 0 1; do
  echo "=== QSB_TMA_STORE=$ts"
  QSB_TMA_STORE=$ts QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30
  QSB_TMA_STORE=$ts timeout 600 python tools/workloads.py 30 2>&1 | grep -v "per pass" | head -6
done
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py tests/test_gpu_layout.py -x -q -p no:cacheprovider > gpurun_out/r2h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_tests.log
tail -3 gpurun_out/r2h_tests.log
timeout 900 python tools/big33.py 33 qft-api qft
