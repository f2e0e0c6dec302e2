set -x
for sp in 0 1; do
  echo "=== QSB_SPLIT_2Q=$sp"
  QSB_SPLIT_2Q=$sp timeout 600 python tools/workloads.py 30 2>&1 | head -9
done
QSB_SPLIT_2Q=1 timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
tail -3 gpurun_out/r2g_tests.log
timeout 600 python -m pytest tests/test_gpu_layout.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2g_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_all.log
tail -5 gpurun_out/r2g_all.log
