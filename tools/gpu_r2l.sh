set -x
timeout 600 python tools/workloads.py 30 2>&1 | head -12
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
tail -3 gpurun_out/r2l_tests.log
