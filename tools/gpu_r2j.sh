set -x
QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py tests/test_gpu_layout.py -x -q -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
tail -3 gpurun_out/r2j_tests.log
timeout 300 python tools/sharded33_check.py 24 8 12
timeout 1200 python tools/sharded33_check.py 33 8 20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 4 -c 4 -o gpurun_out/r2j_qft30 python tools/ncu_workload.py qft 30 f64 > gpurun_out/r2j_ncu_qft.log 2>&1; echo "ncu qft rc $?"
