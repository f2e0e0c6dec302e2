set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "entropy or reduced_density or cli" > gpurun_out/r2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_tests.log
tail -15 gpurun_out/r2d_tests.log
timeout 900 python tools/big33.py 33
timeout 300 python tools/big33.py 30
