set -x
timeout 600 python -m pytest tests/test_gpu_layout.py -x -q -p no:cacheprovider > gpurun_out/r2f_layout.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_layout.log
tail -30 gpurun_out/r2f_layout.log
timeout 900 python tools/big33.py 33 qft trotter
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2f_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_all.log
tail -5 gpurun_out/r2f_all.log
