set -x
timeout 600 python tools/workloads.py 30 2>&1 | grep -v "per pass" | head -8
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2n_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_all.log
tail -4 gpurun_out/r2n_all.log
