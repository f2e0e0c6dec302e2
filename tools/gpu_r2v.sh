QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30 > /tmp/qp.txt 2>&1; cat /tmp/qp.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2v_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_all.log
tail -4 gpurun_out/r2v_all.log
