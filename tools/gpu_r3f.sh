timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3f_all.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_all.log; tail -3 gpurun_out/r3f_all.log
timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; grep "fused\|trotter\|grid" /tmp/w.txt
timeout 900 python tools/big33.py 33 trotter grid > /tmp/b.txt 2>&1; grep -v "^   " /tmp/b.txt
