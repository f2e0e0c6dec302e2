timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3j_all.log 2>&1; echo "rc=$?" >> gpurun_out/r3j_all.log; tail -3 gpurun_out/r3j_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r3j_bench.log 2>&1; tail -c 6000 gpurun_out/r3j_bench.log
