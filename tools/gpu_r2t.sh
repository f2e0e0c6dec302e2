set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2t_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_all.log
tail -4 gpurun_out/r2t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2t_bench.log 2>&1; tail -c 7000 gpurun_out/r2t_bench.log
