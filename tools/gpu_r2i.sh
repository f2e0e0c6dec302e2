set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2i_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_all.log
tail -8 gpurun_out/r2i_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2i_bench.log 2>&1; tail -c 5000 gpurun_out/r2i_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 4 -c 4 -o gpurun_out/r2i_qft30 python tools/ncu_workload.py qft 30 f64 > gpurun_out/r2i_ncu_qft.log 2>&1; echo "ncu qft rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2i_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-workloads > gpurun_out/r2i_ncu_bench.log 2>&1; echo "ncu launches rc $?"
