mkdir -p gpurun_out
timeout 900 python tools/workloads.py 30 > gpurun_out/workloads30.log 2>&1; echo wl rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 9 -c 3 \
  -o gpurun_out/prof_var28 python tools/ncu_workload.py variational 28 f64 > gpurun_out/ncu_var28.log 2>&1; echo ncu rc $?
