mkdir -p gpurun_out
timeout 600 python tools/probe_geometry.py 30 > gpurun_out/probe_geometry.log 2>&1; echo probe rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 10 -c 2 \
  -o gpurun_out/prof_var28 python tools/ncu_workload.py variational 28 f64 > gpurun_out/ncu_var28.log 2>&1; echo ncu rc $?
