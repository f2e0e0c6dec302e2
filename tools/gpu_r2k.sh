set -x
timeout 300 python tools/sharded33_check.py 24 8 12
timeout 1200 python tools/sharded33_check.py 33 8 20
# profiles: variational-30 c64 passes 2 and 4, c128 split pass 2, Trotter step passes
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 11 -c 3 -o gpurun_out/r2k_var30c64 python tools/ncu_workload.py variational 30 f32 > gpurun_out/r2k_ncu1.log 2>&1; echo "ncu rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 11 -c 1 -o gpurun_out/r2k_var30c128 python tools/ncu_workload.py variational 30 f64 > gpurun_out/r2k_ncu2.log 2>&1; echo "ncu rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 5 -c 5 -o gpurun_out/r2k_trot30 python tools/ncu_workload.py trotter 30 f64 > gpurun_out/r2k_ncu3.log 2>&1; echo "ncu rc $?"
