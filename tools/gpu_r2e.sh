set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "entropy or reduced_density or cli" > gpurun_out/r2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests.log
tail -3 gpurun_out/r2e_tests.log
# ncu: QFT-30 (4 passes), variational-30 c128 (10 passes), Trotter step n=30 (5 passes)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 4 -c 4 -o gpurun_out/r2_qft30 python tools/ncu_workload.py qft 30 f64 > gpurun_out/r2_ncu_qft.log 2>&1; echo "ncu qft rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 13 -c 2 -o gpurun_out/r2_var30 python tools/ncu_workload.py variational 30 f64 > gpurun_out/r2_ncu_var.log 2>&1; echo "ncu var rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 5 -c 1 -o gpurun_out/r2_trot30 python tools/ncu_workload.py trotter 30 f64 > gpurun_out/r2_ncu_trot.log 2>&1; echo "ncu trot rc $?"
ls -la gpurun_out/
