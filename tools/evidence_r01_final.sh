#!/bin/bash
# Round-1 end evidence: bench line, launch list of a short bench run, full ncu of the QFT-30
# passes and of variational-30 pass 4 (the slowest 2-qubit-gate pass), on the current build.
mkdir -p gpurun_out
bash tools/ncu_bench_target.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 13 -c 1 \
  -o gpurun_out/prof_var30_p4 python tools/ncu_workload.py variational 30 f64 > gpurun_out/ncu_var30.log 2>&1
echo "var30 ncu rc $?"
python tools/ncu_summary.py gpurun_out/prof_qft30_full.ncu-rep > gpurun_out/qft30_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_var30_p4.ncu-rep > gpurun_out/var30_p4_summary.txt 2>&1
ls -la gpurun_out
