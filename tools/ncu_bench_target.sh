#!/bin/bash
# Evidence captures for profiles/: (1) the bench line, (2) the launch list of a short bench run
# (per-launch device time + DRAM bytes), (3) one full ncu capture of the dominant kernels (the
# four specialised passes of QFT-30 c128).
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-workloads \
  > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 4 -c 4 \
  -o gpurun_out/prof_qft30_full python tools/ncu_jit.py 30 f64 > gpurun_out/ncu_qft30.log 2>&1
