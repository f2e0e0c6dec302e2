# usage: bash tools/gpu_prof.sh <tag> <workload> <n> <prec> <skip> <count>
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s $5 -c $6 \
  -o gpurun_out/prof_$1 python tools/ncu_workload.py $2 $3 $4 > gpurun_out/ncu_$1.log 2>&1; echo ncu $1 rc $?
