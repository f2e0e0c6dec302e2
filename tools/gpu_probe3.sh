mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/workloads.py 30 > gpurun_out/workloads30.log 2>&1; echo wl rc $?
cat gpurun_out/workloads30.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-600
