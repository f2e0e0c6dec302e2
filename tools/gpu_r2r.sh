set -x
for v in 0 1; do
  QSB_IMMEDIATE_C64=$v timeout 600 python tools/workloads.py 30 2>&1 | grep -A1 "f32" | head -4
  QSB_IMMEDIATE_C64=$v QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30 | tail -1
done
QSB_IMMEDIATE_C64=1 timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/evolve_timing.py 26 28
