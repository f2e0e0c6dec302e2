for v in 0 1 0 1; do
  echo "IMMEDIATE_C128=$v"; QSB_IMMEDIATE_C128=$v QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30 > /tmp/qp.txt 2>&1; grep f64 /tmp/qp.txt
done
QSB_IMMEDIATE_C128=1 timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -x -q -p no:cacheprovider -k qft 2>&1 | tail -2
