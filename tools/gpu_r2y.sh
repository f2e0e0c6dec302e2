for b in 0 1 0 1; do echo "BALANCE=$b"; QSB_BALANCE_DIAGONALS=$b QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30 > /tmp/qp.txt 2>&1; cat /tmp/qp.txt; done
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py tests/test_gpu_layout.py -x -q -p no:cacheprovider 2>&1 | tail -2
