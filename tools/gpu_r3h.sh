timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; grep -A1 "fused " /tmp/w.txt | grep -A1 f32 | head -2
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
