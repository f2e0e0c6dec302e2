timeout 300 python tools/permute_bench.py 30
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_sharding.py tests/test_gpu_layout.py -x -q -p no:cacheprovider 2>&1 | tail -2
