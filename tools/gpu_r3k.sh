timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -x -q -p no:cacheprovider -k "window or trotter" 2>&1 | tail -2
timeout 900 python tools/evolve_timing.py 26 28 30
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['workloads'], indent=0)[:2500])"
