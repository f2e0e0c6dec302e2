timeout 1200 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py tests/test_gpu_sharding.py -x -q -p no:cacheprovider -k "trotter or evolve or adiabatic or window" 2>&1 | tail -2
timeout 900 python tools/evolve_timing.py 26 30
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d['workloads'].items(): print(k, round(v['seconds']*1e3,2), 'ms', v.get('passes'), round(v.get('roofline_frac', v.get('hbm_frac',0)),3), round(v.get('fp_floor_s',0)*1e3,2))"
