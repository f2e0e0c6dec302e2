timeout 900 python tools/evolve_window_times.py 30 2>&1 | grep "^templates"
timeout 600 python tools/evolve_timing.py 26 28 30
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d['workloads'].items(): print(k, round(v.get('seconds',0)*1e3,2), 'ms', v.get('passes'), round(v.get('roofline_frac', v.get('hbm_frac',0)),3), round(v.get('fp_floor_s',0)*1e3,2))"
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "trotter or evolve or adiabatic or window or grid or baseline" 2>&1 | tail -2
