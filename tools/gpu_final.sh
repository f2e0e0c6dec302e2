timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -3
timeout 1200 python bench.py > /tmp/b.log 2>&1; tail -1 /tmp/b.log > gpurun_out/bench_line.json; python -c "
import json; d=json.load(open('gpurun_out/bench_line.json'))
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['roofline'], d['clocks'], d['e2e'])
for k,v in d['workloads'].items(): print(k, round(v.get('seconds',0)*1e3,2), 'ms', v.get('passes'), round(v.get('roofline_frac', v.get('hbm_frac',0)),3))"
