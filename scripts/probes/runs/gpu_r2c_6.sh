set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c6.test.log 2>&1; echo "test rc=$?"
tail -3 gpurun_out/c6.test.log
timeout 900 python bench.py --no-cpu > gpurun_out/c6_bench.json 2> gpurun_out/c6_bench.err; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/c6_bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['hankel_svt']['kernel_ms'], d['e2e']['value'])
for k,v in d.get('other_workloads',{}).items():
    print('  ', k, v.get('value'), v.get('ms_per_step'), v.get('svt_ms'), (v.get('e2e') or {}).get('value'))
P
