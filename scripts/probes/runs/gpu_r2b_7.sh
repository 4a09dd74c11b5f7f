set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g2_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g2_gputest.log
timeout 900 python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo "bench rc=$?"
python - <<'P'
import json
l=[x for x in open('gpurun_out/g2_bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['hankel_svt']['kernel_ms'])
for k,v in d.get('other_workloads',{}).items():
    print(k, v.get('value'), v.get('ms_per_step'))
P
