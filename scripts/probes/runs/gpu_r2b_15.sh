set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/td.test.log 2>&1; echo "test rc=$?"
tail -3 gpurun_out/td.test.log
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/td.phase.txt 2>&1; tail -5 gpurun_out/td.phase.txt
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/td_bench.json 2> gpurun_out/td_bench.err; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/td_bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['hankel_svt']['kernel_ms'])
for k,v in d.get('other_workloads',{}).items():
    print('  ', k, v.get('value'), v.get('ms_per_step'), v.get('svt_ms'))
P
