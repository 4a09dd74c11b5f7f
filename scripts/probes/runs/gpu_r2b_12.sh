set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_param.py tests/test_gpu_c2.py tests/test_gpu_svt.py -m gpu -q > gpurun_out/pm.test.log 2>&1; echo "test rc=$?"
tail -3 gpurun_out/pm.test.log
for m in 1 0; do
SHLR_MMA=$m timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/pm_bench$m.json 2> gpurun_out/pm_bench$m.err; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/pm_bench$m.json') if x.startswith('{')]
d=json.loads(l[-1])
print('mma=$m', d['value'], d['ms_per_step'], d['roofline']['frac'], d['hankel_svt']['kernel_ms'])
for k,v in d.get('other_workloads',{}).items():
    print('  ', k, v.get('value'), v.get('ms_per_step'), v.get('svt_ms'))
P
done
