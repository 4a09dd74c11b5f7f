set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pi.py tests/test_golden.py tests/test_dropin_reference.py -m gpu -q > gpurun_out/c1.test.log 2>&1; echo "test rc=$?"
tail -3 gpurun_out/c1.test.log
for c in 1 0; do
if [ $c = 0 ]; then export SHLR_NO_COLOC=1; else unset SHLR_NO_COLOC; fi
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/c1_bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print('coloc=$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['hankel_svt']['kernel_ms'])
for k,v in d.get('other_workloads',{}).items():
    print('  ', k, v.get('value'), v.get('ms_per_step'), v.get('svt_ms'))
P
done
