set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pi.py tests/test_gpu_c2.py tests/test_golden.py tests/test_dropin_reference.py -m gpu -q -x > gpurun_out/c2.test.log 2>&1; echo "test rc=$?"
tail -3 gpurun_out/c2.test.log
ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/c2_probe.txt 2>&1; tail -2 gpurun_out/c2_probe.txt
SHLR_SPIRIT_BULK=0 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/c2_probe_old.txt 2>&1; tail -2 gpurun_out/c2_probe_old.txt
timeout 900 python bench.py --no-cpu --no-extra > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/c2_bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['hankel_svt']['kernel_ms'], d['e2e']['value'])
P
