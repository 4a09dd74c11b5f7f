set -u
mkdir -p gpurun_out
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/c9_phase.txt 2>&1; tail -6 gpurun_out/c9_phase.txt
timeout 900 python bench.py --no-cpu --no-extra > gpurun_out/c9_bench.json 2> gpurun_out/c9_bench.err; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/c9_bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['hankel_svt']['kernel_ms'], d['e2e']['value'])
P
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
timeout 600 ncu --kernel-name-base demangled --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k "regex:svt_subspace_kernel<[^,]*120,[^,]*48," -s 2 -c 1 $B 2>&1 | grep -E "dram__|gpu__time|lts__"
timeout 1200 python -m pytest tests/test_gpu_c2.py tests/test_gpu_param.py -m gpu -q -x 2>&1 | tail -2
