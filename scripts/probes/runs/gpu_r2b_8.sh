set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_pi.py tests/test_golden.py tests/test_gpu_sv.py -m gpu -q > gpurun_out/g3_test.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g3_test.log
for u in 0 1; do
  if [ $u = 1 ]; then export SHLR_CG_UNFUSED=1; else unset SHLR_CG_UNFUSED; fi
  ITERS=8 timeout 300 python scripts/pi_probe.py 2>&1 | tail -1
  python bench.py --no-e2e --no-cpu --no-extra 2>/dev/null | tail -1 | cut -c1-200
done
