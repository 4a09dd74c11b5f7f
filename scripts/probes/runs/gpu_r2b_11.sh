set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_c2.py tests/test_golden.py -m gpu -q -x > gpurun_out/st.test.log 2>&1; echo "test rc=$?"
tail -2 gpurun_out/st.test.log
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/st.phase.txt 2>&1; echo "phase rc=$?"
tail -5 gpurun_out/st.phase.txt
python bench.py --no-e2e --no-cpu --no-extra 2>/dev/null | tail -1 | cut -c1-200
