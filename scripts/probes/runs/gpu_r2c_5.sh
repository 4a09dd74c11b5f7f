set -u
mkdir -p gpurun_out
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/c5_phase.txt 2>&1; tail -7 gpurun_out/c5_phase.txt
timeout 1200 python -m pytest tests/test_gpu_c2.py tests/test_gpu_pi.py tests/test_gpu_param.py tests/test_gpu_svt.py -m gpu -q -x > gpurun_out/c5.test.log 2>&1; echo "test rc=$?"
tail -3 gpurun_out/c5.test.log
