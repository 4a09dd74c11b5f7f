set -u
mkdir -p gpurun_out
python scripts/e2e_probe.py > gpurun_out/c1_e2e.txt 2>&1; tail -5 gpurun_out/c1_e2e.txt
SHLR_Q_COLD=4 python scripts/e2e_probe.py > gpurun_out/c1_e2e_q4.txt 2>&1; tail -2 gpurun_out/c1_e2e_q4.txt
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/c1_phase.txt 2>&1; tail -5 gpurun_out/c1_phase.txt
