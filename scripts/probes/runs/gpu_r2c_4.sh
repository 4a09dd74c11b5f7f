set -u
mkdir -p gpurun_out
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/c4_phase.txt 2>&1; tail -7 gpurun_out/c4_phase.txt
SHLR_NO_COLOC=1 SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/c4_phase_alone.txt 2>&1; tail -7 gpurun_out/c4_phase_alone.txt
