# Phase clocks of the headline SVT (co-located large-d layout vs one CTA per SM)
# and a fresh ncu capture of the kept variant.
set -u
mkdir -p gpurun_out
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/phase_coloc.txt 2>&1; echo "coloc rc=$?"
SHLR_NO_COLOC=1 SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/phase_single.txt 2>&1; echo "single rc=$?"
tail -6 gpurun_out/phase_coloc.txt; tail -6 gpurun_out/phase_single.txt
SKIP_COLS=1 bash scripts/gpu_profiles_r02.sh 2>&1 | grep -v "^-\|^total\|^d" | head -20
