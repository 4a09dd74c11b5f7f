# 3xTF32 mma.sync trial: config-2 parity and phase clocks, co-located and single layouts.
set -u
mkdir -p gpurun_out
for coloc in 1 0; do
  tag=mma_coloc$coloc
  if [ $coloc = 0 ]; then export SHLR_NO_COLOC=1; else unset SHLR_NO_COLOC; fi
  SHLR_MMA=1 timeout 600 python -m pytest tests/test_gpu_c2.py -m gpu -q -x > gpurun_out/$tag.test.log 2>&1; echo "$tag test rc=$?"
  tail -3 gpurun_out/$tag.test.log
  SHLR_MMA=1 SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/$tag.phase.txt 2>&1; echo "$tag phase rc=$?"
  tail -5 gpurun_out/$tag.phase.txt
done
