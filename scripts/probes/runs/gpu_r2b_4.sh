# Newton-Schulz trial on top of the 3xTF32 path: parity, phase clocks, then an
# ncu capture of the single-CTA tensor variant.
set -u
mkdir -p gpurun_out
export SHLR_MMA=1
for ns in 0 1; do
for coloc in 1 0; do
  tag=ns${ns}_coloc$coloc
  if [ $coloc = 0 ]; then export SHLR_NO_COLOC=1; else unset SHLR_NO_COLOC; fi
  SHLR_NS=$ns timeout 600 python -m pytest tests/test_gpu_c2.py -m gpu -q -x > gpurun_out/$tag.test.log 2>&1; echo "$tag test rc=$?"
  tail -3 gpurun_out/$tag.test.log
  SHLR_NS=$ns SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/$tag.phase.txt 2>&1; echo "$tag phase rc=$?"
  tail -5 gpurun_out/$tag.phase.txt
done
done
