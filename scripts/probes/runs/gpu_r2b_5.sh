set -u
mkdir -p gpurun_out
timeout 120 scripts/probes/_bin/mma_rate > gpurun_out/mma_rate2.txt 2>&1; echo "mma_rate rc=$?"
grep mix gpurun_out/mma_rate2.txt
export SHLR_MMA=1 SHLR_NO_COLOC=1
for ns in 0 1; do
  tag=c8_ns${ns}
  SHLR_NS=$ns timeout 600 python -m pytest tests/test_gpu_c2.py -m gpu -q -x > gpurun_out/$tag.test.log 2>&1; echo "$tag test rc=$?"
  tail -2 gpurun_out/$tag.test.log
  SHLR_NS=$ns SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/$tag.phase.txt 2>&1; echo "$tag phase rc=$?"
  tail -5 gpurun_out/$tag.phase.txt
done
