set -u
mkdir -p gpurun_out
export SHLR_MMA=1 SHLR_NS=1
tag=pf_coloc
timeout 600 python -m pytest tests/test_gpu_c2.py -m gpu -q -x > gpurun_out/$tag.test.log 2>&1; echo "$tag test rc=$?"
tail -2 gpurun_out/$tag.test.log
SHLR_PHASE_CLK=1 ITERS=8 timeout 300 python scripts/pi_probe.py > gpurun_out/$tag.phase.txt 2>&1; echo "$tag phase rc=$?"
tail -5 gpurun_out/$tag.phase.txt
unset SHLR_MMA SHLR_NS
timeout 900 python -m pytest tests/test_gpu_large_d.py tests/test_gpu_c3.py tests/test_gpu_sv.py -m gpu -q -x > gpurun_out/pf_large.test.log 2>&1; echo "large-d tests rc=$?"
tail -3 gpurun_out/pf_large.test.log
timeout 300 python scripts/probes/sv_time.py 14 > gpurun_out/pf_sv.txt 2>&1; tail -4 gpurun_out/pf_sv.txt
