# Re-entry validation call: probe, full GPU tests, default bench.
set -u
mkdir -p gpurun_out
timeout 120 scripts/probes/_bin/mma_rate > gpurun_out/mma_rate.txt 2>&1; echo "mma_rate rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g1_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g1_gputest.log
timeout 900 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?"
cat gpurun_out/mma_rate.txt
