set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_large_d.py -m gpu -q -x > gpurun_out/g1_large_d.log 2>&1; echo "large_d rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g1_gputest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --no-extra --no-cpu > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/g1_gputest.log
