set -u
mkdir -p gpurun_out
time (timeout 1500 python bench.py > gpurun_out/c7_bench_full.json 2> gpurun_out/c7_bench_full.err); echo "bench rc=$?"
time (timeout 1500 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/c7_ref.json 2> gpurun_out/c7_ref.err); echo "ref rc=$?"
tail -c 1500 gpurun_out/c7_ref.json
