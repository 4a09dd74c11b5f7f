set -u
mkdir -p gpurun_out
/usr/bin/time -v timeout 1500 python bench.py > gpurun_out/c7_bench_full.json 2> gpurun_out/c7_bench_full.err; echo "bench rc=$?"
grep -E "Elapsed|Maximum resident" gpurun_out/c7_bench_full.err
/usr/bin/time -v timeout 1500 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/c7_ref.json 2> gpurun_out/c7_ref.err; echo "ref rc=$?"
grep -E "Elapsed" gpurun_out/c7_ref.err
tail -c 1500 gpurun_out/c7_ref.json
