# One GPU call: tests, default bench, ncu launch list and one full capture of
# the Hankel-SVT kernel (ncu only after the same command exited 0 without it).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
SHORT="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$SHORT > gpurun_out/short.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
$SHORT > gpurun_out/short2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:svt_subspace -s 2 -c 1 \
    -o gpurun_out/prof_bench $SHORT > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
