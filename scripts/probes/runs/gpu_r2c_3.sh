set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 130 -c 70 --csv --log-file gpurun_out/c3_warm_launches.csv $B > /dev/null 2>&1; echo "rc=$?"
SHLR_SPIRIT_BULK=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 130 -c 70 --csv --log-file gpurun_out/c3_warm_launches_old.csv $B > /dev/null 2>&1; echo "rc=$?"
