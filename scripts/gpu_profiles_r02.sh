# Round-2 profile captures (each program first ran to exit 0 without ncu):
#   launches.csv          launch list of the headline bench (config 2, short)
#   prof_<name>.raw.csv   ncu --set full of one launch, raw page
#   prof_<name>.hot.txt   hottest source lines
set -u
mkdir -p gpurun_out
SHORT="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
if [ -z "${SKIP_LAUNCHES:-}" ]; then
$SHORT > gpurun_out/short.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv $SHORT > /dev/null 2>&1
echo "launch list rc=$?"
fi
cap() {  # name, kernel regex, skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  "$@" > /dev/null 2>&1 || { echo "$name: program failed"; return; }
  rm -f /tmp/prof_$name.ncu-rep
  timeout 1200 ncu --kernel-name-base demangled --set full --clock-control none --import-source on \
    -k "regex:$rx" -s $skip -c 1 -o /tmp/prof_$name "$@" > /dev/null 2>&1
  echo "$name rc=$?"
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_$name.raw.csv 2>/dev/null
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prof_$name.src.csv 2>/dev/null
  python scripts/ncu_hot.py /tmp/prof_$name.src.csv 40 > gpurun_out/prof_$name.hot.txt 2>/dev/null
}
cap c2_svt "svt_subspace_kernel<[^,]*120,[^,]*48," 2 $SHORT
[ -z "${SKIP_COLS:-}" ] && cap c2_cols "k_spirit_cols" 40 $SHORT
cap sv_tall "svt_subspace_kernel<[^,]*248,[^,]*48," 3 python scripts/sv_probe.py 6
cap huge "svt_subspace_kernel<[^,]*496,[^,]*32,[^,]*16,[^,]*(1|true),[^,]*(0|false)," 1 python scripts/sweep_points.py 512,32,15
cap smalld "svt_subspace_kernel<[^,]*56,[^,]*16," 1 python scripts/sweep_points.py 256,8,7
ls -la gpurun_out/
