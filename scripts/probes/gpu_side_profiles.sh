# Launch lists (ncu gpu__time_duration) of the config-4 and config-3 probes
# and full captures of their dominant kernels, exported to CSV on the box
# (raw metrics + source-line stall samples) so only text comes back.
# ncu only after each command exited 0 without it.
set -u
mkdir -p gpurun_out
cap() {  # name kernel-regex skip command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 \
    -o /tmp/$name "$@" > /dev/null 2>&1
  echo "$name full rc=$?"
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$name.src.csv 2>/dev/null
  python scripts/ncu_hot.py /tmp/$name.src.csv 40 > gpurun_out/$name.hot.txt 2>/dev/null
}
python scripts/probes/param_probe.py > gpurun_out/p4.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/param_launches.csv python scripts/probes/param_probe.py > /dev/null 2>&1
echo "param launches rc=$?"
cap prof_param_pe svt_subspace 3 python scripts/probes/param_probe.py
cap prof_param_echo small_svt 3 python scripts/probes/param_probe.py
python scripts/probes/c3_probe.py > gpurun_out/c3.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/c3_launches.csv python scripts/probes/c3_probe.py > /dev/null 2>&1
echo "c3 launches rc=$?"
cap prof_c3 svt_subspace 12 python scripts/probes/c3_probe.py
du -sh gpurun_out
