set -u
mkdir -p gpurun_out
SHORT="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
cap() {
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o /tmp/$name $SHORT > /dev/null 2>&1
  echo "$name rc=$?"
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$name.src.csv 2>/dev/null
  python scripts/ncu_hot.py /tmp/$name.src.csv 40 > gpurun_out/$name.hot.txt 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
}
$SHORT > /dev/null 2>&1 && echo base ok
cap prof_spirit_cols k_spirit_cols 40
cap prof_spirit_rows k_spirit_rows_fwd 40
cap prof_rowinv SpiritRowInvOp 40
cap prof_cgb k_cg_b 40
