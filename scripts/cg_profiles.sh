# Full ncu captures of the SPIRiT CG kernels of config 2 (one warm launch
# each, caches not flushed: P and the vectors stay L2-resident as in the
# step), exported to CSV on the box.  Run after bench.py exited 0 without ncu.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
for k in k_spirit_cols k_spirit_rows_fwd k_cg_b; do
  timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
    -k regex:$k -s 40 -c 1 -o /tmp/prof_$k $B > /dev/null 2>&1
  echo "$k rc=$?"
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_$k.raw.csv 2>/dev/null
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prof_$k.src.csv 2>/dev/null
  python scripts/ncu_hot.py /tmp/prof_$k.src.csv 40 > gpurun_out/prof_$k.hot.txt 2>/dev/null
done
