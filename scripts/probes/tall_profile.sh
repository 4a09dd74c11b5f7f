# ncu capture of the tall large-d subspace kernel (config-5 point 250 x 224),
# exported to CSV on the box.  Run after tall_probe.py exited 0 without ncu.
set -u
mkdir -p gpurun_out
rm -f /tmp/prof_tall.ncu-rep
timeout 900 ncu --kernel-name-base demangled --set full --clock-control none --import-source on -k "regex:svt_subspace_kernel<[^,]*248,[^,]*48," -s 1 -c 1 \
  -o /tmp/prof_tall python scripts/probes/tall_probe.py > /dev/null 2>&1
echo "tall rc=$?"
ncu -i /tmp/prof_tall.ncu-rep --page raw --csv > gpurun_out/prof_tall.raw.csv 2>/dev/null
ncu -i /tmp/prof_tall.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prof_tall.src.csv 2>/dev/null
python scripts/ncu_hot.py /tmp/prof_tall.src.csv 40 > gpurun_out/prof_tall.hot.txt 2>/dev/null
