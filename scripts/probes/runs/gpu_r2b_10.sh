set -u
mkdir -p gpurun_out
python scripts/sweep_points.py 256,1,15 256,1,7 256,1,31 128,1,15 512,1,15 > gpurun_out/tiny_points.txt 2>&1; cat gpurun_out/tiny_points.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tiny_launches.csv python scripts/sweep_points.py 256,1,15 256,1,31 > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/tiny_launches.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    print(r[ki][:90], r[vi])
P
