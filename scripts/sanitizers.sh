# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (scripts/sanitizer_smoke.py); summaries to gpurun_out/sanitizer_<tool>.txt
set -u
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout ${TLIM:-1500} /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    python scripts/sanitizer_smoke.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.txt
  tail -3 gpurun_out/sanitizer_$tool.txt
done
