# Final-variant captures of the round: launch list + ncu --set full of the
# headline SVT kernel (tensor variant) and of the SHLR-SV large-d kernel.
set -u
mkdir -p gpurun_out
SKIP_COLS=1 bash scripts/gpu_profiles_r02.sh 2>&1 | grep "rc="
