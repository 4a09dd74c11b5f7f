set -u
mkdir -p gpurun_out
source <(sed -n '/^cap() {/,/^}/p' scripts/gpu_profiles_r02.sh)
cap huge "svt_subspace_kernel<[^,]*496,[^,]*32,[^,]*16,[^,]*(1|true),[^,]*(0|false)>" 1 python scripts/sweep_points.py 512,32,15
