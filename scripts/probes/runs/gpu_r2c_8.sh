set -u
mkdir -p gpurun_out
python scripts/sweep_points.py 128,8,7 256,8,7 512,8,7 128,8,15 2>&1 | tail -4
SHLR_SMALLD_COLOC=0 python scripts/sweep_points.py 128,8,7 256,8,7 512,8,7 128,8,15 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_svt.py -m gpu -q -x 2>&1 | tail -3
time (timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/c8_ref.json 2> gpurun_out/c8_ref.err); echo "ref rc=$?"
tail -c 600 gpurun_out/c8_ref.json; grep -c libshlr_b200 /proc/self/maps
