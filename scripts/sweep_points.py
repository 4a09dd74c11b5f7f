"""Time chosen config-5 sweep points (slices = 1) on the device:
python scripts/sweep_points.py 256,8,7 128,8,7 ..."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

peak = A.fp32_peak_tflops()
for arg in sys.argv[1:]:
    n, nc, k = (int(x) for x in arg.split(","))
    p, batch = n - k + 1, 2 * n
    e, d = max(p, nc * k), min(p, nc * k)
    dv = torch.from_numpy(synth.sweep_vectors(n, nc, k, batch).astype(np.complex64)).cuda()
    do = torch.empty_like(dv)
    tau = synth.sweep_tau(n, nc, k)
    for _ in range(3):  # warm-up: lazy kernel loading of every level, clocks
        A.hankel_svt_batched_device(dv.data_ptr(), batch, nc, n, p, tau, do.data_ptr())
    torch.cuda.synchronize()
    times = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A.hankel_svt_batched_device(dv.data_ptr(), batch, nc, n, p, tau, do.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    tf = batch * bench.svt_flops(e, d) / (ms * 1e-3) / 1e12
    print(f"{n}x{nc}x{k} ({p}x{nc * k}) batch {batch}: median {ms:.3f} ms (min {min(times):.3f}, max {max(times):.3f}), {tf:.2f} TF/s = {tf / peak:.3f} of FP32 peak",
          flush=True)
