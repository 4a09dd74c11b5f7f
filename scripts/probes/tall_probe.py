"""Config-5 tall large-d point (default N=256, Nc=32, K=7: 250 x 224, batch 2N)
through hankel_svt_batched_device, device-resident, a few cold solves: the
launch an ncu capture of the tall BIG subspace kernel targets."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

n, nc, k = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 32, 7)))
p, batch = n - k + 1, 2 * n
v = synth.sweep_vectors(n, nc, k, batch)
tau = synth.sweep_tau(n, nc, k)
dv = torch.from_numpy(v.astype(np.complex64)).cuda()
do = torch.empty_like(dv)
for _ in range(3):
    A.hankel_svt_batched_device(dv.data_ptr(), batch, nc, n, p, tau, do.data_ptr(), 0,
                                torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print(f"tall probe {p}x{nc * k} batch {batch}: ok, |out| {float(do.abs().sum()):.4e}")
