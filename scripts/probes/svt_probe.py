"""Hankel-SVT kernel probe: config-2-shaped batch (512 x 242x120), sweeps and timing."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2107_11650_b200 import synth
from paper_2107_11650_b200._lib import lib
n, nc, k, b = int(os.environ.get("N", 256)), int(os.environ.get("NC", 8)), int(os.environ.get("K", 15)), int(os.environ.get("B", 512))
p = n - k + 1
v = synth.sweep_vectors(n, nc, k, b)
tau = synth.sweep_tau(n, nc, k)
vd = torch.from_numpy(v.astype(np.complex64)).cuda()
out = torch.empty_like(vd)
sw = torch.zeros(b, dtype=torch.int32, device="cuda")
rc = lib.shlr_cuda_debug_svt_sweeps(C.c_void_p(vd.data_ptr()), b, nc, n, p, tau, C.c_void_p(out.data_ptr()), C.c_void_p(sw.data_ptr()))
torch.cuda.synchronize()
s1, s2 = (sw // 100).float(), (sw % 100).float()
print("rc", rc, "stage1 sweeps mean %.2f max %d | stage2 mean %.2f max %d" % (s1.mean(), s1.max(), s2.mean(), s2.max()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(int(os.environ.get("REPS", 3))):
    e0.record()
    lib.shlr_cuda_hankel_svt_batched(C.c_void_p(vd.data_ptr()), b, nc, n, p, C.c_float(tau), C.c_void_p(out.data_ptr()), None, None)
    e1.record(); torch.cuda.synchronize(); print("svt ms", e0.elapsed_time(e1))
