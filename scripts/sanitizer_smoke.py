"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): PI with SPIRiT + vc (full solver and subspace), the
large-d subspace levels, the parameter path (small-SVT echo kernel, PE
levels), the batched unit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

rng = np.random.default_rng(0)
# PI, full solver (d small), SPIRiT + vc
m, n, j = 24, 24, 3
y = rng.standard_normal((m, n, j)) + 1j * rng.standard_normal((m, n, j))
mask = A.mask_gauss_cartesian(n, 0.5, 6, 1)
g = A.spirit_calibrate(np.where(mask.bits[0][None, :, None].astype(bool), y, 0)[:, 9:15, :], 3)
A.shlr_pi_reconstruct(y, mask, g, A.HankelConfig(pencil=9), A.AdmmConfig(max_outer=2, tol=1e-300,
                                                                            enable_spirit=True, enable_vc=True))
print("pi small ok", flush=True)
# PI, subspace level 1 (d = 72)
ph = synth.pi_phantom(96, 96, 8)
mk = A.mask_gauss_cartesian(96, 0.3, 12, 2)
yk = np.where(mk.bits[0][None, :, None].astype(bool), ph.kspace, 0)
A.shlr_pi_reconstruct(yk, mk, None, A.HankelConfig(pencil=87), A.AdmmConfig(max_outer=2, tol=1e-300))
print("pi subspace ok", flush=True)
# large-d (d = 150, vc)
ph = synth.pi_phantom(160, 160, 8)
mk = A.mask_gauss_cartesian(160, 0.3, 16, 3)
yk = np.where(mk.bits[0][None, :, None].astype(bool), ph.kspace, 0)
A.shlr_pi_reconstruct(yk, mk, None, A.HankelConfig(pencil=150), A.AdmmConfig(max_outer=2, tol=1e-300,
                                                                             enable_vc=True))
print("pi large-d ok", flush=True)
# parameter path
yp = rng.standard_normal((3, 40, 12, 2)) + 1j * rng.standard_normal((3, 40, 12, 2))
bits = np.stack([A.mask_gauss_cartesian(40, 0.4, 6, 10 + e).bits[0] for e in range(12)], axis=1)
A.recon_param_dataset(A.ParameterDataset(yp, [10.0 * (e + 1) for e in range(12)]), A.SamplingMask(40, 12, bits),
                      A.HankelConfig(pencil=28), A.AdmmConfig(max_outer=2, tol=1e-300, enable_vc=True))
print("param ok", flush=True)
# batched unit
v = synth.sweep_vectors(256, 8, 31, 2)
A.hankel_svt_batched(v, 226, synth.sweep_tau(256, 8, 31), want_sv=False)
v = synth.sweep_vectors(128, 8, 15, 2)
A.hankel_svt_batched(v, 114, synth.sweep_tau(128, 8, 15))
print("unit ok", flush=True)
# tall weighted large-d with virtual coils (SHLR-V, 162 x 152)
ph = synth.pi_phantom(180, 180, 4)
mk = A.mask_gauss_cartesian(180, 0.3, 16, 4)
yk = np.where(mk.bits[0][None, :, None].astype(bool), ph.kspace, 0)
A.shlr_pi_reconstruct(yk, mk, None, A.HankelConfig(pencil=162), A.AdmmConfig(max_outer=2, tol=1e-300,
                                                                             enable_vc=True))
print("pi tall large-d ok", flush=True)
# deflation chain (242 x 480, ~90 values above tau) and the HUGE variant (498 x 480)
t = np.arange(256)
v = (rng.standard_normal((1, 32, 256)) + 1j * rng.standard_normal((1, 32, 256))) / np.sqrt(2)
w = rng.uniform(0, 2 * np.pi, size=(1, 1, 90, 1))
a = 4 * (rng.standard_normal((1, 32, 90, 1)) + 1j * rng.standard_normal((1, 32, 90, 1)))
v = v + np.sum(a * np.exp(1j * w * t), axis=2)
A.hankel_svt_batched(v, 242, float(np.sqrt(242) + np.sqrt(480)), want_sv=False)
print("deflation chain ok", flush=True)
v = synth.sweep_vectors(512, 32, 15, 1)
A.hankel_svt_batched(v, 498, synth.sweep_tau(512, 32, 15), want_sv=False)
print("huge ok", flush=True)
# metrics and the lift-stage index dumps
A.ssos(rng.standard_normal((20, 20, 3)) + 0j)
A.mssim(np.abs(rng.standard_normal((20, 20))), np.abs(rng.standard_normal((20, 20))))
A.rlne(np.abs(rng.standard_normal((20, 20))) + 1, np.abs(rng.standard_normal((20, 20))))
for path in (0, 1, 2):
    A.lift_index_map(40, 30, 2, True, path)
print("metrics + index maps ok", flush=True)
