"""Tensor-core precision trial for the Hankel-SVT contractions (VERDICT r1
item 5, north_star: "tensor cores only if 3xTF32 split precision meets the
tolerance").  CPU emulation: the FP64 oracle's PI reconstruction (config-1
geometry 128^2 x 8, K = 9, 30 iterations) with its SVT replaced by a
Gram-eigendecomposition SVT whose two streaming contractions -- the Gram
G = A^H A and Z = A W -- run in one of
  fp32     float32 products, float32 accumulation (the CUDA-core kernel)
  tf32     operands rounded to TF32 (10-bit mantissa), float32 accumulation
           (one tcgen05 kind::tf32 MMA per real product)
  3xtf32   a = hi + lo split, hi*hi + hi*lo + lo*hi in float32 (3 MMAs)
with the small eigendecomposition in FP64.  Reports the image relative L2
error against the unmodified FP64 oracle after 30 iterations (bar 1e-4).
Usage: python scripts/tf32_trial.py [iters]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import shlr_oracle as O  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402


def tf32(a):
    """Round float32 values to TF32 (sign, 8-bit exponent, 10-bit mantissa), nearest even."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 13) & 1
    u = ((u + 0x0FFF + lsb) & ~np.uint64(0x1FFF)).astype(np.uint32)
    return u.view(np.float32)


def cmat(x):
    return x.astype(np.complex64)


def mm(a, b, mode):
    """Complex batched product a @ b with the real products in `mode`."""
    a, b = cmat(a), cmat(b)
    if mode == "fp32":
        return (a @ b).astype(np.complex128)
    ar, ai, br, bi = (np.ascontiguousarray(v, dtype=np.float32) for v in (a.real, a.imag, b.real, b.imag))

    def rp(x, y):  # one real product in the mode
        if mode == "tf32":
            return tf32(x) @ tf32(y)
        xh, yh = tf32(x), tf32(y)
        xl, yl = tf32(x - xh), tf32(y - yh)
        return xh @ yh + (xh @ yl + xl @ yh)

    re = rp(ar, br) - rp(ai, bi)
    im = rp(ar, bi) + rp(ai, br)
    return (re + 1j * im).astype(np.complex128)


def make_svt(mode):
    def svt(m, tau, return_sv=False):
        ah = np.conj(np.swapaxes(m, -1, -2))
        g = mm(ah, m, mode)                       # Gram A^H A (streaming contraction 1)
        g = 0.5 * (g + np.conj(np.swapaxes(g, -1, -2)))
        lam, v = np.linalg.eigh(g)                # small Hermitian eigenproblem, FP64
        sig = np.sqrt(np.maximum(lam, 0.0))
        f = np.where(sig > tau, 1.0 - tau / np.where(sig > 0, sig, 1.0), 0.0)
        w = (v * f[..., None, :]) @ np.conj(np.swapaxes(v, -1, -2))
        z = mm(m, w, mode)                        # Z = A W (streaming contraction 2)
        return (z, sig[..., ::-1]) if return_sv else z
    return svt


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    ph = synth.pi_phantom(128, 128, 8)
    mask = O.mask_gauss_cartesian(128, 0.25, 16, synth.SEED_MASK)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    args = (y, mask, None, O.HankelConfig(pencil=120), O.AdmmConfig(max_outer=iters, tol=1e-300))
    ref, _ = O.shlr_pi_reconstruct(*args)
    orig = O.svt
    for mode in ("fp32", "tf32", "3xtf32"):
        O.svt = make_svt(mode)
        try:
            x, _ = O.shlr_pi_reconstruct(*args)
        finally:
            O.svt = orig
        print(f"{mode:7s} image rel L2 after {iters} iterations: "
              f"{np.linalg.norm(x - ref) / np.linalg.norm(ref):.3e}", flush=True)


if __name__ == "__main__":
    main()
