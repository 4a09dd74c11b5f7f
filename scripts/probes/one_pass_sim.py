"""FP64 simulation (numpy, host) of two warm-started inexact SVT schemes inside
the oracle's ADMM loop, against the exact SVT:

  A  (the kernel's scheme)   V' = orth(A^H A V), Rayleigh-Ritz on A V'
  B  (one pass)              Q = orth(A V), B = Q^H A, SVD of the small B
  C  (carried power step)    V' = orth(W), W = A_old^H A_old V_old carried from the
                             previous outer iteration; one pass Y1 = A V', X2 = A^H Y1,
                             Rayleigh-Ritz on H = V'^H X2; W_next = X2 U

Prints the relative image error of each scheme per outer iteration.  A design
probe only: nothing in the product or the tests imports it.

    python scripts/probes/one_pass_sim.py [N] [J] [pencil] [iters] [kb]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import shlr_oracle as O  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
J = int(sys.argv[2]) if len(sys.argv) > 2 else 8
P = int(sys.argv[3]) if len(sys.argv) > 3 else 114
ITERS = int(sys.argv[4]) if len(sys.argv) > 4 else 12
KB = int(sys.argv[5]) if len(sys.argv) > 5 else 48
SPIRIT = int(os.environ.get("SPIRIT", "1"))

exact_svt = O.svt


class Approx:
    def __init__(self, scheme):
        self.scheme = scheme
        self.V = {}
        self.call = 0
        self.maxrank = 0

    def __call__(self, m, tau, return_sv=False):
        key = self.call % 2
        self.call += 1
        wide = m.shape[-1] > m.shape[-2]
        a = np.conj(np.swapaxes(m, -1, -2)) if wide else m  # e x d, d = min
        if key not in self.V:
            u, s, vh = np.linalg.svd(a, full_matrices=False)
            self.V[key] = np.conj(np.swapaxes(vh, -1, -2))[..., :KB].copy()
            z = (u * np.maximum(s - tau, 0.0)[..., None, :]) @ vh
        else:
            v = self.V[key]
            if self.scheme == "A":
                x = np.conj(np.swapaxes(a, -1, -2)) @ (a @ v)
                q, _ = np.linalg.qr(x)
                y1 = a @ q
                h = np.conj(np.swapaxes(y1, -1, -2)) @ y1
                lam, u = np.linalg.eigh(h)
                lam, u = lam[..., ::-1], u[..., ::-1]
                sig = np.sqrt(np.maximum(lam, 0))
                f = np.where(sig > tau, 1 - tau / np.maximum(sig, 1e-300), 0.0)
                vu = q @ u
                z = ((y1 @ u) * f[..., None, :]) @ np.conj(np.swapaxes(vu, -1, -2))
                self.V[key] = vu
            elif self.scheme == "C":
                # power step with the PREVIOUS matrix (carried W = G_old V_old), then a
                # consistent Rayleigh-Ritz with the new matrix from ONE pass:
                # Y1 = A V', X2 = A^H Y1, H = V'^H X2
                q, _ = np.linalg.qr(v)
                y1 = a @ q
                x2 = np.conj(np.swapaxes(a, -1, -2)) @ y1
                h = np.conj(np.swapaxes(q, -1, -2)) @ x2
                h = 0.5 * (h + np.conj(np.swapaxes(h, -1, -2)))
                lam, u = np.linalg.eigh(h)
                lam, u = lam[..., ::-1], u[..., ::-1]
                sig = np.sqrt(np.maximum(lam, 0))
                f = np.where(sig > tau, 1 - tau / np.maximum(sig, 1e-300), 0.0)
                vu = q @ u
                z = ((y1 @ u) * f[..., None, :]) @ np.conj(np.swapaxes(vu, -1, -2))
                self.V[key] = x2 @ u
            else:
                y = a @ v
                q, _ = np.linalg.qr(y)
                b = np.conj(np.swapaxes(q, -1, -2)) @ a
                ub, sig, wh = np.linalg.svd(b, full_matrices=False)
                z = ((q @ ub) * np.maximum(sig - tau, 0.0)[..., None, :]) @ wh
                self.V[key] = np.conj(np.swapaxes(wh, -1, -2))
            self.maxrank = max(self.maxrank, int((sig > tau).sum(axis=-1).max()))
        if wide:
            z = np.conj(np.swapaxes(z, -1, -2))
        return (z, np.zeros(1)) if return_sv else z


def run(svt_fn, y, mask, g, hcfg, acfg):
    O.svt = svt_fn
    try:
        x, st = O.shlr_pi_reconstruct(y, mask, g, hcfg, acfg, x_iters=tuple(range(1, ITERS + 1)))
    finally:
        O.svt = exact_svt
    return st


def main():
    y0 = synth.pi_phantom(N, N, J, seeds=(2107, 2108, 2109)).kspace
    acs = 24 if N >= 256 else 16
    mk = O.mask_gauss_cartesian(N, 0.25, acs, 11650)
    bits = np.asarray(mk.bits).reshape(1, -1)
    y = np.where(bits[0][None, :, None].astype(bool), y0, 0)
    g = None
    if SPIRIT:
        a0, a1 = O.acs_range(N, acs)
        g = O.spirit_calibrate(y[:, a0:a1, :], 5)
    acfg = O.AdmmConfig(max_outer=ITERS, tol=1e-300, enable_spirit=bool(SPIRIT))
    hcfg = O.HankelConfig(pencil=P)
    ref = run(exact_svt, y, mk, g, hcfg, acfg)
    print("exact done", flush=True)
    for scheme in os.environ.get("SCHEMES", "A,B,C").split(","):
        ap = Approx(scheme)
        st = run(ap, y, mk, g, hcfg, acfg)
        errs = [np.linalg.norm(st.images[k] - ref.images[k]) / np.linalg.norm(ref.images[k])
                for k in range(1, ITERS + 1)]
        print(scheme, "max rank", ap.maxrank, " ".join(f"{e:.1e}" for e in errs), flush=True)


if __name__ == "__main__":
    main()
