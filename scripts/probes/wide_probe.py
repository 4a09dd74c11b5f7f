"""Wide-lift (p < blocks*q) parity probe of the full and subspace solvers vs the oracle:
singular values of L + D/beta at iteration 1 (debug hook) and images after 1..3 iterations."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import shlr_oracle as O  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

m, j, p, vc = (int(a) for a in sys.argv[1:5])
ph = synth.pi_phantom(m, m, j)
mask = A.mask_gauss_cartesian(m, 0.3, 16, 11650)
y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
xo, st = O.shlr_pi_reconstruct(y, O.SamplingMask(1, m, mask.bits), None, O.HankelConfig(pencil=p),
                               O.AdmmConfig(max_outer=3, tol=1e-300, enable_vc=bool(vc)), sv_iters=(1, 2))
for it in (1, 2):
    svs = []
    acfg = A.AdmmConfig(max_outer=it, tol=1e-300, enable_vc=bool(vc))
    A.shlr_pi_reconstruct(y, mask, None, A.HankelConfig(pencil=p), acfg, debug_sv_iter=it, sv_out=svs)
    sr, sc = st.singular_values[it]
    ref = np.concatenate([sr, sc])
    print(f"sv it{it}: rel {rel(svs[0], ref):.3e}  rows {rel(svs[0][:m], sr):.3e} cols {rel(svs[0][m:], sc):.3e}",
          flush=True)
for it in (1, 2, 3):
    acfg = A.AdmmConfig(max_outer=it, tol=1e-300, enable_vc=bool(vc))
    x = A.shlr_pi_reconstruct(y, mask, None, A.HankelConfig(pencil=p), acfg)
    xo_i, _ = O.shlr_pi_reconstruct(y, O.SamplingMask(1, m, mask.bits), None, O.HankelConfig(pencil=p),
                                    O.AdmmConfig(max_outer=it, tol=1e-300, enable_vc=bool(vc)))
    print(f"x it{it}: {rel(x, xo_i):.3e}", flush=True)
