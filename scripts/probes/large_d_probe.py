"""Large-d (d > 128) parity probe vs the oracle: PI 160^2 x 8 vc (pencil 150)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import shlr_oracle as O  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

m, j, p = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (160, 8, 150)
ph = synth.pi_phantom(m, m, j)
mask = A.mask_gauss_cartesian(m, 0.3, 16, 11650)
y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
cache = f"/tmp/orc_{m}_{j}_{p}.npz"
for it in [int(a) for a in os.environ.get('ITS', '1,2,3').split(',')]:
    acfg = A.AdmmConfig(max_outer=it, tol=1e-300, enable_vc=True)
    x = A.shlr_pi_reconstruct(y, mask, None, A.HankelConfig(pencil=p), acfg)
    xo, _ = O.shlr_pi_reconstruct(y, O.SamplingMask(1, m, mask.bits), None, O.HankelConfig(pencil=p),
                                  O.AdmmConfig(max_outer=it, tol=1e-300, enable_vc=True))
    print(it, os.environ.get("SHLR_Q_COLD"), os.environ.get("SHLR_Q_WARM"),
          float(np.linalg.norm(x - xo) / np.linalg.norm(xo)), flush=True)
