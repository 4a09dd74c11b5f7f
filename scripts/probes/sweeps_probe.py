"""Full-solver Jacobi sweep counts (stage1 * 100 + stage2) per matrix, PI cold iteration."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

m, j, p, vc = (int(a) for a in sys.argv[1:5])
ph = synth.pi_phantom(m, m, j)
mask = A.mask_gauss_cartesian(m, 0.3, 16, 11650)
y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
plan = A.PiPlan(y, mask, None, A.HankelConfig(pencil=p), A.AdmmConfig(max_outer=3, tol=1e-300, enable_vc=bool(vc)))
plan.set_timing(True)
for it in range(2):
    plan.run(1)
    plan.sync()
    sw = plan.debug_sweeps()
    s1, s2 = sw // 100, sw % 100
    print(f"it{it + 1}: stage1 max {s1.max()} mean {s1.mean():.1f} | stage2 max {s2.max()} mean {s2.mean():.1f} "
          f"| n(stage1>=20) {(s1 >= 20).sum()} n(stage2>=20) {(s2 >= 20).sum()}", flush=True)
