"""Config 3: solver level of the lifted matrices per outer iteration
(0 level 1, 1 handed to level 2, 3 stays at level 2, 4 / 5 deflation chain)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import make_c3_golden as G  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

y, bits = G.make_inputs()
plan = A.PiPlan(y, A.SamplingMask(256, 256, bits), None, A.HankelConfig(pencil=246),
                A.AdmmConfig(max_outer=50, tol=1e-300, enable_vc=True))
for it in range(1, 51):
    plan.run(1)
    lv = plan.debug_levels()
    if it >= 28:
        print(it, np.bincount(lv, minlength=6), flush=True)
