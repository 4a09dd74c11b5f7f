"""Config 1 (128^2 x 8, 256 lifts of 120 x 72): resident-plan step time."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

ph = synth.pi_phantom(128, 128, 8)
mask = A.mask_gauss_cartesian(128, 0.25, 16, synth.SEED_MASK)
y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
plan = A.PiPlan(y, mask, None, A.HankelConfig(pencil=120), A.AdmmConfig(max_outer=60, tol=1e-300))
plan.run(5)
plan.sync()
for rep in range(3):
    plan.run(15)
    plan.sync()
    _, total_ms, _ = plan.timing()
    print(f"{total_ms / 15:.4f} ms per step", flush=True)
plan.set_timing(True)
plan.run(3)
plan.sync()
svt, tot, _ = plan.timing()
print(f"timing mode: svt {svt / 3:.4f} ms, total {tot / 3:.4f} ms")
