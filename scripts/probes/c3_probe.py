"""Config-3 probe: full-size SHLR-V (256^2 x 32 coils, two rings, random2d mask R=6, K=11)
on the B200 path -- timing and a smoke of the large-d SVT variant."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

t0 = time.time()
ph = synth.pi_phantom(256, 256, 32, rings=2)
mask = A.mask_random2d(256, 256, 1.0 / 6.0, 24, synth.SEED_MASK)
y = np.where(mask.bits.astype(bool)[:, :, None], ph.kspace, 0)
print(f"inputs {time.time() - t0:.1f}s", flush=True)
plan = A.PiPlan(y, mask, None, A.HankelConfig(pencil=246), A.AdmmConfig(max_outer=int(os.environ.get('ITERS', 30)), tol=1e-300, enable_vc=True))
plan.run(3)
plan.sync()
for k in range(3):
    plan.run(8)
    plan.sync()
    _, tot, n = plan.timing()
    print(f"graph iters {3 + 8 * k}..{11 + 8 * k}: {tot / 8:.3f} ms/iter ({n} launches), {8e3 / tot:.1f} it/s",
          flush=True)
plan.reset()
plan.set_timing(True)
plan.run(3)
plan.sync()
svt, tot, n = plan.timing()
print(f"timing mode iters 1-3: {tot / 3:.3f} ms/iter, svt {svt / 3:.3f} ms/iter", flush=True)
plan.set_timing(False)
plan.run(int(os.environ.get('ITERS', 30)) - 3)
plan.sync()
x, st = plan.download()
print("iters", st.outer_iters, "finite", bool(np.isfinite(x).all()))
