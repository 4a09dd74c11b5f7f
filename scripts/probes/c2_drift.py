"""Config 2 drift against the reference's dumped iterations (c2_ref50.npz)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "c2_ref50.npz"))
y, mask, kern, hcfg = bench.make_inputs()
plan = A.PiPlan(y, mask, kern, hcfg, A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True))
done = 0
out = []
for it in (1, 2, 5, 10, 50):
    plan.run(it - done)
    done = it
    x, _ = plan.download()
    c = [int(k) for k in g["coils"]]
    ref = g[f"x{it}_coils"]
    out.append(f"{it}: {float(np.linalg.norm(x[:, :, c] - ref) / np.linalg.norm(ref)):.2e}")
print("drift", " | ".join(out))
