"""Config-2 50-iteration image vs the reference golden (resident plan, bench path) and ms/iter."""
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
plan.run(50)
plan.sync()
x, st = plan.download()
print("rel vs reference x50:", float(np.linalg.norm(x - g["x50"]) / np.linalg.norm(g["x50"])))
plan.reset()
plan.run(3)
plan.sync()
plan.run(20)
plan.sync()
print("ms/iter (iters 4-23):", plan.timing()[1] / 20)
