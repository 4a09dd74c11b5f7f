"""Per-iteration count of Ritz values above the SVT threshold (subspace solvers'
diagnostic, sweeps_out // 1000) for config 3 (large d) or config 2."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from paper_2107_11650_b200 import api as A  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if which == "c3":
    import make_c3_golden as G
    y, bits = G.make_inputs()
    mask = A.SamplingMask(256, 256, bits)
    plan = A.PiPlan(y, mask, None, A.HankelConfig(pencil=246), A.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=True))
else:
    import bench
    y, mask, g, hcfg = bench.make_inputs()
    plan = A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=iters, tol=1e-300, enable_spirit=True))
plan.set_timing(True)
for it in range(iters):
    plan.run(1)
    plan.sync()
    r = plan.debug_sweeps() // 1000
    print(f"it{it + 1}: max r {r.max()} mean {r.mean():.1f} n>40 {(r > 40).sum()} n>56 {(r > 56).sum()}", flush=True)
