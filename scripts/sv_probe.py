"""A few SHLR-SV iterations at the headline geometry (242 x 240 tall weighted
lifts, config-2 inputs + virtual coils) for profiling."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

y, mask, g, hcfg = bench.make_inputs()
plan = A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=12, tol=1e-300, enable_spirit=True, enable_vc=True))
plan.run(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
plan.sync()
plan.download()
print("sv probe ok")
