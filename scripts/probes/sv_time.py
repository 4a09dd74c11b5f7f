"""SHLR-SV (242 x 240 tall weighted lifts, config-2 inputs + virtual coils):
per-iteration SVT time of the large-d path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

y, mask, g, hcfg = bench.make_inputs()
plan = A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=30, tol=1e-300, enable_spirit=True, enable_vc=True))
plan.set_timing(True)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 14):
    plan.run(1)
    plan.sync()
    svt_ms, tot, _ = plan.timing()
    print(f"iter {it + 1}: svt {svt_ms:.2f} ms total {tot:.2f} ms", flush=True)
