"""Config-2 plan probe: per-iteration sweeps (warm start) and SVT timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_11650_b200 import api as A
y, mask, g, hcfg = bench.make_inputs()
warm = int(os.environ.get("WARM", 1))
acfg = A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True)
plan = A.PiPlan(y, mask, g, hcfg, acfg)
plan.set_warm_start(bool(warm))
plan.set_timing(True)
iters = int(os.environ.get("ITERS", 12))
for it in range(iters):
    plan.run(1); plan.sync()
    svt_ms, tot, _ = plan.timing()
    sw = plan.debug_sweeps()
    s1, s2 = sw // 100, sw % 100
    print(f"iter {it+1}: svt {svt_ms:.2f} ms total {tot:.2f} ms | stage1 mean {s1.mean():.2f} max {s1.max()} | stage2 mean {s2.mean():.2f} max {s2.max()}", flush=True)
