"""Where the e2e (one full shlr_pi_reconstruct call) time goes: plan create /
run / download / destroy, twice."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

y, mask, g, hcfg = bench.make_inputs()
acfg = A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True)
for rep in range(3):
    t0 = time.perf_counter()
    plan = A.PiPlan(y, mask, g, hcfg, acfg)
    t1 = time.perf_counter()
    plan.run(1)
    plan.sync()
    t2 = time.perf_counter()
    plan.run(49)
    plan.sync()
    t3 = time.perf_counter()
    x, st = plan.download()
    t4 = time.perf_counter()
    plan.close()
    t5 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, iter1 {1e3*(t2-t1):.1f}, iters2-50 {1e3*(t3-t2):.1f}, "
          f"download {1e3*(t4-t3):.1f}, destroy {1e3*(t5-t4):.1f}", flush=True)
t0 = time.perf_counter()
A.shlr_pi_reconstruct(y, mask, g, hcfg, acfg)
print(f"one call {1e3*(time.perf_counter()-t0):.1f} ms")
