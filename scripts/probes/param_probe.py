"""Config-4 timing probe: resident ParamPlan, warm-up, then graph-mode and
timing-mode (per-launch SVT events) iterations.  Usage: python scripts/param_probe.py [M] [vc]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = dict(bench.CFG4)
if len(sys.argv) > 2:
    cfg["vc"] = bool(int(sys.argv[2]))
t0 = time.time()
ds, mask, hcfg, acfg = bench.make_param_inputs(cfg, m=m)
print(f"inputs {time.time() - t0:.1f}s", flush=True)
t0 = time.time()
plan = A.ParamPlan(ds.data, mask, hcfg, acfg, dataset=True)
print(f"plan {time.time() - t0:.1f}s", flush=True)
plan.run(3)
plan.sync()
plan.run(10)
plan.sync()
_, tot, n = plan.timing()
print(f"graph: {tot / 10:.3f} ms/iter ({n} launches/iter), {1e3 * 10 / tot:.1f} it/s", flush=True)
plan.set_timing(True)
plan.run(5)
plan.sync()
svt, tot, n = plan.timing()
print(f"timing mode: {tot / 5:.3f} ms/iter, svt {svt / 5:.3f} ms/iter", flush=True)
