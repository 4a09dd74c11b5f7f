"""Config-4 e2e breakdown: one recon_param_dataset call (50 iterations) vs the resident plan."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

ds, mask, hcfg, acfg = bench.make_param_inputs()
acfg.max_outer = 1
A.recon_param_dataset(ds, mask, hcfg, acfg)
acfg.max_outer = 50
for rep in range(2):
    t0 = time.perf_counter()
    A.recon_param_dataset(ds, mask, hcfg, acfg)
    print(f"call {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
t0 = time.perf_counter()
plan = A.ParamPlan(ds.data, mask, hcfg, acfg, dataset=True)
t1 = time.perf_counter()
plan.run(1); plan.sync()
t2 = time.perf_counter()
plan.run(49); plan.sync()
t3 = time.perf_counter()
plan.download()
t4 = time.perf_counter()
plan.close()
print(f"create {1e3*(t1-t0):.1f} iter1 {1e3*(t2-t1):.1f} iters2-50 {1e3*(t3-t2):.1f} download(log) {1e3*(t4-t3):.1f}")
