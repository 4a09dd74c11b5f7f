import os, sys
sys.path.insert(0, '/root/repo')
import bench
from paper_2107_11650_b200 import api as A
ds, mask, hcfg, acfg = bench.make_param_inputs()
acfg.max_outer = 50
plan = A.ParamPlan(ds.data, mask, hcfg, acfg, dataset=True)
plan.set_timing(True)
plan.run(50); plan.sync()
