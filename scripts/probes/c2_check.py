"""Config-2 parity margins vs the reference run (tests/golden/c2_ref50.npz):
image after N iterations through the resident plan (bench path), and the
singular values at iteration 50 through the debug path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_11650_b200 import api as A

z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/c2_ref50.npz"))
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
y, mask, g, hcfg = bench.make_inputs()
plan = A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True))
plan.run(50); plan.sync()
x, st = plan.download()
t0 = time.time()
plan.reset(); plan.run(50); plan.sync()
print(f"plan: x50 rel {rel(x, z['x50']):.3e}  ({(time.time()-t0)*1e3/50:.2f} ms/iter wall)")
if os.environ.get("SV", "1") == "1":
    svs = []
    A.shlr_pi_reconstruct(y, mask, g, hcfg, A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True),
                          debug_sv_iter=50, sv_out=svs)
    print(f"sv50 rel {rel(svs[0], z['sv50']):.3e}")
