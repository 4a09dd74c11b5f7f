"""Config 3 against the reference's 50-iteration run (tests/golden/c3_ref50.npz):
relative L2 errors at the dumped iterations and the solver levels."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import make_c3_golden as G  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "c3_ref50.npz"))
y, bits = G.make_inputs()
plan = A.PiPlan(y, A.SamplingMask(256, 256, bits), None, A.HankelConfig(pencil=246),
                A.AdmmConfig(max_outer=50, tol=1e-300, enable_vc=True))
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
coils = [int(c) for c in g["coils"]]
done = 0
for it in [int(i) for i in g["iters"]]:
    t0 = time.perf_counter()
    plan.run(it - done)
    plan.sync()
    dt = (time.perf_counter() - t0) / (it - done) * 1e3
    done = it
    lv = np.bincount(plan.debug_levels(), minlength=6)
    log = []
    x, _ = plan.download(log)
    e1 = rel(x[:, :, coils], g[f"x{it}_coils"])
    e2 = rel(np.sqrt((np.abs(x) ** 2).sum(axis=2)), g[f"rss{it}"].astype(np.float64))
    print(f"iteration {it}: coils {e1:.2e} rss {e2:.2e} levels {lv.tolist()} ({dt:.1f} ms per iteration)", flush=True)
if "log" in g:
    cg = [l.split()[2] for l in log]
    print("cg_iters equal to the reference's:", cg == [str(l).split()[2] for l in g["log"]])
