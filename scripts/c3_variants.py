"""Config 3 (246 x 704 lifts, d = 246): ms per iteration over 30 iterations
and parity against the reference's own 30-iteration run (c3_ref30.npz) for
the large-d settings in the environment."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import make_c3_golden as G  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "c3_ref30.npz"))
y, bits = G.make_inputs()
plan = A.PiPlan(y, A.SamplingMask(256, 256, bits), None, A.HankelConfig(pencil=246),
                A.AdmmConfig(max_outer=30, tol=1e-300, enable_vc=True))
plan.run(30)
plan.sync()
_, total_ms, _ = plan.timing()
x, _ = plan.download()
coils = [int(c) for c in g["coils"]]
e1 = np.linalg.norm(x[:, :, coils] - g["x30_coils"]) / np.linalg.norm(g["x30_coils"])
rss = np.sqrt((np.abs(x) ** 2).sum(2))
e2 = np.linalg.norm(rss - g["rss30"]) / np.linalg.norm(g["rss30"])
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SHLR_"))
print(f"c3 {env or '(defaults)'}: {total_ms / 30:.2f} ms/iter, coils {e1:.2e}, rss {e2:.2e}", flush=True)
