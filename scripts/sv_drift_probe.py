"""SHLR-SV headline geometry (242 x 240 tall weighted lifts): drift vs the
reference's run at iterations 1, 2, 5, 12 (tests/golden/sv_ref12.npz), and
per-iteration time, for the subspace solver's warm-pass settings in the
environment (SHLR_Q_WARM, SHLR_INNER_QR, ...)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "sv"
g = dict(np.load(os.path.join(ROOT, "tests", "golden", "sv_ref12.npz" if which == "sv" else "c2_ref50.npz")))
iters = (1, 2, 5, 12) if which == "sv" else (1, 2, 5, 10, 50)
cfg = bench.CFG2
ph = synth.pi_phantom(256, 256, 8)
mask = A.mask_gauss_cartesian(256, cfg["rate"], cfg["acs"], synth.SEED_MASK)
y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
ker = A.SpiritKernels(5, 8, g["kernels"])
plan = A.PiPlan(y, mask, ker, A.HankelConfig(pencil=242),
                A.AdmmConfig(max_outer=max(iters), tol=1e-300, enable_spirit=True, enable_vc=(which == "sv")))
done, out = 0, []
t0 = time.perf_counter()
for it in iters:
    plan.run(it - done)
    plan.sync()
    done = it
    x, _ = plan.download()
    c = [int(i) for i in g["coils"]]
    e = max(np.linalg.norm(x[:, :, c] - g[f"x{it}_coils"]) / np.linalg.norm(g[f"x{it}_coils"]),
            np.linalg.norm(np.sqrt((np.abs(x) ** 2).sum(2)) - g[f"rss{it}"]) / np.linalg.norm(g[f"rss{it}"]))
    out.append(f"{it}:{e:.2e}")
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SHLR_"))
print(which, env or "(defaults)", " ".join(out), f"total {time.perf_counter() - t0:.3f}s", flush=True)
