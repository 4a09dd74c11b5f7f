"""Bitwise repeatability of full-size runs (two independent plans each): a race
in a kernel shows up as differing bits (compute-sanitizer is closed on this
pool: profiles/r02_sanitizer_refused.txt)."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import bench  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402
from paper_2107_11650_b200 import synth  # noqa: E402


def digest(x):
    return hashlib.sha1(np.ascontiguousarray(x).tobytes()).hexdigest()[:16]


def twice(name, make, iters):
    d = []
    for _ in range(2):
        plan = make()
        plan.run(iters)
        plan.sync()
        x, _ = plan.download()
        plan.close()
        d.append(digest(x))
    print(f"{name}: {d[0]} {d[1]} {'EQUAL' if d[0] == d[1] else 'DIFFERENT'}", flush=True)
    return d[0] == d[1]


ok = True
y, mask, g, hcfg = bench.make_inputs()
ok &= twice("config 2 (SHLR-S, 50 iterations)",
            lambda: A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True)), 50)
ok &= twice("SHLR-SV (12 iterations)",
            lambda: A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=12, tol=1e-300, enable_spirit=True, enable_vc=True)), 12)
ph = synth.pi_phantom(128, 128, 8)
m1 = A.mask_gauss_cartesian(128, 0.25, 16, synth.SEED_MASK)
y1 = np.where(m1.bits[0][None, :, None].astype(bool), ph.kspace, 0)
ok &= twice("config 1 (30 iterations)",
            lambda: A.PiPlan(y1, m1, None, A.HankelConfig(pencil=120), A.AdmmConfig(max_outer=30, tol=1e-300)), 30)
import make_c3_golden as G  # noqa: E402
y3, bits3 = G.make_inputs()
ok &= twice("config 3 (50 iterations, deflation chain)",
            lambda: A.PiPlan(y3, A.SamplingMask(256, 256, bits3), None, A.HankelConfig(pencil=246),
                             A.AdmmConfig(max_outer=50, tol=1e-300, enable_vc=True)), 50)
print("ALL EQUAL" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
