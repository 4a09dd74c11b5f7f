"""Config 3 beyond level 2: 50 iterations run (level-3 deflation), and a
small large-d case forced through level 3 against the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import shlr_oracle as O  # noqa: E402
from paper_2107_11650_b200 import api as A  # noqa: E402

# unit-level: wide 242 x 480 lifts with 90 signal components -> level 3
rng = np.random.default_rng(5)
n, nc, k, r = 256, 32, 15, 90
p = n - k + 1
t = np.arange(n)
v = (rng.standard_normal((4, nc, n)) + 1j * rng.standard_normal((4, nc, n))) / np.sqrt(2)
w = rng.uniform(0, 2 * np.pi, size=(4, 1, r, 1))
a = 4 * (rng.standard_normal((4, nc, r, 1)) + 1j * rng.standard_normal((4, nc, r, 1)))
v = v + np.sum(a * np.exp(1j * w * t), axis=2)
tau = float(np.sqrt(p) + np.sqrt(nc * k))
adj_o, sv_o = O.hankel_svt_unit(v, p, tau)
print("rank above tau:", (sv_o > tau).sum(axis=1))
try:
    adj, _ = A.hankel_svt_batched(v, p, tau, want_sv=False)
    print("unit rel:", float(np.linalg.norm(adj - adj_o) / np.linalg.norm(adj_o)))
except Exception as e:
    print("unit:", type(e).__name__, str(e)[:120])
