"""Large-d probes: (A) deflation-chain accuracy of the batched unit vs the
oracle for ranks beyond the 64-column level 2, per pass count; (B) per-
iteration drift of a tall SHLR-SV reconstruction vs the oracle, with the
oracle's rank above the threshold per iteration."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def unit(r):
    import shlr_oracle as O
    from paper_2107_11650_b200 import api as A
    rng = np.random.default_rng(5)
    n, nc, k = 256, 32, 15
    p = n - k + 1
    t = np.arange(n)
    v = (rng.standard_normal((4, nc, n)) + 1j * rng.standard_normal((4, nc, n))) / np.sqrt(2)
    w = rng.uniform(0, 2 * np.pi, size=(4, 1, r, 1))
    a = 4 * (rng.standard_normal((4, nc, r, 1)) + 1j * rng.standard_normal((4, nc, r, 1)))
    v = v + np.sum(a * np.exp(1j * w * t), axis=2)
    tau = float(np.sqrt(p) + np.sqrt(nc * k))
    adj, _ = A.hankel_svt_batched(v, p, tau, want_sv=False)
    adj_o, sv_o = O.hankel_svt_unit(v, p, tau)
    print(f"unit r={r} L2_Q={os.environ.get('SHLR_L2_Q')} L3_Q={os.environ.get('SHLR_L3_Q')} "
          f"rank={(sv_o > tau).sum(axis=1).tolist()} rel={rel(adj, adj_o):.3e} "
          f"per-matrix={[round(rel(adj[i], adj_o[i]), 7) for i in range(4)]}", flush=True)


def drift(m, j, pencil, vc, spirit, iters, rate=0.3, acs=16):
    import shlr_oracle as O
    from paper_2107_11650_b200 import api as A
    from paper_2107_11650_b200 import synth
    ph = synth.pi_phantom(m, m, j)
    mask = A.mask_gauss_cartesian(m, rate, acs, 11650)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    g = None
    if spirit:
        a0, a1 = A.acs_range(m, acs)
        g = A.spirit_calibrate(y[:, a0:a1, :], 5)
    acfg = A.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=vc, enable_spirit=spirit)
    plan = A.PiPlan(y, mask, g, A.HankelConfig(pencil=pencil), acfg)
    its = list(range(1, iters + 1))
    xo, st = O.shlr_pi_reconstruct(
        y, O.SamplingMask(1, m, mask.bits), O.SpiritKernels(5, j, g.weights) if spirit else None,
        O.HankelConfig(pencil=pencil), O.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=vc, enable_spirit=spirit),
        sv_iters=its, x_iters=its)
    tau = 1.0
    for it in its:
        plan.run(1)
        plan.sync()
        x, _ = plan.download()
        sr, sc = st.singular_values[it]
        rk = np.concatenate([(sr > tau).sum(axis=-1), (sc > tau).sum(axis=-1)])
        print(f"pi {m}x{j} p={pencil} vc={vc} spirit={spirit} it={it} rel={rel(x, st.images[it]):.3e} "
              f"rank max={rk.max()} mean={rk.mean():.1f}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "unit":
        unit(int(sys.argv[2]))
    elif len(sys.argv) > 1 and sys.argv[1] == "drift":
        drift(*(int(a) for a in sys.argv[2:8]))
    elif len(sys.argv) > 1 and sys.argv[1] == "config1":
        drift(128, 8, 120, 0, 0, 30, 0.25, 16)
    else:
        for r in (170, 240):
            for q2, q3 in ((5, 4), (8, 8), (16, 16)):
                env = dict(os.environ, SHLR_L2_Q=str(q2), SHLR_L3_Q=str(q3))
                subprocess.run([sys.executable, __file__, "unit", str(r)], env=env)
        drift(180, 4, 162, 1, 1, 14)
        drift(180, 4, 162, 1, 0, 14)
