"""Quick GPU sanity run: FFT, lift map, batched SVT, small PI recon vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import shlr_oracle as O
from paper_2107_11650_b200 import api as A

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

print("devices", A.device_count(), flush=True)
rng = np.random.default_rng(0)
x = rng.standard_normal((6, 256, 3)) + 1j * rng.standard_normal((6, 256, 3))
for ax in (0, 1, 2):
    for inv in (False, True):
        g = A.fft_along_axis(x, ax, inv); o = O.fft_along_axis(x, ax, inv)
        print("fft", ax, inv, rel(g, o), flush=True)
m = A.lift_index_map(20, 7, 3, True)
print("liftmap shape", m.shape, flush=True)
for (n, nc, k, b) in [(64, 2, 7, 5), (128, 8, 15, 6), (256, 8, 15, 8), (128, 1, 31, 4), (256, 1, 7, 4)]:
    p = n - k + 1
    v = rng.standard_normal((b, nc, n)) + 1j * rng.standard_normal((b, nc, n))
    tau = np.sqrt(p) + np.sqrt(nc * k)
    t0 = time.time(); g, sg = A.hankel_svt_batched(v, p, tau); t1 = time.time()
    o, so = O.hankel_svt_unit(v, p, tau)
    print("svt", n, nc, k, "adj rel", rel(g, o), "sv rel", rel(sg, so[:, :sg.shape[1]]), "%.3fs" % (t1 - t0), flush=True)
# small PI recon
M, N, J = 32, 24, 3
y = rng.standard_normal((M, N, J)) + 1j * rng.standard_normal((M, N, J))
mk = O.mask_gauss_cartesian(N, 0.5, 6, 5)
for vc in (False, True):
    for sp in (False, True):
        g = None
        if sp:
            a0, a1 = O.acs_range(N, 6)
            g = O.spirit_calibrate(O.apply_mask(y, mk)[:, a0:a1, :], 3)
        h = O.HankelConfig(pencil=9)
        ac = O.AdmmConfig(max_outer=4, tol=1e-300, enable_vc=vc, enable_spirit=sp)
        xo, st = O.shlr_pi_reconstruct(y, mk, g, h, ac, sv_iters=(4,))
        log = []; stg = A.SolveStats()
        xg = A.shlr_pi_reconstruct(y, A.SamplingMask(1, N, mk.bits), A.SpiritKernels(3, J, g.weights) if g else None,
                                   A.HankelConfig(pencil=9), A.AdmmConfig(max_outer=4, tol=1e-300, enable_vc=vc, enable_spirit=sp), log=log, stats=stg)
        print("pi vc", vc, "sp", sp, "x rel", rel(xg, xo), stg.outer_iters, flush=True)
        print("   gpu:", log[-1]); print("   ora:", st.log[-1])
