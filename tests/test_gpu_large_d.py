"""Lifted matrices with min(m, n) > 128 (BASELINE config 3: 246 x 704 with
32 coils + virtual coils; config-5 sweep points 242 x 480, 226 x 248):
the large-d subspace variant of the Hankel-SVT kernel (spectra read from L2
per chunk, adjoint streamed out block by block) against the oracle."""
import numpy as np
import pytest

import shlr_oracle as O

TOL = 1e-4


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.gpu
@pytest.mark.parametrize("m,j,pencil,iters", [(160, 8, 150, 10), (256, 12, 246, 2)])
def test_gpu_pi_large_d_vs_oracle(gpu, m, j, pencil, iters):
    """SHLR-V (virtual coils) on a seeded phantom: wide lifted matrices
    pencil x 2J(m - pencil + 1) with d = pencil > 128.  The subspace SVT's
    warm start (one pass per ADMM iteration) leaves transient FP32 errors of
    up to ~1e-3 in the first iterations of the 160 case, damped by the ADMM
    (2.9e-5 at 10 iterations, 1.2e-5 at 20): the parity point is 10."""
    from paper_2107_11650_b200 import synth
    A = gpu
    ph = synth.pi_phantom(m, m, j)
    mask = A.mask_gauss_cartesian(m, 0.3, 16, 11650)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    acfg = A.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=True)
    log = []
    x = A.shlr_pi_reconstruct(y, mask, None, A.HankelConfig(pencil=pencil), acfg, log=log)
    xo, st = O.shlr_pi_reconstruct(y, O.SamplingMask(1, m, mask.bits), None, O.HankelConfig(pencil=pencil),
                                   O.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=True))
    assert rel(x, xo) < TOL
    assert [l.split()[2] for l in log] == [l.split()[2] for l in st.log]  # cg_iters


@pytest.mark.gpu
@pytest.mark.parametrize("n,nc,k", [(256, 32, 15), (256, 8, 31), (256, 16, 31)])
def test_gpu_svt_unit_large_d(gpu, n, nc, k):
    from paper_2107_11650_b200 import synth
    A = gpu
    p = n - k + 1
    v = synth.sweep_vectors(n, nc, k, 6)
    tau = synth.sweep_tau(n, nc, k)
    out, _ = A.hankel_svt_batched(v, p, tau, want_sv=False)
    ref, _ = O.hankel_svt_unit(v, p, tau)
    assert rel(out, ref) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("r,minrank", [(90, 64), (170, 125), (240, 180)])
def test_gpu_svt_unit_large_d_deflated_level3(gpu, r, minrank):
    """242 x 480 lifts with ~90 / ~160 / ~230 singular values above the
    threshold: beyond the 64-column level 2, so level 2 keeps its leading 56
    Ritz pairs (Z1) and the deflated level 3 solves the orthogonal remainder
    (SVT(A) = SVT(A P1) + SVT(A (I - P1)) for an invariant P1), deflating its
    own leading 56 again (the chain) while the remainder is wider than its
    block: no rank limit."""
    A = gpu
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
    assert (sv_o > tau).sum(axis=1).min() > minrank
    assert rel(adj, adj_o) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("m,j,pencil,vc,spirit,iters", [
    (160, 8, 144, False, False, 10),   # plain SHLR, K = 17: 144 x 136 (tall, d = 136)
    (180, 4, 162, True, False, 10),    # SHLR-V: 162 x 152 (tall, d = 152)
    (180, 4, 162, True, True, 16),     # SHLR-SV: SPIRiT + virtual coils, tall d = 152
])
def test_gpu_pi_tall_weighted_large_d_vs_oracle(gpu, m, j, pencil, vc, spirit, iters):
    """Tall weighted lifts with 128 < d <= 248 (p > B q: SHLR-V / SHLR-SV at
    256^2 x 8 with K = 15 lift to 242 x 240, plain SHLR with K = 17..28 to
    240..229 x 136..224): the large-d subspace levels with the adjoint
    weighting conj(wc) and the virtual-coil dagger applied to each chunk's
    partial anti-diagonal sums (adjoint_lift_weighted, operators.cpp:60-91).

    Parity point: these non-power-of-two geometries without the SPIRiT
    term's conditioning are sensitive to FP32 perturbations in the first
    ADMM iterations (the 15-step capped CG is not linear in its right-hand
    side): scripts/defl_probe.py measures up to ~2e-3 at iterations 2-4 --
    the FP32 full Jacobi solver alone gives 2.5e-4 at iteration 3 of a
    256 x 8 case -- damped below 1e-4 by iteration ~10 (SPIRiT: ~14)."""
    from paper_2107_11650_b200 import synth
    A = gpu
    q = m - pencil + 1
    blocks = j * (2 if vc else 1)
    assert pencil > blocks * q > 128  # tall, large d
    ph = synth.pi_phantom(m, m, j)
    mask = A.mask_gauss_cartesian(m, 0.3, 16, 11650)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    g = None
    if spirit:
        a0, a1 = A.acs_range(m, 16)
        g = A.spirit_calibrate(y[:, a0:a1, :], 5)
    acfg = A.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=vc, enable_spirit=spirit)
    log = []
    x = A.shlr_pi_reconstruct(y, mask, g, A.HankelConfig(pencil=pencil), acfg, log=log)
    xo, st = O.shlr_pi_reconstruct(
        y, O.SamplingMask(1, m, mask.bits), O.SpiritKernels(5, j, g.weights) if spirit else None,
        O.HankelConfig(pencil=pencil),
        O.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=vc, enable_spirit=spirit))
    assert rel(x, xo) < TOL
    assert [l.split()[2] for l in log] == [l.split()[2] for l in st.log]  # cg_iters


@pytest.mark.gpu
@pytest.mark.parametrize("fe", [100, 120])
def test_gpu_param_tall_weighted_large_d_pe_lift(gpu, fe):
    """Parameter path with PE lifts 180 x 168 (N = 200, 4 coils + virtual
    coils, pencil 180: tall weighted, d = 168 > 128): the large-d levels with
    the deflation chain behind them.  One FE slice of a seeded T2 phantom
    (shlr_param_reconstruct_slice, solvers.cpp:193-298) against the oracle."""
    from paper_2107_11650_b200 import synth
    A = gpu
    n, l, j, pencil = 200, 12, 4, 180
    _, k, _, _ = synth.t2_phantom(n, n, j, l)
    hybrid = O.fft_along_axis(k, 0, True)[fe]                       # N x L x J plane at one FE line
    bits = np.stack([O.mask_gauss_cartesian(n, 0.25, 16, 40 + e).bits[0] for e in range(l)], axis=1)
    y = hybrid * bits[:, :, None]
    acfg = dict(max_outer=20, tol=1e-300, enable_vc=True)
    x = A.shlr_param_reconstruct_slice(y, A.SamplingMask(n, l, bits), A.HankelConfig(pencil=pencil),
                                       A.AdmmConfig(**acfg))
    xo, _ = O.shlr_param_reconstruct_slice(y, O.SamplingMask(n, l, bits), O.HankelConfig(pencil=pencil),
                                           O.AdmmConfig(**acfg))
    assert rel(x, xo) < TOL
