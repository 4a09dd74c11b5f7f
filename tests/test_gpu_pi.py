"""GPU parity of the parallel-imaging path against the oracle at sizes the
oracle finishes in seconds, plus the reference's behavioural contracts
(determinism, stopping, divergence, full sampling, plan reuse)."""
import os
import subprocess

import numpy as np
import pytest

import shlr_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-4


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def phantom(m, n, j, seed=0):
    from paper_2107_11650_b200 import synth
    return synth.pi_phantom(m, n, j, seeds=(2107 + seed, 2108 + seed, 2109 + seed)).kspace


@pytest.mark.parametrize("shape,axis", [((6, 256, 3), 1), ((256, 5, 2), 0), ((3, 12, 7), 1),
                                        ((15, 4), 0), ((2, 128, 16), 1)])
def test_fft_matches_oracle(gpu, shape, axis):
    rng = np.random.default_rng(1)
    x = rng.normal(size=shape) + 1j * rng.normal(size=shape)
    for inv in (False, True):
        assert rel(gpu.fft_along_axis(x, axis, inv), O.fft_along_axis(x, axis, inv)) < 1e-6


def test_config1_scale_parity(gpu):
    """BASELINE config 1 geometry (128^2 x 8 coils, K = 9 -> 120 x 72 lifted
    matrices, R = 4 with 16 ACS lines, SHLR) for 8 outer iterations vs the
    oracle; singular values at the last iteration too."""
    A = gpu
    y0 = phantom(128, 128, 8)
    mk = A.mask_gauss_cartesian(128, 0.25, 16, 11650)
    y = np.where(mk.bits[0][None, :, None].astype(bool), y0, 0)
    iters = 8
    acfg = A.AdmmConfig(max_outer=iters, tol=1e-300)
    log, svs = [], []
    x = A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(pencil=120), acfg, log=log,
                              debug_sv_iter=iters, sv_out=svs)
    xo, st = O.shlr_pi_reconstruct(y, O.SamplingMask(1, 128, mk.bits), None, O.HankelConfig(pencil=120),
                                   O.AdmmConfig(max_outer=iters, tol=1e-300), sv_iters=(iters,))
    assert rel(x, xo) < TOL
    sr, sc = st.singular_values[iters]
    assert rel(svs[0], np.concatenate([sr, sc])) < TOL
    assert [l.split()[2] for l in log] == [l.split()[2] for l in st.log]


def test_config1_full_run_parity(gpu):
    """BASELINE config 1 as specified: 30 ADMM iterations on the 128^2 x 8-coil
    phantom, through the resident plan (CUDA graph, subspace SVT with warm
    start), image within 1e-4 of the oracle; the stop-rule trace too."""
    A = gpu
    y0 = phantom(128, 128, 8)
    mk = A.mask_gauss_cartesian(128, 0.25, 16, 11650)
    y = np.where(mk.bits[0][None, :, None].astype(bool), y0, 0)
    iters = 30
    plan = A.PiPlan(y, mk, None, A.HankelConfig(pencil=120), A.AdmmConfig(max_outer=iters, tol=1e-300))
    plan.run(iters)
    plan.sync()
    log = []
    x, st = plan.download(log)
    plan.close()
    xo, sto = O.shlr_pi_reconstruct(y, O.SamplingMask(1, 128, mk.bits), None, O.HankelConfig(pencil=120),
                                    O.AdmmConfig(max_outer=iters, tol=1e-300))
    assert st.outer_iters == iters
    assert rel(x, xo) < TOL
    rc = np.array([float(l.split("relchange=")[1].split()[0]) for l in log])
    rco = np.array([float(l.split("relchange=")[1].split()[0]) for l in sto.log])
    np.testing.assert_allclose(rc[:10], rco[:10], rtol=1e-2)


def test_bitwise_determinism_and_plan_reset(gpu):
    A = gpu
    y = phantom(32, 32, 4, seed=3)
    mk = A.mask_gauss_cartesian(32, 0.5, 8, 3)
    y = np.where(mk.bits[0][None, :, None].astype(bool), y, 0)
    a0, a1 = A.acs_range(32, 8)
    g = A.spirit_calibrate(y[:, a0:a1, :], 3)
    acfg = A.AdmmConfig(max_outer=5, tol=1e-300, enable_spirit=True, enable_vc=True)
    h = A.HankelConfig(pencil=11)
    x1 = A.shlr_pi_reconstruct(y, mk, g, h, acfg)
    x2 = A.shlr_pi_reconstruct(y, mk, g, h, acfg)
    assert np.array_equal(x1, x2)
    plan = A.PiPlan(y, mk, g, h, acfg)
    plan.run(5)
    plan.sync()
    x3, s3 = plan.download()
    plan.reset()
    plan.run(2)
    plan.run(3)
    plan.sync()
    x4, s4 = plan.download()
    plan.close()
    assert np.array_equal(x1, x3) and np.array_equal(x3, x4)
    assert s3.outer_iters == s4.outer_iters == 5


def test_stopping_rules_match_reference(gpu):
    """solvers.cpp:183-189: relchange < tol stops; stats record the iteration."""
    A = gpu
    y = phantom(16, 16, 2, seed=4)
    mk = A.mask_gauss_cartesian(16, 0.6, 4, 2)
    y = np.where(mk.bits[0][None, :, None].astype(bool), y, 0)
    st = A.SolveStats()
    A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(), A.AdmmConfig(max_outer=2), stats=st)
    assert st.outer_iters == 2
    A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(), A.AdmmConfig(tol=1e9), stats=st)
    assert st.outer_iters == 1
    # a realistic tolerance stops at the same iteration as the oracle
    acfg = A.AdmmConfig(max_outer=40, tol=1e-4)
    A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(), acfg, stats=st)
    _, sto = O.shlr_pi_reconstruct(y, O.SamplingMask(1, 16, mk.bits), None, O.HankelConfig(),
                                   O.AdmmConfig(max_outer=40, tol=1e-4))
    assert st.outer_iters == sto.outer_iters


def test_divergence_error(gpu):
    A = gpu
    y = phantom(16, 16, 2)
    y[8, 8, 0] = np.nan
    mk = A.mask_gauss_cartesian(16, 1.0, 0, 1)
    with pytest.raises(A.DivergenceError):
        A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(), A.AdmmConfig(max_outer=2))


def test_zero_data_returns_zeros(gpu):
    """cg_solve returns zeros for b == 0 (solvers.cpp:30-33)."""
    A = gpu
    y = np.zeros((16, 16, 2), complex)
    mk = A.mask_gauss_cartesian(16, 0.5, 4, 2)
    # D0 = 1 makes b != 0 in the first iteration; with y = 0 the solve is still finite
    x = A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(), A.AdmmConfig(max_outer=2, tol=1e-300))
    xo, _ = O.shlr_pi_reconstruct(y, O.SamplingMask(1, 16, mk.bits), None, O.HankelConfig(),
                                  O.AdmmConfig(max_outer=2, tol=1e-300))
    assert rel(x, xo) < TOL


def test_full_sampling_is_exact(gpu):
    """tests/test_solvers.cpp:184-196."""
    A = gpu
    k = phantom(32, 32, 2, seed=5)
    full = A.mask_gauss_cartesian(32, 1.0, 4, 1)
    x = A.shlr_pi_reconstruct(k, full, None, A.HankelConfig(),
                              A.AdmmConfig(lam=1e6, enable_vc=True, max_outer=10))
    direct = O.ifft2d_centered(k)
    assert rel(x, direct) < 1e-3


def test_two_dimensional_mask(gpu):
    """2D masks are allowed by apply_mask (operators.cpp:203)."""
    A = gpu
    k = phantom(32, 32, 3, seed=6)
    mk = A.mask_random2d(32, 32, 0.4, 8, 5)
    y = np.where(mk.bits[:, :, None].astype(bool), k, 0)
    x = A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(pencil=12),
                              A.AdmmConfig(max_outer=4, tol=1e-300, enable_vc=True))
    xo, _ = O.shlr_pi_reconstruct(y, O.SamplingMask(32, 32, mk.bits), None, O.HankelConfig(pencil=12),
                                  O.AdmmConfig(max_outer=4, tol=1e-300, enable_vc=True))
    assert rel(x, xo) < TOL


def test_cpp_dropin_suite(gpu):
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,j,vc,spirit", [(24, 32, 2, False, False), (40, 24, 3, True, False),
                                             (20, 28, 1, True, False), (32, 24, 2, False, True)])
def test_non_square_and_single_coil(gpu, m, n, j, vc, spirit):
    """Rows use pencil_for(N), columns pencil_for(M) (solvers.cpp:113-114): a
    non-square image has different row / column lift geometries; J = 1."""
    A = gpu
    y0 = phantom(m, n, j, seed=m + n)
    mk = A.mask_gauss_cartesian(n, 0.5, 6, 3)
    y = np.where(mk.bits[0][None, :, None].astype(bool), y0, 0)
    kern, kern_o = None, None
    if spirit:
        a0, a1 = A.acs_range(n, 6)
        kern = A.spirit_calibrate(y[:, a0:a1, :], 3)
        kern_o = O.SpiritKernels(3, j, kern.weights)
    acfg = A.AdmmConfig(max_outer=3, tol=1e-300, enable_vc=vc, enable_spirit=spirit)
    x = A.shlr_pi_reconstruct(y, mk, kern, A.HankelConfig(), acfg)
    xo, _ = O.shlr_pi_reconstruct(y, O.SamplingMask(1, n, mk.bits), kern_o, O.HankelConfig(),
                                  O.AdmmConfig(max_outer=3, tol=1e-300, enable_vc=vc, enable_spirit=spirit))
    assert rel(x, xo) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,pencil", [(5, 5, 5), (6, 7, 1), (9, 9, 0)])
def test_tiny_images_and_extreme_pencils(gpu, m, n, pencil):
    """Tiny images; pencil = N (q = 1), pencil = 1 (one-row lifts), default rule."""
    A = gpu
    y0 = phantom(m, n, 2, seed=m * n)
    mk = A.mask_gauss_cartesian(n, 0.6, 2, 4)
    y = np.where(mk.bits[0][None, :, None].astype(bool), y0, 0)
    if pencil > min(m, n):
        pytest.skip("pencil longer than a dimension")
    x = A.shlr_pi_reconstruct(y, mk, None, A.HankelConfig(pencil=pencil),
                              A.AdmmConfig(max_outer=3, tol=1e-300, enable_vc=True))
    xo, _ = O.shlr_pi_reconstruct(y, O.SamplingMask(1, n, mk.bits), None, O.HankelConfig(pencil=pencil),
                                  O.AdmmConfig(max_outer=3, tol=1e-300, enable_vc=True))
    assert rel(x, xo) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("spirit,vc,m,n,j", [(False, False, 32, 32, 3), (False, True, 32, 40, 3),
                                             (True, False, 32, 32, 3), (True, True, 24, 40, 3),
                                             (True, True, 64, 64, 3),
                                             # 8 coils: the packed Hermitian P + bulk-copy column stage
                                             # (k_spirit_cols_bulk), power-of-two and direct-DFT column lengths
                                             (True, False, 32, 32, 8), (True, True, 24, 40, 8),
                                             (True, False, 30, 20, 8), (True, False, 128, 64, 8)])
def test_gpu_normal_operator_alone_vs_oracle(gpu, spirit, vc, m, n, j):
    """The X-update operator on its own (normal_apply, operators.cpp:213-248):
    lambda F* U F + beta (row + column lift normals, weighted, virtual coils)
    + lambda1 (G - I)^H (G - I), evaluated by the device's k-space diagonal
    and SPIRiT stages (shlr_cuda_debug_normal_apply), against the oracle on a
    random image.  FP32 operator: bar 1e-5 relative L2."""
    import shlr_oracle as O
    A = gpu
    rng = np.random.default_rng(m + n + 7 * spirit + 3 * vc)
    y = rng.standard_normal((m, n, j)) + 1j * rng.standard_normal((m, n, j))
    x = rng.standard_normal((m, n, j)) + 1j * rng.standard_normal((m, n, j))
    mask = A.mask_gauss_cartesian(n, 0.5, 8, 11)
    g = None
    if spirit:
        a0, a1 = A.acs_range(n, 8)
        g = A.spirit_calibrate(np.where(mask.bits[0][None, :, None].astype(bool), y, 0)[:, a0:a1, :], 3)
    pencil = max(2, 2 * min(m, n) // 3)
    acfg = A.AdmmConfig(enable_spirit=spirit, enable_vc=vc)
    got = A.debug_normal_apply(y, mask, g, A.HankelConfig(pencil=pencil), acfg, x)
    cfg = O.HankelConfig(pencil=pencil, virtual_coil=vc)
    gop = O.SpiritImageOp(O.SpiritKernels(3, j, g.weights), m, n) if spirit else None
    want = O.normal_apply(x, O.SamplingMask(1, n, mask.bits), gop, cfg, acfg.lam, acfg.lambda1 if spirit else 0.0,
                          acfg.beta)
    assert rel(got, want) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(32, 32), (24, 40)])
def test_eight_coil_spirit_run_vs_oracle(gpu, m, n):
    """SHLR-S with 8 coils at oracle-sized geometries: the CG loop runs the
    bulk-prefetch column stage (packed Hermitian P) on power-of-two and
    direct-DFT column lengths; image and per-iteration CG counts against the
    oracle."""
    A = gpu
    y0 = phantom(m, n, 8, seed=m + n)
    mk = A.mask_gauss_cartesian(n, 0.5, 8, 5)
    y = np.where(mk.bits[0][None, :, None].astype(bool), y0, 0)
    a0, a1 = A.acs_range(n, 8)
    g = A.spirit_calibrate(y[:, a0:a1, :], 3)
    iters = 6
    acfg = A.AdmmConfig(max_outer=iters, tol=1e-300, enable_spirit=True)
    pencil = 2 * min(m, n) // 3
    log = []
    x = A.shlr_pi_reconstruct(y, mk, g, A.HankelConfig(pencil=pencil), acfg, log=log)
    xo, st = O.shlr_pi_reconstruct(y, O.SamplingMask(1, n, mk.bits), O.SpiritKernels(3, 8, g.weights),
                                   O.HankelConfig(pencil=pencil),
                                   O.AdmmConfig(max_outer=iters, tol=1e-300, enable_spirit=True))
    assert rel(x, xo) < TOL
    assert [l.split()[2] for l in log] == [l.split()[2] for l in st.log]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,axis", [((256, 256, 8), 0), ((256, 256, 8), 1), ((128, 512, 2), 1),
                                        ((96, 242, 4), 1), ((45, 64, 3), 0)])
def test_fft_cross_checked_against_cufft(gpu, shape, axis):
    """north_star: the hand-written radix / direct-DFT kernels cross-checked
    against cuFFT (torch.fft on the device, complex128), for correctness only:
    the centred unitary transform of fft.cpp:100-140 is
    fftshift(fft(ifftshift(x), norm='ortho')) along the axis."""
    import torch
    rng = np.random.default_rng(shape[0] + 7 * axis)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    xt = torch.from_numpy(x).cuda()
    for inv in (False, True):
        f = torch.fft.ifft if inv else torch.fft.fft
        ref = torch.fft.fftshift(f(torch.fft.ifftshift(xt, dim=axis), dim=axis, norm="ortho"), dim=axis).cpu().numpy()
        assert rel(gpu.fft_along_axis(x, axis, inv), ref) < 1e-6
