"""GPU parity of the batched Hankel-SVT unit (BASELINE config 5) against the
oracle on the sweep's synthetic inputs: every sweep point with d = min(p, Nc K)
<= 128 (singular values and adjoints), every point with 128 < d <= 248
(adjoints: the large-d subspace path has no exact singular-value output),
loud NotImplementedError for d > 248; plus size-independent properties at
full batch."""
import numpy as np
import pytest

import shlr_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


SWEEP = [(n, nc, k) for n in (128, 256, 512) for nc in (1, 8, 32) for k in (7, 15, 31)
         if min(n - k + 1, nc * k) <= 128]


@pytest.mark.parametrize("n,nc,k", SWEEP)
def test_sweep_point_parity(gpu, n, nc, k):
    from paper_2107_11650_b200 import synth
    b = 6
    v = synth.sweep_vectors(n, nc, k, b)
    tau = synth.sweep_tau(n, nc, k)
    p = n - k + 1
    adj, sv = gpu.hankel_svt_batched(v, p, tau)
    adj_o, sv_o = O.hankel_svt_unit(v, p, tau)
    assert rel(sv, sv_o) < TOL
    assert rel(adj, adj_o) < TOL


def test_threshold_extremes(gpu):
    rng = np.random.default_rng(0)
    v = rng.normal(size=(4, 3, 40)) + 1j * rng.normal(size=(4, 3, 40))
    # tau = 0: identity on the lifted matrix -> adjoint of the lift = counts * v
    adj, _ = gpu.hankel_svt_batched(v, 31, 0.0)
    assert rel(adj, O.hankel_counts(40, 31) * v) < 1e-5
    # tau above sigma_max: annihilation
    adj, sv = gpu.hankel_svt_batched(v, 31, 1e6)
    assert np.max(np.abs(adj)) == 0.0
    assert sv.shape == (4, 30)


def test_rank_one_analytic(gpu):
    """Rank-1 Hankel: v = a e^{jwt} lifts to a rank-1 matrix with sigma =
    |a| sqrt(p q); SVT scales it by (1 - tau/sigma) (test_solvers.cpp:47)."""
    n, p = 64, 40
    q = n - p + 1
    t = np.arange(n)
    v = (2.0 * np.exp(1j * 0.3 * t)).reshape(1, 1, n)
    sigma = 2.0 * np.sqrt(p * q)
    tau = 0.25 * sigma
    adj, sv = gpu.hankel_svt_batched(v, p, tau)
    assert abs(sv[0, 0] - sigma) < 1e-5 * sigma
    assert np.max(sv[0, 1:]) < 1e-3 * sigma
    assert rel(adj, 0.75 * O.hankel_counts(n, p) * v) < 1e-5


def test_full_batch_properties(gpu):
    """BASELINE config-2 geometry at full batch (512 x 242 x 120): singular
    values match the oracle on a sample and the SVT is non-expansive."""
    from paper_2107_11650_b200 import synth
    n, nc, k, b = 256, 8, 15, 512
    v = synth.sweep_vectors(n, nc, k, b)
    tau = synth.sweep_tau(n, nc, k)
    adj, sv = gpu.hankel_svt_batched(v, n - k + 1, tau)
    idx = [0, 17, 255, 511]
    adj_o, sv_o = O.hankel_svt_unit(v[idx], n - k + 1, tau)
    assert rel(sv[idx], sv_o) < TOL
    assert rel(adj[idx], adj_o) < TOL
    assert np.all(np.diff(sv, axis=1) <= 0)
    w = v + 0.01 * np.random.default_rng(1).normal(size=v.shape)
    adj2, _ = gpu.hankel_svt_batched(w, n - k + 1, tau)
    # non-expansive in the lifted domain -> adjoint differences bounded by counts * input diff
    lhs = np.linalg.norm(adj2 - adj)
    rhs = np.linalg.norm(O.hankel_counts(n, n - k + 1) * (w - v))
    assert lhs <= rhs * (1 + 1e-4)


ALL = [(n, nc, k) for n in (128, 256, 512) for nc in (1, 8, 32) for k in (7, 15, 31)]
BIG = [(n, nc, k) for n, nc, k in ALL if 128 < min(n - k + 1, nc * k) <= 248]
HUGE = [(n, nc, k) for n, nc, k in ALL if min(n - k + 1, nc * k) > 248]


@pytest.mark.parametrize("n,nc,k", BIG)
def test_sweep_point_large_d_parity(gpu, n, nc, k):
    from paper_2107_11650_b200 import synth
    v = synth.sweep_vectors(n, nc, k, 4)
    tau = synth.sweep_tau(n, nc, k)
    p = n - k + 1
    adj, _ = gpu.hankel_svt_batched(v, p, tau, want_sv=False)
    adj_o, _ = O.hankel_svt_unit(v, p, tau)
    assert rel(adj, adj_o) < TOL


@pytest.mark.parametrize("n,nc,k", HUGE)
def test_sweep_point_huge_d_parity(gpu, n, nc, k):
    """Config-5 points with d > 248 (498 x 480, 482 x 992): the HUGE variant
    (32-column block, 16-row chunks, deflation chain beyond the block)."""
    from paper_2107_11650_b200 import synth
    v = synth.sweep_vectors(n, nc, k, 3)
    tau = synth.sweep_tau(n, nc, k)
    p = n - k + 1
    adj, _ = gpu.hankel_svt_batched(v, p, tau, want_sv=False)
    adj_o, _ = O.hankel_svt_unit(v, p, tau)
    assert rel(adj, adj_o) < TOL


@pytest.mark.parametrize("r", [40, 120])
def test_huge_d_deflation_chain(gpu, r):
    """498 x 480 lifts with ~40 / ~120 singular values above the threshold:
    beyond the HUGE 32-column block, so level 1 and every chain step keep 24
    Ritz pairs and the next step solves the orthogonal remainder."""
    n, nc, k = 512, 32, 15
    p = n - k + 1
    v = _rank_r_vectors(n, nc, r, 2, 300 + r)
    tau = float(np.sqrt(p) + np.sqrt(nc * k))
    adj, _ = gpu.hankel_svt_batched(v, p, tau, want_sv=False)
    adj_o, sv_o = O.hankel_svt_unit(v, p, tau)
    assert (sv_o > tau).sum(axis=1).min() > 30
    assert rel(adj, adj_o) < TOL


def test_beyond_huge_fails_loudly(gpu):
    """min(m, n) > 496 is outside this build: SHLR_EUNSUPPORTED, never a
    silent fallback (BASELINE's sweep stops at 482)."""
    rng = np.random.default_rng(1)
    v = rng.standard_normal((1, 2, 1100)) + 1j * rng.standard_normal((1, 2, 1100))
    with pytest.raises(NotImplementedError):
        gpu.hankel_svt_batched(v, 550, 10.0, want_sv=False)


def test_exact_singular_values_need_full_solver(gpu):
    """The exact singular-value output needs the full eigen-solver (d <= 128)."""
    from paper_2107_11650_b200 import synth
    v = synth.sweep_vectors(256, 32, 15, 2)
    with pytest.raises(NotImplementedError):
        gpu.hankel_svt_batched(v, 242, 10.0)


def _rank_r_vectors(n, nc, r, batch, seed):
    """nc vectors of length n: r complex exponentials (amplitude ~4) + CN(0,1)."""
    rng = np.random.default_rng(seed)
    t = np.arange(n)
    v = (rng.standard_normal((batch, nc, n)) + 1j * rng.standard_normal((batch, nc, n))) / np.sqrt(2)
    w = rng.uniform(0, 2 * np.pi, size=(batch, 1, r, 1))
    a = 4 * (rng.standard_normal((batch, nc, r, 1)) + 1j * rng.standard_normal((batch, nc, r, 1)))
    return v + np.sum(a * np.exp(1j * w * t), axis=2)


@pytest.mark.parametrize("r", [10, 30, 45])
def test_subspace_levels(gpu, r):
    """242 x 120 lifts with r signal components: r = 10 stays at level 1 (32
    columns), r = 30 is handed to level 2 (48 columns), r = 45 overflows level
    2 and is redone by the full solver -- every route matches the oracle."""
    n, nc, k = 256, 8, 15
    p = n - k + 1
    v = _rank_r_vectors(n, nc, r, 6, 100 + r)
    tau = float(np.sqrt(p) + np.sqrt(nc * k))
    adj, _ = gpu.hankel_svt_batched(v, p, tau, want_sv=False)
    adj_o, sv_o = O.hankel_svt_unit(v, p, tau)
    assert rel(adj, adj_o) < TOL
    above = (sv_o > tau).sum(axis=1)
    assert above.min() >= min(r, 40) - 2  # the route the case is meant to take


def test_empty_batch_and_degenerate_pencils(gpu):
    """Empty batch; pencil = N (one column per coil block) and pencil = 1
    (one row), against the oracle."""
    v = np.zeros((0, 3, 20), np.complex128)
    out, sv = gpu.hankel_svt_batched(v, 5, 1.0)
    assert out.shape == (0, 3, 20) and sv.shape[0] == 0
    rng = np.random.default_rng(3)
    v = rng.standard_normal((3, 2, 9)) + 1j * rng.standard_normal((3, 2, 9))
    for p in (9, 1):
        adj, s = gpu.hankel_svt_batched(v, p, 0.5)
        adj_o, s_o = O.hankel_svt_unit(v, p, 0.5)
        assert rel(adj, adj_o) < TOL and rel(s, s_o) < TOL
