"""Pins the numpy oracle (oracle/shlr_oracle.py) to the known-answer tests
the reference holds for this path.  Each case restates a
reference test; the file:line is given in the docstring."""
import math

import numpy as np
import pytest

import shlr_oracle as O


def test_hankel_lift_definition():
    """tests/test_hankel.cpp:13-24."""
    m = O.hankel_lift(np.array([1, 2, 3, 4], complex), 2)
    assert m.shape == (2, 3)
    assert np.array_equal(m, np.array([[1, 2, 3], [2, 3, 4]], complex))


def test_pencil_extremes():
    """tests/test_hankel.cpp:26-40."""
    v = np.arange(5) + 1j
    assert O.hankel_lift(v, 1).shape == (1, 5)
    assert O.hankel_lift(v, 5).shape == (5, 1)
    assert np.array_equal(O.hankel_lift(v, 5)[:, 0], v)


def test_hankel_adjoint_antidiagonal_sums():
    """tests/test_hankel.cpp:42-52."""
    v = O.hankel_adjoint(np.ones((2, 3), complex), 4)
    assert np.array_equal(v, np.array([1, 2, 2, 1], complex))
    with pytest.raises(ValueError):
        O.hankel_adjoint(np.ones((2, 3), complex), 5)


def test_lift_adjoint_inner_product_identity():
    """tests/test_hankel.cpp:54-68."""
    rng = np.random.default_rng(2)
    n, p = 11, 4
    v = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    m = rng.uniform(-1, 1, (p, n - p + 1)) + 1j * rng.uniform(-1, 1, (p, n - p + 1))
    lhs = np.sum(O.hankel_lift(v, p) * np.conj(m))
    rhs = np.sum(v * np.conj(O.hankel_adjoint(m, n)))
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)


def test_counts():
    """tests/test_hankel.cpp:70-92 (multiplicity and brute force)."""
    assert np.array_equal(O.hankel_counts(4, 2), [1, 2, 2, 1])
    for n in (6, 9):
        for p in range(1, n + 1):
            brute = np.zeros(n)
            for i in range(p):
                for j in range(n - p + 1):
                    brute[i + j] += 1
            assert np.array_equal(O.hankel_counts(n, p), brute)


def test_dims_published_block_size():
    """tests/test_hankel.cpp:94-108: 2116 x 54756 vs 23 x 936 / 23 x 1872."""
    assert O.hankel_dims(256, 256, 4, 23, False) == (23, 936, 2116, 54756)
    assert O.hankel_dims(256, 256, 4, 23, True) == (23, 1872, 2116, 54756)


def test_filter_weights_analytic():
    """tests/test_hankel.cpp:110-122: [1,-1] at N=4 -> [0, 1+i, 2, 1-i]."""
    w = O.weights_from_filter([1, -1], 4)
    assert np.allclose(w, [0, 1 + 1j, 2, 1 - 1j], atol=1e-14)
    assert np.allclose(O.weights_from_filter([1], 7), np.ones(7), atol=1e-14)


def test_centered_weights_shift():
    """tests/test_hankel.cpp:140-149."""
    rng = np.random.default_rng(12)
    taps = rng.uniform(-1, 1, 3) + 1j * rng.uniform(-1, 1, 3)
    nat = O.weights_from_filter(taps, 8)
    cen = O.weights_centered(taps, 8)
    assert cen[4] == nat[0]
    for k in range(8):
        assert cen[(k + 4) % 8] == nat[k]


def test_dagger():
    """tests/test_hankel.cpp:151-165: definition, involution, fixpoint."""
    d = O.virtual_coil_dagger(np.array([1 + 2j, 3, 4 - 1j]))
    assert np.array_equal(d, [4 + 1j, 3, 1 - 2j])
    r = np.random.default_rng(4).normal(size=9) + 1j
    assert np.array_equal(O.virtual_coil_dagger(O.virtual_coil_dagger(r)), r)
    sym = np.array([1, 2, 5, 2, 1], complex)
    assert np.array_equal(O.virtual_coil_dagger(sym), sym)


@pytest.mark.parametrize("n", [4, 5, 8, 9, 16])
def test_dagger_fixes_real_spectra(n):
    """tests/test_hankel.cpp:167-180."""
    x = np.random.default_rng(n).normal(size=n).astype(complex)
    s = O.fft1d_centered(x)
    assert np.allclose(O.virtual_coil_dagger(s), s, atol=1e-12)


def test_pencil_rule():
    """tests/test_hankel.cpp:182-190: 256 -> 23, 48 -> 17, 7 -> 4."""
    h = O.HankelConfig()
    assert (h.pencil_for(256), h.pencil_for(48), h.pencil_for(7)) == (23, 17, 4)


def test_fft_delta():
    """tests/test_fft.cpp:43-48."""
    v = np.zeros(4, complex)
    v[2] = 1
    assert np.allclose(O.fft1d_centered(v), 0.5, atol=1e-14)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 8, 15, 16, 31, 45])
def test_fft_analytic_matrix(n):
    """tests/test_fft.cpp:13-32,69-77: centred DFT F[k,m] = w^{(k-c)(m-c)}/sqrt(N)."""
    rng = np.random.default_rng(n)
    v = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    c = n // 2
    k = np.arange(n)
    for inv, sgn in ((False, -1.0), (True, 1.0)):
        f = np.exp(sgn * 2j * np.pi * np.outer(k - c, k - c) / n) / math.sqrt(n)
        assert np.max(np.abs(O.fft1d_centered(v, inverse=inv) - f @ v)) < 1e-11


def test_parseval_and_roundtrip():
    """tests/test_fft.cpp:50-67."""
    for n in (5, 8, 12, 17, 30):
        v = np.random.default_rng(100 + n).normal(size=n) + 1j
        assert abs(np.linalg.norm(v) - np.linalg.norm(O.fft1d_centered(v))) < 1e-12
        assert np.max(np.abs(O.fft1d_centered(O.fft1d_centered(v), inverse=True) - v)) < 1e-12


def test_splitmix64_golden():
    """tests/test_sampling.cpp:144-150."""
    r = O.SeededRng(0)
    assert [r.next_u64() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                0x06C45D188009454F]


def test_acs_range():
    """tests/test_sampling.cpp:23-32."""
    assert O.acs_range(12, 2) == (5, 7)
    assert O.acs_range(256, 20) == (118, 138)
    assert O.acs_range(9, 0)[1] == 0
    with pytest.raises(ValueError):
        O.acs_range(8, 9)


def test_mask_counts_and_acs():
    """tests/test_sampling.cpp:54-86: exact counts 88 and 738, ACS coverage,
    determinism, seed sensitivity."""
    a = O.mask_gauss_cartesian(256, 0.34, 22, 42)
    assert int(a.bits.sum()) == 88
    s, e = O.acs_range(256, 22)
    assert a.bits[0, s:e].all()
    assert np.array_equal(a.bits, O.mask_gauss_cartesian(256, 0.34, 22, 42).bits)
    assert not np.array_equal(a.bits, O.mask_gauss_cartesian(256, 0.34, 22, 43).bits)
    assert int(O.mask_gauss_cartesian(32, 1.0, 4, 1).bits.sum()) == 32
    with pytest.raises(ValueError):
        O.mask_gauss_cartesian(64, 0.05, 16, 1)
    b = O.mask_random2d(64, 64, 0.18, 12, 7)
    assert int(b.bits.sum()) == 738
    rs, re_ = O.acs_range(64, 12)
    assert b.bits[rs:re_, rs:re_].all()
    with pytest.raises(ValueError):
        O.mask_random2d(16, 16, 0.1, 10, 1)


def test_uniform_mask_example():
    """tests/test_sampling.cpp:34-37: lines {0, 4, 5, 6, 8}."""
    m = O.mask_uniform(12, 4, 2)
    assert set(np.flatnonzero(m.bits[0])) == {0, 4, 5, 6, 8}


def test_svt_zero_threshold_and_rank_one():
    """tests/test_solvers.cpp:42-56."""
    rng = np.random.default_rng(1)
    m = rng.uniform(-1, 1, (5, 7)) + 1j * rng.uniform(-1, 1, (5, 7))
    assert np.max(np.abs(O.svt(m, 0.0) - m)) < 1e-12
    u = np.array([0.6, 0.8j, 0])
    v = np.array([0.5, 0.5, 0.5, 0.5])
    mm = 5.0 * np.outer(u, np.conj(v))
    assert np.max(np.abs(O.svt(mm, 2.0) - 3.0 * np.outer(u, np.conj(v)))) < 1e-12
    assert np.max(np.abs(O.svt(mm, 6.0))) < 1e-12


def test_svt_nonexpansive_and_rank():
    """tests/test_solvers.cpp:72-93."""
    rng = np.random.default_rng(3)
    for _ in range(10):
        a = rng.uniform(-1, 1, (6, 5)) + 1j * rng.uniform(-1, 1, (6, 5))
        b = rng.uniform(-1, 1, (6, 5)) + 1j * rng.uniform(-1, 1, (6, 5))
        assert np.linalg.norm(O.svt(a, 0.5) - O.svt(b, 0.5)) <= np.linalg.norm(a - b) + 1e-12
        s = np.linalg.svd(a, compute_uv=False)
        s2 = np.linalg.svd(O.svt(a, 0.5), compute_uv=False)
        assert np.sum(s2 > 1e-10) == np.sum(s > 0.5)
        assert abs(np.sum(s2) - np.sum(np.maximum(s - 0.5, 0))) < 1e-10


def test_cg_known_answers():
    """tests/test_solvers.cpp:95-182: identity, diagonal, zero rhs, NaN."""
    ident = lambda t: t
    b = np.array([1, 2, 4], complex)
    x, it, _ = O.cg_solve(ident, b, np.zeros(3, complex), 10, 1e-12)
    assert it == 1 and np.max(np.abs(x - b)) < 1e-12
    diag = lambda t: t * np.array([1, 2, 4])
    x, _, _ = O.cg_solve(diag, b, np.zeros(3, complex), 10, 1e-12)
    assert np.max(np.abs(x - 1)) < 1e-10
    x, it, rel = O.cg_solve(diag, np.zeros(3, complex), np.ones(3, complex), 10, 1e-12)
    assert it == 0 and rel == 0.0 and not x.any()
    with pytest.raises(O.DivergenceError):
        O.cg_solve(lambda t: t * np.nan, b, np.zeros(3, complex), 5, 1e-10)


def test_normal_apply_is_adjoint_composition():
    """tests/test_operators.cpp:97,198-233: lift_weighted_normal = L^H L
    (real pairing with vc) and the normal operator is self-adjoint PSD."""
    rng = np.random.default_rng(5)
    for vc in (False, True):
        cfg = O.HankelConfig(pencil=4, virtual_coil=vc)
        vecs = rng.normal(size=(3, 2, 10)) + 1j * rng.normal(size=(3, 2, 10))
        lhs = O.lift_weighted_normal(vecs, cfg)
        rhs = O.adjoint_lift_weighted(O.lift_weighted(vecs, cfg), 10, 2, cfg)
        assert np.max(np.abs(lhs - rhs)) < 1e-12
        x = rng.normal(size=(6, 6, 2)) + 1j * rng.normal(size=(6, 6, 2))
        z = rng.normal(size=(6, 6, 2)) + 1j * rng.normal(size=(6, 6, 2))
        mk = O.mask_uniform(6, 2, 2)
        ax = O.normal_apply(x, mk, None, cfg, 3.0, 0.0, 1.5)
        az = O.normal_apply(z, mk, None, cfg, 3.0, 0.0, 1.5)
        assert abs(O.rdot(ax, z) - O.rdot(x, az)) < 1e-10 * abs(O.rdot(ax, z))
        assert O.rdot(ax, x) > 0
