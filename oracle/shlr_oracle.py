"""CPU restatement (numpy, FP64) of the reference SHLR hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker or the timed CPU baseline -- never as the
thing measured or shipped.  The product path (``paper_2107_11650_b200``) does
not import it and fails loudly when its CUDA library is missing.

Every function restates the reference algorithm and cites the file:line it
follows (paths relative to ``/root/reference/proj``).  The restatement is
*pinned* twice:
  * against the reference's own known-answer tests (``tests/test_hankel.cpp``,
    ``tests/test_fft.cpp``, ``tests/test_sampling.cpp``, ``tests/test_solvers.cpp``),
    restated in ``tests/test_oracle_pins.py``;
  * against the reference itself, compiled unmodified into ``oracle/_ref`` (see
    ``oracle/Makefile``), through golden vectors it produced on seeded inputs
    (``tests/golden/*.npz``, checked in ``tests/test_golden.py``).

Arrays are complex128 numpy arrays with the reference's layouts: an M x N x J
tensor is ``x[m, n, j]`` (row-major, coil fastest; ``tensor.hpp:16-119``).
Lifted matrices are returned batched as ``(batch, p, blocks*q)``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

# --------------------------------------------------------------------------- rng
_M64 = (1 << 64) - 1


class SeededRng:
    """splitmix64 (``include/shlr/sampling.hpp:11-29``)."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * (2.0 ** -53)


# ------------------------------------------------------------------------ masks
@dataclass
class SamplingMask:
    """``include/shlr/sampling.hpp:33-52``: rows == 1 means a line mask that is
    broadcast along dim 0 when applied."""

    rows: int
    cols: int
    bits: np.ndarray  # uint8 (rows, cols)
    generator: str = ""
    seed: int = 0
    rate: float = 0.0
    acs: int = 0

    def sampled(self) -> np.ndarray:
        return self.bits.astype(bool)


def acs_range(n: int, acs: int) -> Tuple[int, int]:
    """``src/sampling.cpp:31-41``."""
    if acs == 0:
        return 0, 0
    if acs > n:
        raise ValueError("acs_range: acs exceeds grid size")
    c = n // 2
    half_up = (acs + 1) // 2
    if half_up > c:
        raise ValueError("acs_range: acs block does not fit")
    return c - half_up, c - half_up + acs


def _draw_weighted(bits: np.ndarray, candidates: List[int], weight: List[float],
                   want: int, rng: SeededRng) -> None:
    """Exact-count weighted sampling without replacement
    (``src/sampling.cpp:64-88``); sequential sums keep it bit-exact."""
    pool = list(candidates)
    w = [weight[i] for i in pool]
    for _ in range(want):
        total = 0.0
        for x in w:
            total += x
        u = rng.next_double() * total
        pick = len(pool) - 1
        acc = 0.0
        for i, x in enumerate(w):
            acc += x
            if u < acc:
                pick = i
                break
        bits[pool[pick]] = 1
        del pool[pick]
        del w[pick]


def mask_uniform(n: int, r: int, acs: int) -> SamplingMask:
    """``src/sampling.cpp:43-58``."""
    a0, a1 = acs_range(n, acs)
    bits = np.zeros(n, np.uint8)
    bits[::r] = 1
    bits[a0:a1] = 1
    if r == 1:
        bits[:] = 1
    return SamplingMask(1, n, bits.reshape(1, n), "uniform", 0, float(bits.sum()) / n, acs)


def mask_gauss_cartesian(n: int, rate: float, acs: int, seed: int) -> SamplingMask:
    """``src/sampling.cpp:92-128``."""
    if n == 0 or rate <= 0.0 or rate > 1.0:
        raise ValueError("mask_gauss_cartesian: invalid rate")
    want = int(math.ceil(rate * float(n)))
    if want < acs:
        raise ValueError("mask_gauss_cartesian: rate too small to fit the ACS block")
    a0, a1 = acs_range(n, acs)
    bits = np.zeros(n, np.uint8)
    bits[a0:a1] = 1
    sigma = float(n) / 6.0
    c = float(n // 2)
    weight = []
    for i in range(n):
        d = float(i) - c
        weight.append(math.exp(-d * d / (2.0 * sigma * sigma)))
    candidates = [i for i in range(n) if not bits[i]]
    _draw_weighted(bits, candidates, weight, want - (a1 - a0), SeededRng(seed))
    return SamplingMask(1, n, bits.reshape(1, n), "gauss_cartesian", seed, rate, acs)


def mask_random2d(rows: int, cols: int, rate: float, center: int, seed: int) -> SamplingMask:
    """``src/sampling.cpp:130-173``."""
    total = rows * cols
    want = int(math.ceil(rate * float(total)))
    r0, r1 = acs_range(rows, center)
    c0, c1 = acs_range(cols, center)
    block = (r1 - r0) * (c1 - c0)
    if block > want:
        raise ValueError("mask_random2d: center block exceeds budget")
    bits = np.zeros(total, np.uint8)
    for r in range(r0, r1):
        bits[r * cols + c0:r * cols + c1] = 1
    sigma = float(min(rows, cols)) / 6.0
    cr, cc = float(rows // 2), float(cols // 2)
    weight = []
    for r in range(rows):
        for c in range(cols):
            dr, dc = float(r) - cr, float(c) - cc
            weight.append(math.exp(-(dr * dr + dc * dc) / (2.0 * sigma * sigma)))
    candidates = [i for i in range(total) if not bits[i]]
    _draw_weighted(bits, candidates, weight, want - block, SeededRng(seed))
    return SamplingMask(rows, cols, bits.reshape(rows, cols), "random2d", seed, rate, center)


# -------------------------------------------------------------------------- fft
def fftshift(v: np.ndarray, axis: int = -1) -> np.ndarray:
    """``src/fft.cpp:75-81``: out[(i + c) % n] = v[i], c = floor(n/2)."""
    return np.fft.fftshift(v, axes=axis)


def ifftshift(v: np.ndarray, axis: int = -1) -> np.ndarray:
    """``src/fft.cpp:83-89``: out[i] = v[(i + c) % n]."""
    return np.fft.ifftshift(v, axes=axis)


def fft1d_centered(v: np.ndarray, axis: int = -1, inverse: bool = False) -> np.ndarray:
    """Unitary centered DFT, DC at floor(N/2) (``src/fft.cpp:91-106``); the
    reference's radix-2/Bluestein kernels (``:13-71``) compute the same DFT."""
    w = ifftshift(v, axis)
    w = np.fft.ifft(w, axis=axis, norm="ortho") if inverse else np.fft.fft(w, axis=axis, norm="ortho")
    return fftshift(w, axis)


def fft_along_axis(x: np.ndarray, axis: int, inverse: bool) -> np.ndarray:
    """``src/fft.cpp:108-128``."""
    return fft1d_centered(x, axis=axis, inverse=inverse)


def fft2d_centered(x: np.ndarray) -> np.ndarray:
    """``src/fft.cpp:130-134`` (axis 0 then axis 1, per coil)."""
    return fft_along_axis(fft_along_axis(x, 0, False), 1, False)


def ifft2d_centered(x: np.ndarray) -> np.ndarray:
    """``src/fft.cpp:136-140``."""
    return fft_along_axis(fft_along_axis(x, 0, True), 1, True)


# ----------------------------------------------------------------------- hankel
@dataclass
class HankelConfig:
    """``include/shlr/hankel.hpp:15-25``."""

    pencil: int = 0
    pencil_param: int = 0
    filter_taps: Sequence[complex] = (1.0 + 0j, -1.0 + 0j)
    virtual_coil: bool = False

    def pencil_for(self, length: int) -> int:
        """``src/hankel.cpp:10-18``."""
        if self.pencil != 0:
            if self.pencil > length:
                raise ValueError("HankelConfig: pencil exceeds signal length")
            return self.pencil
        if length >= 64:
            return 23
        return length // 3 + (1 if length % 3 else 0) + 1

    def pencil_for_param(self, length: int) -> int:
        """``src/hankel.cpp:20-29``."""
        if self.pencil_param != 0:
            if self.pencil_param > length:
                raise ValueError("HankelConfig: parameter pencil exceeds signal length")
            return self.pencil_param
        if length >= 64:
            return 23
        return length // 3 + (1 if length % 3 else 0) + 1


def hankel_lift(v: np.ndarray, p: int) -> np.ndarray:
    """``src/hankel.cpp:31-41``: out[i, j] = v[i + j], batched on leading dims."""
    n = v.shape[-1]
    idx = np.arange(p)[:, None] + np.arange(n - p + 1)[None, :]
    return v[..., idx]


def hankel_adjoint(m: np.ndarray, n: int) -> np.ndarray:
    """``src/hankel.cpp:43-54``: anti-diagonal sums, batched."""
    p, q = m.shape[-2], m.shape[-1]
    if p + q != n + 1:
        raise ValueError("hankel_adjoint: dims inconsistent with n")
    out = np.zeros(m.shape[:-2] + (n,), dtype=np.result_type(m.dtype, np.complex128))
    for i in range(p):
        out[..., i:i + q] += m[..., i, :]
    return out


def hankel_counts(n: int, p: int) -> np.ndarray:
    """``src/hankel.cpp:56-62``."""
    q = n - p + 1
    counts = np.zeros(n)
    for i in range(p):
        counts[i:i + q] += 1.0
    return counts


def hankel_dims(m: int, n: int, j: int, p: int, vc: bool) -> Tuple[int, int, int, int]:
    """``src/hankel.cpp:64-73``."""
    c = 2 if vc else 1
    return p, c * j * (n - p + 1), p * p * j, (m - p + 1) * (n - p + 1)


def weights_from_filter(taps: Sequence[complex], n: int) -> np.ndarray:
    """``src/hankel.cpp:75-92``: direct DFT of the zero-padded taps."""
    k = np.arange(n, dtype=np.float64)
    w = np.zeros(n, np.complex128)
    for t, tap in enumerate(taps):
        ang = -2.0 * np.pi * k * float(t) / float(n)
        w += complex(tap) * (np.cos(ang) + 1j * np.sin(ang))
    return w


def weights_centered(taps: Sequence[complex], n: int) -> np.ndarray:
    """``src/hankel.cpp:94-97``."""
    return fftshift(weights_from_filter(taps, n))


def dagger_index(n: int) -> np.ndarray:
    """Index map of ``virtual_coil_dagger`` (``src/hankel.cpp:99-113``):
    out[i] = conj(v[(2 floor(n/2) + n - i) mod n])."""
    c2 = 2 * (n // 2)
    return (c2 + n - np.arange(n)) % n


def virtual_coil_dagger(v: np.ndarray) -> np.ndarray:
    """``src/hankel.cpp:99-113``, along the last axis."""
    return np.conj(v[..., dagger_index(v.shape[-1])])


# -------------------------------------------------------------------- operators
def lift_weighted(vecs: np.ndarray, cfg: HankelConfig) -> np.ndarray:
    """``src/operators.cpp:25-58``.  vecs: (batch, J, n) coil vectors.
    Returns (batch, p, blocks*q): regular blocks first, then vc blocks."""
    n = vecs.shape[-1]
    p = cfg.pencil_for(n)
    q = n - p + 1
    wc = weights_centered(cfg.filter_taps, n)
    s = fft1d_centered(vecs, axis=-1)
    blocks = [wc * s]
    if cfg.virtual_coil:
        blocks.append(wc * virtual_coil_dagger(s))
    wb = np.concatenate(blocks, axis=-2)            # (batch, blocks, n)
    lifted = hankel_lift(wb, p)                     # (batch, blocks, p, q)
    b = lifted.shape[-3]
    return np.moveaxis(lifted, -3, -2).reshape(lifted.shape[:-3] + (p, b * q))


def adjoint_lift_weighted(m: np.ndarray, length: int, coils: int, cfg: HankelConfig) -> np.ndarray:
    """``src/operators.cpp:60-91`` (real adjoint).  m: (batch, p, blocks*q).
    Returns (batch, coils, length)."""
    p = cfg.pencil_for(length)
    q = length - p + 1
    blocks = coils * (2 if cfg.virtual_coil else 1)
    if m.shape[-2] != p or m.shape[-1] != blocks * q:
        raise ValueError("adjoint_lift_weighted: matrix dims mismatch")
    wc = weights_centered(cfg.filter_taps, length)
    mb = np.moveaxis(m.reshape(m.shape[:-1] + (blocks, q)), -2, -3)  # (batch, blocks, p, q)
    v = hankel_adjoint(mb, length)                                    # (batch, blocks, len)
    s_adj = np.conj(wc) * v[..., :coils, :]
    if cfg.virtual_coil:
        s_adj = s_adj + virtual_coil_dagger(np.conj(wc) * v[..., coils:, :])
    return fft1d_centered(s_adj, axis=-1, inverse=True)


def lift_plain(vecs: np.ndarray, p: int) -> np.ndarray:
    """``src/operators.cpp:93-103``.  vecs: (batch, J, n)."""
    n = vecs.shape[-1]
    q = n - p + 1
    lifted = hankel_lift(vecs, p)                    # (batch, J, p, q)
    j = lifted.shape[-3]
    return np.moveaxis(lifted, -3, -2).reshape(lifted.shape[:-3] + (p, j * q))


def adjoint_lift_plain(m: np.ndarray, length: int, coils: int) -> np.ndarray:
    """``src/operators.cpp:105-119``."""
    p = m.shape[-2]
    q = length - p + 1
    if m.shape[-1] != coils * q:
        raise ValueError("adjoint_lift_plain: matrix dims mismatch")
    mb = np.moveaxis(m.reshape(m.shape[:-1] + (coils, q)), -2, -3)
    return hankel_adjoint(mb, length)


def rows_of(x: np.ndarray) -> np.ndarray:
    """``extract_rows`` for every row (``src/operators.cpp:121-130``):
    (M, N, J) -> (M, J, N)."""
    return np.transpose(x, (0, 2, 1))


def cols_of(x: np.ndarray) -> np.ndarray:
    """``extract_cols`` for every column (``src/operators.cpp:132-141``):
    (M, N, J) -> (N, J, M)."""
    return np.transpose(x, (1, 2, 0))


def lift_rows_all(x: np.ndarray, cfg: HankelConfig) -> np.ndarray:
    """``lift_rows`` (``src/operators.cpp:143-146``) for all rows."""
    return lift_weighted(rows_of(x), cfg)


def lift_cols_all(x: np.ndarray, cfg: HankelConfig) -> np.ndarray:
    """``lift_cols`` (``src/operators.cpp:148-151``) for all columns."""
    return lift_weighted(cols_of(x), cfg)


def adjoint_lift_rows_all(mats: np.ndarray, dims: Tuple[int, int, int], cfg: HankelConfig) -> np.ndarray:
    """Sum over r of ``adjoint_lift_rows`` (``src/operators.cpp:153-161``)."""
    m, n, j = dims
    v = adjoint_lift_weighted(mats, n, j, cfg)       # (M, J, N)
    return np.transpose(v, (0, 2, 1))


def adjoint_lift_cols_all(mats: np.ndarray, dims: Tuple[int, int, int], cfg: HankelConfig) -> np.ndarray:
    """Sum over c of ``adjoint_lift_cols`` (``src/operators.cpp:163-171``)."""
    m, n, j = dims
    v = adjoint_lift_weighted(mats, m, j, cfg)       # (N, J, M)
    return np.transpose(v, (2, 0, 1))


def lift_weighted_normal(vecs: np.ndarray, cfg: HankelConfig) -> np.ndarray:
    """``src/operators.cpp:173-197``: L^H L on (batch, J, n) without the lift."""
    n = vecs.shape[-1]
    p = cfg.pencil_for(n)
    wc = weights_centered(cfg.filter_taps, n)
    counts = hankel_counts(n, p)
    g = np.conj(wc) * counts * wc
    s = fft1d_centered(vecs, axis=-1)
    acc = g * s
    if cfg.virtual_coil:
        acc = acc + virtual_coil_dagger(g * virtual_coil_dagger(s))
    return fft1d_centered(acc, axis=-1, inverse=True)


def apply_mask(k: np.ndarray, mask: SamplingMask) -> np.ndarray:
    """``src/operators.cpp:199-211`` (line masks broadcast over dim 0)."""
    m, n, _ = k.shape
    if mask.cols != n or (mask.rows != 1 and mask.rows != m):
        raise ValueError("apply_mask: mask dims mismatch")
    s = mask.sampled()
    s = np.broadcast_to(s, (m, n)) if mask.rows == 1 else s
    return np.where(s[:, :, None], k, 0)


def normal_apply(x: np.ndarray, mask: SamplingMask, g: Optional["SpiritImageOp"],
                 cfg: HankelConfig, lam: float, lam1: float, beta: float) -> np.ndarray:
    """``src/operators.cpp:213-248``."""
    out = np.zeros_like(x)
    if lam != 0.0:
        out = out + lam * ifft2d_centered(apply_mask(fft2d_centered(x), mask))
    if beta != 0.0:
        out = out + beta * np.transpose(lift_weighted_normal(rows_of(x), cfg), (0, 2, 1))
        out = out + beta * np.transpose(lift_weighted_normal(cols_of(x), cfg), (2, 0, 1))
    if lam1 != 0.0:
        if g is None:
            raise ValueError("normal_apply: lambda1 > 0 needs kernels")
        out = out + lam1 * g.normal_minus_identity(x)
    return out


# ----------------------------------------------------------------------- spirit
@dataclass
class SpiritKernels:
    """``include/shlr/spirit.hpp:12-36``.  weights has the reference's flat
    index ((di+h)*k + (dj+h))*J + src)*J + dst, stored as (k, k, J, J)."""

    kernel_size: int
    coils: int
    weights: np.ndarray  # complex (k, k, J, J)

    def weight(self, di: int, dj: int, src: int, dst: int) -> complex:
        h = self.kernel_size // 2
        return complex(self.weights[di + h, dj + h, src, dst])


def spirit_calibrate(acs: np.ndarray, kernel_size: int = 5, tikhonov: float = 1e-4) -> SpiritKernels:
    """``src/spirit.cpp:22-94``: Tikhonov-filtered SVD least squares per target
    coil with the self centre tap dropped."""
    a, b, j = acs.shape
    k = kernel_size
    if k % 2 == 0 or k == 0:
        raise ValueError("spirit_calibrate: kernel size must be odd")
    h = k // 2
    nr = (a - k + 1) * (b - k + 1)
    nf = k * k * j
    feat = np.zeros((nr, nf), np.complex128)
    centers = np.zeros((nr, j), np.complex128)
    row = 0
    for r in range(h, a - h):
        for c in range(h, b - h):
            patch = acs[r - h:r + h + 1, c - h:c + h + 1, :]   # (k, k, J) in (di, dj, s) order
            feat[row] = patch.reshape(-1)
            centers[row] = acs[r, c, :]
            row += 1
    weights = np.zeros((k * k * j * j,), np.complex128)
    center_block = (h * k + h) * j
    for dst in range(j):
        colmap = [c for c in range(nf) if c != center_block + dst]
        ad = feat[:, colmap]
        u, s, vh = np.linalg.svd(ad, full_matrices=False)
        mu = tikhonov * s[0]
        rhs = (u.conj().T @ centers[:, dst]) * (s / (s * s + mu * mu))
        w = vh.conj().T @ rhs
        for ci, full in enumerate(colmap):
            tap, src = divmod(full, j)
            weights[(tap * j + src) * j + dst] = w[ci]
    return SpiritKernels(k, j, weights.reshape(k, k, j, j))


class SpiritImageOp:
    """``src/spirit.cpp:104-165``: per-pixel J x J image-domain operator."""

    def __init__(self, g: SpiritKernels, m: int, n: int):
        self.m, self.n, self.j = m, n, g.coils
        k1 = fft2d_centered(np.ones((m, n, 1), np.complex128))[:, :, 0]
        h = g.kernel_size // 2
        maps = np.zeros((m, n, self.j, self.j), np.complex128)   # [r, c, src, dst]
        for di in range(-h, h + 1):
            for dj in range(-h, h + 1):
                # conv[r, c] += w * k1[(r + di) % m, (c + dj) % n]
                shifted = np.roll(np.roll(k1, -di, axis=0), -dj, axis=1)
                maps += shifted[:, :, None, None] * g.weights[di + h, dj + h][None, None, :, :]
        # maps = ifft2c(conv) per (src, dst) plane
        self.maps = ifft2d_centered(maps.reshape(m, n, self.j * self.j)).reshape(m, n, self.j, self.j)

    def apply(self, x: np.ndarray) -> np.ndarray:
        """``src/spirit.cpp:137-149``: out[dst] += map[src, dst] * x[src]."""
        return np.einsum("rcsd,rcs->rcd", self.maps, x)

    def normal_minus_identity(self, x: np.ndarray) -> np.ndarray:
        """``src/spirit.cpp:151-165``: (G - I)^H (G - I) x."""
        y = self.apply(x) - x
        return np.einsum("rcsd,rcd->rcs", np.conj(self.maps), y) - y


# ---------------------------------------------------------------------- solvers
@dataclass
class AdmmConfig:
    """``include/shlr/solvers.hpp:16-34``."""

    lam: float = 1e4
    lam1: float = 1e2
    lam2: float = 2.0
    beta: float = 1.0
    tau: float = 1.0
    max_outer: int = 50
    tol: float = 1e-6
    cg_max: int = 15
    cg_tol: float = 1e-8
    enable_spirit: bool = False
    enable_vc: bool = False

    def validate(self) -> None:
        if (self.lam <= 0 or self.lam1 < 0 or self.lam2 < 0 or self.beta <= 0 or self.tau <= 0
                or self.tol <= 0 or self.cg_tol <= 0):
            raise ValueError("AdmmConfig: invalid parameter")


class DivergenceError(RuntimeError):
    """``include/shlr/solvers.hpp:41-43``."""


@dataclass
class SolveStats:
    outer_iters: int = 0
    final_rel_change: float = 0.0
    log: List[str] = field(default_factory=list)
    singular_values: dict = field(default_factory=dict)
    images: dict = field(default_factory=dict)


def svt(m: np.ndarray, tau: float, return_sv: bool = False):
    """``src/solvers.cpp:11-21``: U max(S - tau, 0) V^H, batched."""
    if tau < 0:
        raise ValueError("svt: negative threshold")
    u, s, vh = np.linalg.svd(m, full_matrices=False)
    z = (u * np.maximum(s - tau, 0.0)[..., None, :]) @ vh
    if tau == 0.0:
        z = m.copy()
    return (z, s) if return_sv else z


def rdot(a: np.ndarray, b: np.ndarray) -> float:
    """``include/shlr/tensor.hpp:158-160``."""
    return float(np.vdot(b.ravel(), a.ravel()).real)


def norm2(a: np.ndarray) -> float:
    """``include/shlr/tensor.hpp:162-166``."""
    return float(np.sqrt(np.sum(np.abs(a) ** 2)))


def cg_solve(apply_a, b: np.ndarray, x0: np.ndarray, max_iter: int, tol: float):
    """``src/solvers.cpp:23-67`` (warm start, real pairing, cap, quirks)."""
    x = x0.copy()
    r = b - apply_a(x)
    bnorm = norm2(b)
    if bnorm == 0.0:
        return np.zeros_like(b), 0, 0.0
    rel = norm2(r) / bnorm
    if not np.isfinite(rel):
        raise DivergenceError("cg_solve: non-finite residual")
    it = 0
    if rel > tol:
        p = r.copy()
        rho = rdot(r, r)
        while it < max_iter:
            ap = apply_a(p)
            denom = rdot(p, ap)
            if not np.isfinite(denom) or denom <= 0.0:
                raise DivergenceError("cg_solve: operator not positive definite")
            alpha = rho / denom
            x = x + alpha * p
            r = r - alpha * ap
            rho_next = rdot(r, r)
            if not np.isfinite(rho_next):
                raise DivergenceError("cg_solve: non-finite residual")
            rel = math.sqrt(rho_next) / bnorm
            if rel <= tol:
                it += 1
                break
            p = r + (rho_next / rho) * p
            rho = rho_next
            it += 1
    return x, it, rel


def rel_change_sq(x_new: np.ndarray, x_old: np.ndarray) -> float:
    """``src/solvers.cpp:80-87``."""
    num = float(np.sum(np.abs(x_new - x_old) ** 2))
    den = float(np.sum(np.abs(x_old) ** 2))
    return num / den if den > 0.0 else (1.0 if num > 0.0 else 0.0)


def log_line(it: int, relchange: float, cg_iters: int, cg_res: float) -> str:
    """``src/solvers.cpp:71-78`` (std::scientific, precision 3)."""
    return f"iter={it} relchange={relchange:.3e} cg_iters={cg_iters} cg_res={cg_res:.3e}"


def shlr_pi_reconstruct(y: np.ndarray, mask: SamplingMask, g: Optional[SpiritKernels],
                        hcfg: HankelConfig, acfg: AdmmConfig,
                        sv_iters: Sequence[int] = (), x_iters: Sequence[int] = ()) -> Tuple[np.ndarray, SolveStats]:
    """``src/solvers.cpp:95-191`` (Algorithm S1).  sv_iters: 1-based outer
    iterations whose singular values of L + D/beta are recorded (rows first,
    then columns); x_iters: iterations whose image x is recorded
    (stats.images).  Neither changes the arithmetic."""
    acfg.validate()
    if y.ndim != 3:
        raise ValueError("shlr_pi_reconstruct: expected M x N x J")
    if acfg.enable_spirit and g is None:
        raise ValueError("shlr_pi_reconstruct: spirit enabled without kernels")
    m, n, j = y.shape
    if mask.cols != n or (mask.rows != 1 and mask.rows != m):
        raise ValueError("shlr_pi_reconstruct: mask dims mismatch")
    cfg = HankelConfig(hcfg.pencil, hcfg.pencil_param, tuple(hcfg.filter_taps), acfg.enable_vc)
    p_row, p_col = cfg.pencil_for(n), cfg.pencil_for(m)
    blocks = j * (2 if acfg.enable_vc else 1)
    lam1 = acfg.lam1 if acfg.enable_spirit else 0.0
    gop = None
    if acfg.enable_spirit and lam1 > 0.0:
        if g.coils != j:
            raise ValueError("shlr_pi_reconstruct: kernel coil mismatch")
        gop = SpiritImageOp(g, m, n)
    y_masked = apply_mask(y, mask)
    fid_rhs = ifft2d_centered(y_masked)
    z_row = np.zeros((m, p_row, blocks * (n - p_row + 1)), np.complex128)
    d_row = np.ones_like(z_row)
    z_col = np.zeros((n, p_col, blocks * (m - p_col + 1)), np.complex128)
    d_col = np.ones_like(z_col)
    x = fid_rhs.copy()
    beta = acfg.beta
    stats = SolveStats()

    def apply_a(v):
        return normal_apply(v, mask, gop, cfg, acfg.lam, lam1, beta)

    relchange = 1.0
    for k in range(acfg.max_outer):
        b = acfg.lam * fid_rhs
        b = b + beta * adjoint_lift_rows_all(z_row - d_row / beta, (m, n, j), cfg)
        b = b + beta * adjoint_lift_cols_all(z_col - d_col / beta, (m, n, j), cfg)
        x_new, cg_it, cg_res = cg_solve(apply_a, b, x, acfg.cg_max, acfg.cg_tol)
        lr = lift_rows_all(x_new, cfg)
        z_row, s_r = svt(lr + d_row / beta, 1.0 / beta, return_sv=True)
        d_row = d_row + acfg.tau * (lr - z_row)
        lc = lift_cols_all(x_new, cfg)
        z_col, s_c = svt(lc + d_col / beta, 1.0 / beta, return_sv=True)
        d_col = d_col + acfg.tau * (lc - z_col)
        if (k + 1) in sv_iters:
            stats.singular_values[k + 1] = (s_r, s_c)
        if (k + 1) in x_iters:
            stats.images[k + 1] = x_new.copy()
        relchange = rel_change_sq(x_new, x)
        x = x_new
        stats.outer_iters = k + 1
        stats.log.append(log_line(k + 1, relchange, cg_it, cg_res))
        if relchange < acfg.tol:
            break
    stats.final_rel_change = relchange
    return x, stats


def shlr_param_reconstruct_slice(y_m: np.ndarray, mask: SamplingMask, hcfg: HankelConfig,
                                 acfg: AdmmConfig) -> Tuple[np.ndarray, SolveStats]:
    """``src/solvers.cpp:193-298`` (Algorithm S2) on one N x L x J plane."""
    acfg.validate()
    n, l, j = y_m.shape
    if mask.rows != n or mask.cols != l:
        raise ValueError("shlr_param_reconstruct_slice: mask dims mismatch")
    cfg = HankelConfig(hcfg.pencil, hcfg.pencil_param, tuple(hcfg.filter_taps), acfg.enable_vc)
    p_pe, p_par = cfg.pencil_for(n), cfg.pencil_for_param(l)
    blocks_pe = j * (2 if acfg.enable_vc else 1)
    counts_par = hankel_counts(l, p_par)
    sel = mask.sampled()
    y_masked = np.where(sel[:, :, None], y_m, 0)
    fid_rhs = fft_along_axis(y_masked, 0, True)
    z_pe = np.zeros((n, p_par, j * (l - p_par + 1)), np.complex128)
    d_pe = np.ones_like(z_pe)
    z_p = np.zeros((l, p_pe, blocks_pe * (n - p_pe + 1)), np.complex128)
    d_p = np.ones_like(z_p)
    x = fid_rhs.copy()
    beta = acfg.beta

    def apply_a(v):
        out = acfg.lam * fft_along_axis(np.where(sel[:, :, None], fft_along_axis(v, 0, False), 0), 0, True)
        out = out + beta * counts_par[None, :, None] * v
        t = lift_weighted_normal(np.transpose(v, (1, 2, 0)), cfg)   # (L, J, N)
        return out + beta * np.transpose(t, (2, 0, 1))

    stats = SolveStats()
    relchange = 1.0
    for k in range(acfg.max_outer):
        b = acfg.lam * fid_rhs
        rows = adjoint_lift_plain(z_pe - d_pe / beta, l, j)          # (N, J, L)
        b = b + beta * np.transpose(rows, (0, 2, 1))
        adj = adjoint_lift_weighted(z_p - d_p / beta, n, j, cfg)      # (L, J, N)
        b = b + beta * np.transpose(adj, (2, 0, 1))
        x_new, cg_it, cg_res = cg_solve(apply_a, b, x, acfg.cg_max, acfg.cg_tol)
        lp = lift_plain(np.transpose(x_new, (0, 2, 1)), p_par)        # rows: (N, J, L)
        z_pe = svt(lp + d_pe / beta, acfg.lam2 / beta)
        d_pe = d_pe + acfg.tau * (lp - z_pe)
        lc = lift_weighted(np.transpose(x_new, (1, 2, 0)), cfg)       # cols: (L, J, N)
        z_p = svt(lc + d_p / beta, 1.0 / beta)
        d_p = d_p + acfg.tau * (lc - z_p)
        relchange = rel_change_sq(x_new, x)
        x = x_new
        stats.outer_iters = k + 1
        stats.log.append(log_line(k + 1, relchange, cg_it, cg_res))
        if relchange < acfg.tol:
            break
    stats.final_rel_change = relchange
    return x, stats


def recon_param_dataset(y: np.ndarray, mask: SamplingMask, hcfg: HankelConfig,
                        acfg: AdmmConfig) -> Tuple[np.ndarray, int]:
    """``src/parammap.cpp:21-54``: iFFT along FE, independent slice solves."""
    m, n, l, j = y.shape
    if mask.rows != n or mask.cols != l:
        raise ValueError("recon_param_dataset: mask dims mismatch")
    hybrid = fft_along_axis(y, 0, True)
    out = np.zeros_like(hybrid)
    total = 0
    for fe in range(m):
        rec, st = shlr_param_reconstruct_slice(hybrid[fe], mask, hcfg, acfg)
        out[fe] = rec
        total += st.outer_iters
    return out, total


def hankel_svt_unit(vecs: np.ndarray, p: int, tau: float):
    """Config-5 unit: ``lift_plain`` -> ``svt`` -> ``adjoint_lift_plain``
    (composition of ``src/operators.cpp:93-119`` and ``src/solvers.cpp:11-21``
    as used at ``src/solvers.cpp:264-268,280-282``).  vecs: (B, Nc, N).
    Returns (adjoint vectors (B, Nc, N), singular values (B, d))."""
    b, nc, n = vecs.shape
    lifted = lift_plain(vecs, p)
    z, s = svt(lifted, tau, return_sv=True)
    return adjoint_lift_plain(z, n, nc), s


# ---------------------------------------------------------------- metrics
def ssos(x: np.ndarray) -> np.ndarray:
    """``src/io.cpp:105-117``: sqrt(sum_k |x[r, c, k]|^2), k ascending."""
    x = np.asarray(x)
    if x.ndim != 3:
        raise ValueError("ssos: expected an M x N x J tensor")
    s = np.zeros(x.shape[:2])
    for k in range(x.shape[2]):
        s = s + (x[:, :, k].real * x[:, :, k].real + x[:, :, k].imag * x[:, :, k].imag)
    return np.sqrt(s)


def rlne(ref: np.ndarray, rec: np.ndarray) -> float:
    """``src/metrics.cpp:9-21``: ||ref - rec|| / ||ref||."""
    if ref.shape != rec.shape:
        raise ValueError("rlne: dimension mismatch")
    den = float(np.sum(ref * ref))
    if den == 0.0:
        raise ValueError("rlne: reference image is identically zero")
    return float(np.sqrt(np.sum((ref - rec) ** 2) / den))


def mssim(ref: np.ndarray, rec: np.ndarray) -> float:
    """``src/metrics.cpp:23-75``: mean SSIM over every 11 x 11 window, Gaussian
    weights sigma = 1.5 normalised to sum 1, C1 = (0.01 max ref)^2,
    C2 = (0.03 max ref)^2, variances / covariance about the window means."""
    if ref.shape != rec.shape:
        raise ValueError("mssim: dimension mismatch")
    k = 11
    if ref.shape[0] < k or ref.shape[1] < k:
        raise ValueError("mssim: image smaller than the 11x11 window")
    d = np.arange(k) - 5.0
    w = np.exp(-(d[:, None] ** 2 + d[None, :] ** 2) / (2.0 * 1.5 * 1.5))
    w = w / w.sum()
    mx = max(float(ref.max()), 0.0)
    c1, c2 = (0.01 * mx) ** 2, (0.03 * mx) ** 2
    from numpy.lib.stride_tricks import sliding_window_view
    a = sliding_window_view(ref, (k, k))
    b = sliding_window_view(rec, (k, k))
    mu_a = np.einsum("rcij,ij->rc", a, w)
    mu_b = np.einsum("rcij,ij->rc", b, w)
    da = a - mu_a[:, :, None, None]
    db = b - mu_b[:, :, None, None]
    var_a = np.einsum("rcij,ij->rc", da * da, w)
    var_b = np.einsum("rcij,ij->rc", db * db, w)
    cov = np.einsum("rcij,ij->rc", da * db, w)
    ssim = ((2 * mu_a * mu_b + c1) * (2 * cov + c2)) / ((mu_a ** 2 + mu_b ** 2 + c1) * (var_a + var_b + c2))
    return float(ssim.mean())
