"""Seeded synthetic inputs for the BASELINE.json workloads (harness only).

The reference's in-vivo datasets are absent and its own
``synth`` phantom (proj/src/synth.cpp:33-135) is not the BASELINE phantom, so
these generators follow BASELINE.json / SURVEY.md section 8(d):

* phantom: 10 axis-aligned ellipses, centres U[0.15, 0.85] FOV, semi-axes
  U[5, 40] px, magnitudes U[0.2, 1], later ellipses overwrite earlier ones
  (as paint_shapes, synth.cpp:87-96); smooth phase exp(i 2 pi p(x, y)) with p
  a full 2nd-order polynomial in normalised coordinates, 6 coefficients
  U[-0.5, 0.5];
* coils: J Gaussian sensitivities (sigma = 0.6 FOV) centred evenly on a circle
  of radius 0.7 FOV about the image centre, each with a U[0, 2 pi) constant
  phase (config 3: two staggered rings);
* k-space: centred unitary 2D FFT per coil (fft.cpp:130-134 convention) plus
  complex Gaussian noise of per-sample variance mean|k|^2 10^(-SNR/10),
  SNR = 40 dB;
* T2 (config 4): per-ellipse T2 ~ U[30, 150] ms, PD ~ U[0.3, 1], TE = 10 e ms.

Random streams are splitmix64 (the reference's SeededRng, sampling.hpp:11-29)
with the seeds of SURVEY.md 8(d): phantom 2107, coils 2108, noise 2109,
mask 11650 (+e), sweep 7 + slice.  Normal deviates use Box-Muller
(synth.cpp:123-132 style).  The generator is vectorised: the k-th draw of a
stream is splitmix64's output for state seed + (k+1) * 0x9e3779b97f4a7c15.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
SEED_PHANTOM, SEED_COILS, SEED_NOISE, SEED_MASK, SEED_SWEEP = 2107, 2108, 2109, 11650, 7


class Stream:
    """Vectorised splitmix64 stream."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed)
        self.count = 0

    def u64(self, n: int) -> np.ndarray:
        k = np.arange(self.count + 1, self.count + n + 1, dtype=np.uint64)
        self.count += n
        with np.errstate(over="ignore"):
            z = self.state + k * GOLDEN
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        return z

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        u = (self.u64(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return lo + (hi - lo) * u

    def normal(self, n: int) -> np.ndarray:
        m = (n + 1) // 2
        u1 = self.uniform(m)
        u2 = self.uniform(m)
        r = np.sqrt(-2.0 * np.log1p(-u1))
        z = np.concatenate([r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)])
        return z[:n]


def fft2c(x: np.ndarray) -> np.ndarray:
    """Centred unitary 2D FFT over axes (0, 1) (harness-side input generation)."""
    y = np.fft.ifftshift(x, axes=(0, 1))
    y = np.fft.fft2(y, axes=(0, 1), norm="ortho")
    return np.fft.fftshift(y, axes=(0, 1))


@dataclass
class Phantom:
    image: np.ndarray        # (M, N) complex magnitude * phase
    labels: np.ndarray       # (M, N) int: index of the ellipse that painted the pixel, -1 outside
    sens: np.ndarray         # (M, N, J) coil sensitivities
    truth: np.ndarray        # (M, N, J) coil images
    kspace: np.ndarray       # (M, N, J) noisy centred k-space


def ellipses(m: int, n: int, count: int, rng: Stream) -> Tuple[np.ndarray, np.ndarray]:
    cr = rng.uniform(count, 0.15, 0.85) * m
    cc = rng.uniform(count, 0.15, 0.85) * n
    ar = rng.uniform(count, 5.0, 40.0)
    ac = rng.uniform(count, 5.0, 40.0)
    mag = rng.uniform(count, 0.2, 1.0)
    rr, cc_ = np.meshgrid(np.arange(m, dtype=np.float64), np.arange(n, dtype=np.float64), indexing="ij")
    img = np.zeros((m, n))
    lab = -np.ones((m, n), np.int64)
    for e in range(count):
        inside = ((rr - cr[e]) / ar[e]) ** 2 + ((cc_ - cc[e]) / ac[e]) ** 2 <= 1.0
        img[inside] = mag[e]
        lab[inside] = e
    return img, lab


def smooth_phase(m: int, n: int, rng: Stream) -> np.ndarray:
    c = rng.uniform(6, -0.5, 0.5)
    y, x = np.meshgrid(np.linspace(-1, 1, m), np.linspace(-1, 1, n), indexing="ij")
    p = c[0] + c[1] * x + c[2] * y + c[3] * x * x + c[4] * x * y + c[5] * y * y
    return np.exp(1j * 2 * np.pi * p)


def coil_maps(m: int, n: int, j: int, rng: Stream, rings: int = 1) -> np.ndarray:
    fov = float(max(m, n))
    y, x = np.meshgrid(np.arange(m) - m / 2.0, np.arange(n) - n / 2.0, indexing="ij")
    sig = 0.6 * fov
    ph = rng.uniform(j, 0.0, 2 * np.pi)
    maps = np.zeros((m, n, j), np.complex128)
    per_ring = j // rings
    for q in range(j):
        ring = q // per_ring if rings > 1 else 0
        k = q % per_ring if rings > 1 else q
        stagger = (0.5 * ring) if rings > 1 else 0.0
        ang = 2 * np.pi * (k + stagger) / per_ring
        rad = 0.7 * fov * (1.0 if ring == 0 else 0.85)
        cy, cx = rad * np.sin(ang), rad * np.cos(ang)
        g = np.exp(-((y - cy) ** 2 + (x - cx) ** 2) / (2 * sig * sig))
        maps[:, :, q] = g * np.exp(1j * ph[q])
    return maps


def add_noise(k: np.ndarray, snr_db: float, rng: Stream) -> np.ndarray:
    var = float(np.mean(np.abs(k) ** 2)) * 10.0 ** (-snr_db / 10.0)
    z = rng.normal(2 * k.size).reshape(2, *k.shape)
    return k + np.sqrt(var / 2.0) * (z[0] + 1j * z[1])


def pi_phantom(m: int, n: int, j: int, rings: int = 1, snr_db: float = 40.0,
               seeds=(SEED_PHANTOM, SEED_COILS, SEED_NOISE)) -> Phantom:
    rng_p = Stream(seeds[0])
    mag, lab = ellipses(m, n, 10, rng_p)
    img = mag * smooth_phase(m, n, rng_p)
    sens = coil_maps(m, n, j, Stream(seeds[1]), rings)
    truth = img[:, :, None] * sens
    k = fft2c(truth)
    k = add_noise(k, snr_db, Stream(seeds[2]))
    return Phantom(img, lab, sens, truth, k)


def t2_phantom(m: int, n: int, j: int, echoes: int, snr_db: float = 40.0):
    """Config 4: returns (truth (M,N,L,J), kspace (M,N,L,J), tes_ms, t2 per ellipse)."""
    rng_p = Stream(SEED_PHANTOM)
    _, lab = ellipses(m, n, 10, rng_p)
    phase = smooth_phase(m, n, rng_p)
    t2 = rng_p.uniform(10, 30.0, 150.0)
    pd = rng_p.uniform(10, 0.3, 1.0)
    sens = coil_maps(m, n, j, Stream(SEED_COILS))
    tes = 10.0 * np.arange(1, echoes + 1)
    truth = np.zeros((m, n, echoes, j), np.complex128)
    for e, te in enumerate(tes):
        amp = np.where(lab >= 0, pd[np.maximum(lab, 0)] * np.exp(-te / t2[np.maximum(lab, 0)]), 0.0)
        truth[:, :, e, :] = (amp * phase)[:, :, None] * sens
    k = np.stack([fft2c(truth[:, :, e, :]) for e in range(echoes)], axis=2)
    k = add_noise(k, snr_db, Stream(SEED_NOISE))
    return truth, k, tes, t2


def sweep_vectors(n: int, nc: int, k: int, batch: int, slice_seed: int = 0) -> np.ndarray:
    """Config 5: (batch, nc, n) complex: CN(0,1) + sum_{i<r} a_ci e^{j w_i t},
    r = floor(K/2), w_i ~ U[0, 2 pi) shared by a matrix's coils, a ~ 4 CN(0,1)."""
    rng = Stream(SEED_SWEEP + slice_seed)
    r = k // 2
    z = rng.normal(2 * batch * nc * n).reshape(2, batch, nc, n)
    v = (z[0] + 1j * z[1]) / np.sqrt(2.0)
    w = rng.uniform(batch * r, 0.0, 2 * np.pi).reshape(batch, 1, r, 1)
    a = rng.normal(2 * batch * nc * r).reshape(2, batch, nc, r, 1)
    a = 4.0 * (a[0] + 1j * a[1]) / np.sqrt(2.0)
    t = np.arange(n, dtype=np.float64).reshape(1, 1, 1, n)
    v += np.sum(a * np.exp(1j * w * t), axis=2)
    return v


def sweep_tau(n: int, nc: int, k: int) -> float:
    """tau = sqrt(m) + sqrt(n) of the p x (nc*K) matrix (noise spectral edge)."""
    p = n - k + 1
    return float(np.sqrt(p) + np.sqrt(nc * k))
