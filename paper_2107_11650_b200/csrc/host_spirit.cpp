// SPIRiT kernel calibration on the host (setup, outside the per-iteration hot
// path; SURVEY.md 8(f) row 2 moves it to the device later).
//
// Reference: spirit_calibrate (proj/src/spirit.cpp:22-94) solves, per target
// coil dst, the Tikhonov-filtered least-squares problem
//     w = V diag(s / (s^2 + mu^2)) U^H b,   mu = tikhonov * s_max,
// on the (a-k+1)(b-k+1) x (k^2 J - 1) patch matrix with the self centre tap
// removed.  That filter is algebraically the ridge solution
//     (A^H A + mu^2 I) w = A^H b,
// which is what this file computes in FP64: one Hermitian Gram of the full
// patch matrix shared by all targets, s_max^2 by power iteration on the
// reduced Gram, and a Cholesky solve.
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "../../include/shlr_cuda.h"

namespace {

using cd = std::complex<double>;

double lambda_max(const std::vector<cd>& g, size_t n) {
  std::vector<cd> v(n, cd(1.0, 0.0)), w(n);
  double lam = 0.0;
  for (int it = 0; it < 20000; ++it) {
    for (size_t i = 0; i < n; ++i) {
      cd s(0, 0);
      for (size_t k = 0; k < n; ++k) s += g[i * n + k] * v[k];
      w[i] = s;
    }
    double nv = 0, num = 0;
    for (size_t i = 0; i < n; ++i) {
      nv += std::norm(v[i]);
      num += (std::conj(v[i]) * w[i]).real();
    }
    const double rq = num / nv;
    double nw = 0;
    for (size_t i = 0; i < n; ++i) nw += std::norm(w[i]);
    nw = std::sqrt(nw);
    if (nw == 0.0) return 0.0;
    for (size_t i = 0; i < n; ++i) v[i] = w[i] / nw;
    if (it > 10 && std::abs(rq - lam) <= 1e-15 * std::abs(rq)) return rq;
    lam = rq;
  }
  return lam;
}

bool cholesky_solve(std::vector<cd>& a, size_t n, std::vector<cd>& b) {
  for (size_t j = 0; j < n; ++j) {
    double d = a[j * n + j].real();
    for (size_t k = 0; k < j; ++k) d -= std::norm(a[j * n + k]);
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    a[j * n + j] = d;
    for (size_t i = j + 1; i < n; ++i) {
      cd s = a[i * n + j];
      for (size_t k = 0; k < j; ++k) s -= a[i * n + k] * std::conj(a[j * n + k]);
      a[i * n + j] = s / d;
    }
  }
  for (size_t i = 0; i < n; ++i) {  // L y = b
    cd s = b[i];
    for (size_t k = 0; k < i; ++k) s -= a[i * n + k] * b[k];
    b[i] = s / a[i * n + i].real();
  }
  for (size_t i = n; i-- > 0;) {  // L^H x = y
    cd s = b[i];
    for (size_t k = i + 1; k < n; ++k) s -= std::conj(a[k * n + i]) * b[k];
    b[i] = s / a[i * n + i].real();
  }
  return true;
}

}  // namespace

extern "C" int shlr_spirit_calibrate(const double* acs, size_t a, size_t b, size_t j, size_t k,
                                     double tikhonov, double* weights_out) {
  if (!acs || !weights_out || j == 0 || k == 0 || k % 2 == 0 || tikhonov < 0) return SHLR_EINVAL;
  if (a <= k || b <= k) return SHLR_EINVAL;  // CalibrationError in the reference
  const cd* x = reinterpret_cast<const cd*>(acs);
  double energy = 0;
  for (size_t i = 0; i < a * b * j; ++i) energy += std::norm(x[i]);
  if (energy == 0.0) return SHLR_EINVAL;
  const size_t h = k / 2;
  const size_t nf = k * k * j;
  const size_t nr = (a - k + 1) * (b - k + 1);
  // patch matrix rows in the reference's (r, c) order; feature (di, dj, src)
  std::vector<cd> feat(nr * nf), cen(nr * j);
  size_t row = 0;
  for (size_t r = h; r + h < a; ++r)
    for (size_t c = h; c + h < b; ++c, ++row) {
      size_t col = 0;
      for (size_t di = 0; di < k; ++di)
        for (size_t dj = 0; dj < k; ++dj)
          for (size_t s = 0; s < j; ++s, ++col)
            feat[row * nf + col] = x[((r + di - h) * b + (c + dj - h)) * j + s];
      for (size_t s = 0; s < j; ++s) cen[row * j + s] = x[(r * b + c) * j + s];
    }
  // Gram F^H F and F^H centres (shared by all targets)
  std::vector<cd> gram(nf * nf, cd(0, 0)), fc(nf * j, cd(0, 0));
  for (size_t rr = 0; rr < nr; ++rr) {
    const cd* fr = &feat[rr * nf];
    for (size_t p = 0; p < nf; ++p) {
      const cd cp = std::conj(fr[p]);
      cd* gp = &gram[p * nf];
      for (size_t q = p; q < nf; ++q) gp[q] += cp * fr[q];
      for (size_t s = 0; s < j; ++s) fc[p * j + s] += cp * cen[rr * j + s];
    }
  }
  for (size_t p = 0; p < nf; ++p)
    for (size_t q = 0; q < p; ++q) gram[p * nf + q] = std::conj(gram[q * nf + p]);
  std::memset(weights_out, 0, sizeof(double) * 2 * k * k * j * j);
  const size_t center_block = (h * k + h) * j;
  const size_t n = nf - 1;
  std::vector<size_t> colmap(n);
  for (size_t dst = 0; dst < j; ++dst) {
    size_t t = 0;
    for (size_t c = 0; c < nf; ++c)
      if (c != center_block + dst) colmap[t++] = c;
    std::vector<cd> g(n * n), rhs(n);
    for (size_t p = 0; p < n; ++p) {
      for (size_t q = 0; q < n; ++q) g[p * n + q] = gram[colmap[p] * nf + colmap[q]];
      rhs[p] = fc[colmap[p] * j + dst];
    }
    const double smax2 = lambda_max(g, n);
    const double mu2 = tikhonov * tikhonov * smax2;
    for (size_t p = 0; p < n; ++p) g[p * n + p] += mu2;
    if (!cholesky_solve(g, n, rhs)) return SHLR_EINVAL;
    for (size_t c = 0; c < n; ++c) {
      const size_t full = colmap[c];
      const size_t tap = full / j, src = full % j;
      const size_t wi = (tap * j + src) * j + dst;
      weights_out[2 * wi] = rhs[c].real();
      weights_out[2 * wi + 1] = rhs[c].imag();
    }
  }
  return SHLR_OK;
}
