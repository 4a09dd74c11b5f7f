// C++ drop-in tests of include/shlr_b200/shlr.hpp (the reference API over the
// C-ABI), written like the reference's own solver tests
// (proj/tests/test_solvers.cpp:184-302) but with the BASELINE parity
// tolerance for the FP32 device path.  Built by __graft_entry__.build() into
// tests/cpp/_build/test_dropin and run on the GPU by tests/test_dropin_cpp.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "../../oracle/doctest_shim/doctest.h"

#include <cmath>
#include <limits>
#include <random>
#include <sstream>

#include "shlr_b200/shlr.hpp"

using namespace shlr_b200;

namespace {

// Smooth complex phantom with J coil weightings, returned as centred k-space.
ComplexTensor phantom_kspace(std::size_t n, std::size_t coils, std::uint32_t seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  ComplexTensor img({n, n, coils});
  const double c = static_cast<double>(n) / 2.0;
  for (std::size_t r = 0; r < n; ++r)
    for (std::size_t q = 0; q < n; ++q) {
      const double dr = (static_cast<double>(r) - c) / (0.7 * c);
      const double dq = (static_cast<double>(q) - c) / (0.75 * c);
      double mag = dr * dr + dq * dq <= 1.0 ? 1.0 : 0.0;
      if (std::abs(static_cast<double>(r) - 0.7 * c) < 0.18 * c &&
          std::abs(static_cast<double>(q) - 0.8 * c) < 0.25 * c)
        mag = 1.8;
      const double ph = 0.05 * (static_cast<double>(r) + 0.5 * static_cast<double>(q));
      for (std::size_t j = 0; j < coils; ++j) {
        const double w = 1.0 + 0.3 * std::cos(static_cast<double>(j) + 0.1 * static_cast<double>(r));
        img.at(r, q, j) = mag * w * cplx{std::cos(ph), std::sin(ph)} + 1e-3 * cplx{u(rng), u(rng)};
      }
    }
  return fft2d_centered(img);
}

double rel_diff(const ComplexTensor& a, const ComplexTensor& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(a[i]);
  }
  return std::sqrt(num / den);
}

double max_abs_diff(const ComplexTensor& a, const ComplexTensor& b) {
  double m = 0;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

}  // namespace

TEST_CASE("parallel imaging: full sampling with strong fidelity is exact") {
  ComplexTensor k = phantom_kspace(32, 2, 11);
  SamplingMask full = mask_gauss_cartesian(32, 1.0, 4, 1);
  HankelConfig hcfg;
  AdmmConfig acfg;
  acfg.lambda = 1e6;
  acfg.enable_vc = true;
  acfg.max_outer = 10;
  ComplexTensor rec = shlr_pi_reconstruct(k, full, nullptr, hcfg, acfg);
  ComplexTensor direct = ifft2d_centered(k);
  CHECK(rel_diff(direct, rec) < 1e-3);
}

TEST_CASE("parallel imaging: determinism and progress log format") {
  ComplexTensor k = phantom_kspace(24, 2, 21);
  SamplingMask mask = mask_gauss_cartesian(24, 0.6, 6, 5);
  HankelConfig hcfg;
  AdmmConfig acfg;
  acfg.max_outer = 3;
  std::ostringstream log;
  SolveStats stats;
  ComplexTensor a = shlr_pi_reconstruct(k, mask, nullptr, hcfg, acfg, &log, &stats);
  ComplexTensor b = shlr_pi_reconstruct(k, mask, nullptr, hcfg, acfg);
  CHECK(max_abs_diff(a, b) == 0.0);
  CHECK(stats.outer_iters == 3);
  std::istringstream in(log.str());
  std::string line;
  std::size_t lines = 0;
  while (std::getline(in, line)) {
    CHECK(line.find("iter=") != std::string::npos);
    CHECK(line.find("relchange=") != std::string::npos);
    CHECK(line.find("cg_iters=") != std::string::npos);
    CHECK(line.find("cg_res=") != std::string::npos);
    ++lines;
  }
  CHECK(lines == 3);
}

TEST_CASE("variant nesting: vc off equals the base model bitwise") {
  ComplexTensor k = phantom_kspace(16, 2, 31);
  SamplingMask mask = mask_gauss_cartesian(16, 0.75, 4, 9);
  HankelConfig hcfg;
  AdmmConfig base;
  base.max_outer = 4;
  AdmmConfig same = base;
  same.enable_vc = false;
  same.enable_spirit = false;
  ComplexTensor a = shlr_pi_reconstruct(k, mask, nullptr, hcfg, base);
  ComplexTensor b = shlr_pi_reconstruct(k, mask, nullptr, hcfg, same);
  CHECK(max_abs_diff(a, b) == 0.0);
}

TEST_CASE("parallel imaging: missing kernels with spirit enabled is an error") {
  ComplexTensor y({8, 8, 2});
  y.at(4, 4, 0) = {1, 0};
  SamplingMask mask = mask_gauss_cartesian(8, 1.0, 0, 1);
  HankelConfig hcfg;
  AdmmConfig acfg;
  acfg.enable_spirit = true;
  CHECK_THROWS_AS(shlr_pi_reconstruct(y, mask, nullptr, hcfg, acfg), std::invalid_argument);
}

TEST_CASE("argument validation mirrors the reference") {
  ComplexTensor y({8, 8, 2});
  SamplingMask mask = mask_gauss_cartesian(8, 1.0, 0, 1);
  HankelConfig hcfg;
  AdmmConfig bad;
  bad.beta = 0.0;
  CHECK_THROWS_AS(shlr_pi_reconstruct(y, mask, nullptr, hcfg, bad), std::invalid_argument);
  SamplingMask wrong = mask_gauss_cartesian(6, 1.0, 0, 1);
  CHECK_THROWS_AS(shlr_pi_reconstruct(y, wrong, nullptr, hcfg, AdmmConfig{}), std::invalid_argument);
  ComplexTensor flat({8, 8});
  CHECK_THROWS_AS(shlr_pi_reconstruct(flat, mask, nullptr, hcfg, AdmmConfig{}), std::invalid_argument);
  HankelConfig too_long;
  too_long.pencil = 9;
  CHECK_THROWS_AS(shlr_pi_reconstruct(y, mask, nullptr, too_long, AdmmConfig{}), std::invalid_argument);
  CHECK_THROWS_AS(SpiritKernels(4, 1, std::vector<cplx>(16)), std::invalid_argument);
}

TEST_CASE("non-finite data raises DivergenceError") {
  ComplexTensor y = phantom_kspace(16, 2, 3);
  y.at(8, 8, 0) = cplx{std::numeric_limits<double>::quiet_NaN(), 0.0};
  SamplingMask mask = mask_gauss_cartesian(16, 1.0, 0, 1);
  AdmmConfig acfg;
  acfg.max_outer = 2;
  CHECK_THROWS_AS(shlr_pi_reconstruct(y, mask, nullptr, HankelConfig{}, acfg), DivergenceError);
}

TEST_CASE("stopping rules: iteration caps and early exit on stagnation") {
  ComplexTensor k = phantom_kspace(16, 2, 41);
  SamplingMask mask = mask_gauss_cartesian(16, 0.6, 4, 2);
  HankelConfig hcfg;
  AdmmConfig capped;
  capped.max_outer = 2;
  SolveStats stats;
  shlr_pi_reconstruct(k, mask, nullptr, hcfg, capped, nullptr, &stats);
  CHECK(stats.outer_iters == 2);
  AdmmConfig loose;
  loose.tol = 1e9;
  shlr_pi_reconstruct(k, mask, nullptr, hcfg, loose, nullptr, &stats);
  CHECK(stats.outer_iters == 1);
}

TEST_CASE("SHLR-SV with calibrated kernels runs and improves on zero filling") {
  ComplexTensor k = phantom_kspace(32, 4, 51);
  SamplingMask mask = mask_gauss_cartesian(32, 0.5, 8, 7);
  ComplexTensor y({32, 32, 4});
  for (std::size_t r = 0; r < 32; ++r)
    for (std::size_t c = 0; c < 32; ++c)
      if (mask.sampled(r, c))
        for (std::size_t j = 0; j < 4; ++j) y.at(r, c, j) = k.at(r, c, j);
  auto [a0, a1] = acs_range(32, 8);
  ComplexTensor acs({32, a1 - a0, 4});
  for (std::size_t r = 0; r < 32; ++r)
    for (std::size_t c = a0; c < a1; ++c)
      for (std::size_t j = 0; j < 4; ++j) acs.at(r, c - a0, j) = y.at(r, c, j);
  SpiritKernels g = spirit_calibrate(acs, 3);
  AdmmConfig acfg;
  acfg.enable_spirit = true;
  acfg.enable_vc = true;
  acfg.max_outer = 20;
  HankelConfig hcfg;
  hcfg.pencil = 11;
  ComplexTensor rec = shlr_pi_reconstruct(y, mask, &g, hcfg, acfg);
  ComplexTensor truth = ifft2d_centered(k);
  ComplexTensor zf = ifft2d_centered(y);
  CHECK(rel_diff(truth, rec) < rel_diff(truth, zf));
}

// ---------------------------------------------------------------- parameter imaging
namespace {
// N x L x J plane: mono-exponential decays along the echoes (low rank in the
// echo lift), smooth along PE, in PE k-space.
ComplexTensor param_plane(std::size_t n, std::size_t l, std::size_t coils, std::uint32_t seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  ComplexTensor img({n, l, coils});
  for (std::size_t r = 0; r < n; ++r) {
    const double pd = std::abs(static_cast<double>(r) - n / 2.0) < n / 3.0 ? 1.0 : 0.2;
    const double t2 = 40.0 + 60.0 * static_cast<double>(r % 7) / 7.0;
    for (std::size_t e = 0; e < l; ++e)
      for (std::size_t j = 0; j < coils; ++j)
        img.at(r, e, j) = pd * std::exp(-10.0 * static_cast<double>(e + 1) / t2) *
                              (1.0 + 0.2 * static_cast<double>(j)) +
                          1e-3 * cplx{u(rng), u(rng)};
  }
  return fft_along_axis(img, 0, false);
}
}  // namespace

TEST_CASE("parameter imaging: full sampling with strong fidelity is exact") {
  const std::size_t n = 32, l = 9, j = 2;
  ComplexTensor y = param_plane(n, l, j, 5);
  SamplingMask mask{n, l, std::vector<std::uint8_t>(n * l, 1)};
  AdmmConfig acfg;
  acfg.lambda = 1e6;
  acfg.max_outer = 5;
  const ComplexTensor rec = shlr_param_reconstruct_slice(y, mask, HankelConfig{}, acfg);
  CHECK(rel_diff(fft_along_axis(y, 0, true), rec) < 1e-3);
}

TEST_CASE("parameter imaging: determinism, log format, SHLR-VP differs from SHLR-P") {
  const std::size_t n = 32, l = 9, j = 2;
  ComplexTensor y = param_plane(n, l, j, 6);
  SamplingMask mask{n, l, std::vector<std::uint8_t>(n * l, 0)};
  for (std::size_t r = 0; r < n; ++r)
    for (std::size_t e = 0; e < l; ++e) mask.bits[r * l + e] = ((r + 3 * e) % 3 == 0 || (r > 12 && r < 20));
  AdmmConfig acfg;
  acfg.max_outer = 3;
  acfg.tol = 1e-300;
  std::ostringstream log;
  SolveStats stats;
  const ComplexTensor a = shlr_param_reconstruct_slice(y, mask, HankelConfig{}, acfg, &log, &stats);
  const ComplexTensor b = shlr_param_reconstruct_slice(y, mask, HankelConfig{}, acfg);
  CHECK(max_abs_diff(a, b) == 0.0);
  CHECK(stats.outer_iters == 3);
  std::istringstream in(log.str());
  std::string line;
  int lines = 0;
  while (std::getline(in, line)) {
    CHECK(line.find("iter=") == 0);
    CHECK(line.find("cg_iters=") != std::string::npos);
    ++lines;
  }
  CHECK(lines == 3);
  AdmmConfig vp = acfg;
  vp.enable_vc = true;
  const ComplexTensor c = shlr_param_reconstruct_slice(y, mask, HankelConfig{}, vp);
  const ComplexTensor c2 = shlr_param_reconstruct_slice(y, mask, HankelConfig{}, vp);
  CHECK(max_abs_diff(c, c2) == 0.0);
  CHECK(max_abs_diff(a, c) > 0.0);
}

TEST_CASE("parameter imaging: dataset = per-slice solves, argument validation") {
  const std::size_t m = 3, n = 24, l = 8, j = 2;
  ComplexTensor plane = param_plane(n, l, j, 7);
  ParameterDataset ds;
  ds.data = ComplexTensor({m, n, l, j});
  for (std::size_t f = 0; f < m; ++f)
    for (std::size_t i = 0; i < n * l * j; ++i) ds.data[f * n * l * j + i] = plane[i] * (1.0 + 0.5 * f);
  for (std::size_t e = 0; e < l; ++e) ds.tes_ms.push_back(10.0 * static_cast<double>(e + 1));
  SamplingMask mask{n, l, std::vector<std::uint8_t>(n * l, 0)};
  for (std::size_t r = 0; r < n; ++r)
    for (std::size_t e = 0; e < l; ++e) mask.bits[r * l + e] = ((r + e) % 2 == 0 || (r > 9 && r < 15));
  AdmmConfig acfg;
  acfg.max_outer = 2;
  acfg.tol = 1e-300;
  std::size_t total = 0;
  const ParameterDataset rec = recon_param_dataset(ds, mask, HankelConfig{}, acfg, nullptr, &total);
  CHECK(total == m * 2);
  // slice f of the dataset = the slice solve of the FE-iFFT of the data
  const ComplexTensor hybrid = fft_along_axis(ds.data, 0, true);
  for (std::size_t f = 0; f < m; ++f) {
    ComplexTensor yf({n, l, j});
    for (std::size_t i = 0; i < n * l * j; ++i) yf[i] = hybrid[f * n * l * j + i];
    const ComplexTensor xf = shlr_param_reconstruct_slice(yf, mask, HankelConfig{}, acfg);
    ComplexTensor rf({n, l, j});
    for (std::size_t i = 0; i < n * l * j; ++i) rf[i] = rec.data[f * n * l * j + i];
    CHECK(rel_diff(xf, rf) < 1e-4);
  }
  ParameterDataset bad = ds;
  bad.tes_ms[1] = bad.tes_ms[0];
  CHECK_THROWS_AS(recon_param_dataset(bad, mask, HankelConfig{}, acfg), std::invalid_argument);
  SamplingMask wrong{n, l + 1, std::vector<std::uint8_t>(n * (l + 1), 1)};
  CHECK_THROWS_AS(recon_param_dataset(ds, wrong, HankelConfig{}, acfg), std::invalid_argument);
  HankelConfig hp;
  hp.pencil_param = l + 1;
  CHECK_THROWS_AS(shlr_param_reconstruct_slice(plane, mask, hp, acfg), std::invalid_argument);
}

TEST_CASE("SPIRiT calibration: device FP64 equals the host restatement") {
  const std::size_t n = 32, j = 3;
  ComplexTensor k = phantom_kspace(n, j, 9);
  ComplexTensor acs({n, 12, j});
  for (std::size_t r = 0; r < n; ++r)
    for (std::size_t c = 0; c < 12; ++c)
      for (std::size_t q = 0; q < j; ++q) acs.at(r, c, q) = k.at(r, c + 10, q);
  const SpiritKernels h = spirit_calibrate(acs, 5, 1e-4);
  const SpiritKernels d = spirit_calibrate_device(acs, 5, 1e-4);
  double mx = 0, md = 0;
  for (std::size_t i = 0; i < h.raw().size(); ++i) {
    mx = std::max(mx, std::abs(h.raw()[i]));
    md = std::max(md, std::abs(h.raw()[i] - d.raw()[i]));
  }
  // both solve the same ridge system in FP64 with different summation orders;
  // cond(A^H A + mu^2 I) <= 1 / tikhonov^2 = 1e8
  CHECK(md <= 1e-6 * mx);
  CHECK_THROWS_AS(spirit_calibrate_device(ComplexTensor({4, 4, j}), 5, 1e-4), CalibrationError);
}
