// Host-side helpers of the C-ABI boundary: the reference's seeded mask
// generators and pencil rule, bit-exact (the masks are inputs of the hot path
// and must match the reference exactly; BASELINE "mask bit-exact").
//   splitmix64 SeededRng      proj/include/shlr/sampling.hpp:11-29
//   acs_range                 proj/src/sampling.cpp:31-41
//   exact-count draw          proj/src/sampling.cpp:64-88
//   mask_gauss_cartesian      proj/src/sampling.cpp:92-128
//   mask_random2d             proj/src/sampling.cpp:130-173
//   HankelConfig::pencil_for  proj/src/hankel.cpp:10-18
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/shlr_cuda.h"

namespace {

struct SplitMix64 {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

bool acs_bounds(size_t n, size_t acs, size_t* a0, size_t* a1) {
  if (acs == 0) {
    *a0 = *a1 = 0;
    return true;
  }
  if (acs > n) return false;
  const size_t c = n / 2, half_up = (acs + 1) / 2;
  if (half_up > c) return false;
  *a0 = c - half_up;
  *a1 = *a0 + acs;
  return true;
}

// Sequential sums in index order keep the draw bit-exact with the reference.
void draw_exact(uint8_t* bits, std::vector<size_t> pool, const std::vector<double>& weight,
                size_t want, SplitMix64& rng) {
  std::vector<double> w;
  w.reserve(pool.size());
  for (size_t i : pool) w.push_back(weight[i]);
  for (size_t k = 0; k < want; ++k) {
    double total = 0.0;
    for (double v : w) total += v;
    const double u = rng.uniform() * total;
    size_t pick = pool.size() - 1;
    double acc = 0.0;
    for (size_t i = 0; i < pool.size(); ++i) {
      acc += w[i];
      if (u < acc) {
        pick = i;
        break;
      }
    }
    bits[pool[pick]] = 1;
    pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(pick));
    w.erase(w.begin() + static_cast<std::ptrdiff_t>(pick));
  }
}

}  // namespace

extern "C" {

int shlr_acs_range(size_t n, size_t acs, size_t* start, size_t* end) {
  size_t a0, a1;
  if (!acs_bounds(n, acs, &a0, &a1)) return SHLR_EINVAL;
  if (start) *start = a0;
  if (end) *end = a1;
  return SHLR_OK;
}

size_t shlr_pencil_for(size_t pencil, size_t len) {
  if (pencil != 0) return pencil > len ? 0 : pencil;  // 0 signals "exceeds length"
  if (len >= 64) return 23;
  return len / 3 + (len % 3 ? 1 : 0) + 1;
}

// HankelConfig::pencil_for_param (proj/src/hankel.cpp:20-29): the same rule
// on its own field.
size_t shlr_pencil_for_param(size_t pencil_param, size_t len) {
  return shlr_pencil_for(pencil_param, len);
}

int shlr_mask_gauss_cartesian(size_t n, double rate, size_t acs, uint64_t seed, uint8_t* bits) {
  if (n == 0 || !(rate > 0.0) || rate > 1.0 || !bits) return SHLR_EINVAL;
  const size_t want = static_cast<size_t>(std::ceil(rate * static_cast<double>(n)));
  if (want < acs) return SHLR_EINVAL;
  size_t a0, a1;
  if (!acs_bounds(n, acs, &a0, &a1)) return SHLR_EINVAL;
  std::memset(bits, 0, n);
  for (size_t i = a0; i < a1; ++i) bits[i] = 1;
  const double sigma = static_cast<double>(n) / 6.0;
  const double c = static_cast<double>(n / 2);
  std::vector<double> weight(n);
  for (size_t i = 0; i < n; ++i) {
    const double d = static_cast<double>(i) - c;
    weight[i] = std::exp(-d * d / (2.0 * sigma * sigma));
  }
  std::vector<size_t> pool;
  for (size_t i = 0; i < n; ++i)
    if (!bits[i]) pool.push_back(i);
  SplitMix64 rng{seed};
  draw_exact(bits, pool, weight, want - (a1 - a0), rng);
  return SHLR_OK;
}

int shlr_mask_random2d(size_t rows, size_t cols, double rate, size_t center, uint64_t seed,
                       uint8_t* bits) {
  if (rows == 0 || cols == 0 || !(rate > 0.0) || rate > 1.0 || !bits) return SHLR_EINVAL;
  const size_t total = rows * cols;
  const size_t want = static_cast<size_t>(std::ceil(rate * static_cast<double>(total)));
  size_t r0, r1, c0, c1;
  if (!acs_bounds(rows, center, &r0, &r1) || !acs_bounds(cols, center, &c0, &c1)) return SHLR_EINVAL;
  const size_t block = (r1 - r0) * (c1 - c0);
  if (block > want) return SHLR_EINVAL;
  std::memset(bits, 0, total);
  for (size_t r = r0; r < r1; ++r)
    for (size_t c = c0; c < c1; ++c) bits[r * cols + c] = 1;
  const double sigma = static_cast<double>(rows < cols ? rows : cols) / 6.0;
  const double cr = static_cast<double>(rows / 2), cc = static_cast<double>(cols / 2);
  std::vector<double> weight(total);
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < cols; ++c) {
      const double dr = static_cast<double>(r) - cr, dc = static_cast<double>(c) - cc;
      weight[r * cols + c] = std::exp(-(dr * dr + dc * dc) / (2.0 * sigma * sigma));
    }
  std::vector<size_t> pool;
  for (size_t i = 0; i < total; ++i)
    if (!bits[i]) pool.push_back(i);
  SplitMix64 rng{seed};
  draw_exact(bits, pool, weight, want - block, rng);
  return SHLR_OK;
}

}  // extern "C"
