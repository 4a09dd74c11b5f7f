// Helpers shared by the ADMM drivers (pi_solver.cu, param_solver.cu):
// deterministic FP64 block reductions, device allocation, grid sizing and
// the FP64 host-side constants of the Hankel operators.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace shlr_b200 {
namespace util {

constexpr int kThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (valid in thread 0; sh holds >= 32 doubles).
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double t = 0.0;
  if (warp == 0) {
    t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

// Block sum broadcast to every thread (fixed summation order).
__device__ __forceinline__ double block_sum_all(double v, double* sh) {
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) sh[32] = t;
  __syncthreads();
  const double r = sh[32];
  __syncthreads();
  return r;
}

template <class T>
inline T* dalloc(size_t n) {
  T* p = nullptr;
  SHLR_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return p;
}

// Stream-ordered allocation from the device's default pool, which is told to
// keep freed memory (release threshold: unlimited), so a plan created after
// another one was destroyed reuses its memory without cudaMalloc/cudaFree.
inline void keep_pool_memory() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  SHLR_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  SHLR_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = UINT64_MAX;
  SHLR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done = true;
}
template <class T>
inline T* dalloc_s(size_t n, cudaStream_t s) {
  keep_pool_memory();
  T* p = nullptr;
  SHLR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), s));
  return p;
}

inline int grid_for(size_t n) {
  const size_t blocks = (n + kThreads * 4 - 1) / (kThreads * 4);
  return (int)std::max<size_t>(1, std::min<size_t>(blocks, (size_t)num_sms() * 4));
}

// hankel_counts (proj/src/hankel.cpp:56-62)
inline std::vector<double> hankel_counts_h(int n, int p) {
  std::vector<double> c(n, 0.0);
  const int q = n - p + 1;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < q; ++j) c[i + j] += 1.0;
  return c;
}

// weights_centered (proj/src/hankel.cpp:75-97), as (re, im) pairs.
inline std::vector<double> weights_centered_h(const double* taps, size_t ntaps, int n) {
  std::vector<double> w(2 * n, 0.0), out(2 * n, 0.0);
  for (int k = 0; k < n; ++k) {
    double sr = 0, si = 0;
    for (size_t t = 0; t < ntaps; ++t) {
      const double ang = -2.0 * M_PI * (double)k * (double)t / (double)n;
      const double c = std::cos(ang), s = std::sin(ang);
      sr += taps[2 * t] * c - taps[2 * t + 1] * s;
      si += taps[2 * t] * s + taps[2 * t + 1] * c;
    }
    w[2 * k] = sr;
    w[2 * k + 1] = si;
  }
  const int c = n / 2;
  for (int i = 0; i < n; ++i) {  // fftshift: out[(i + c) % n] = w[i]
    out[2 * ((i + c) % n)] = w[2 * i];
    out[2 * ((i + c) % n) + 1] = w[2 * i + 1];
  }
  return out;
}

inline int dagger_h(int i, int n) { return (2 * (n / 2) + n - i) % n; }

// Diagonal of the weighted-lift normal operator in k-space,
// a_n(k) = |wc[k]|^2 counts[k] (+ the virtual-coil mirror a_n(fl(k))):
// lift_weighted_normal (proj/src/operators.cpp:173-197).
inline std::vector<double> lift_normal_diag_h(const std::vector<double>& w,
                                              const std::vector<double>& cnt, int n, bool vc) {
  std::vector<double> a(n);
  for (int k = 0; k < n; ++k) {
    a[k] = (w[2 * k] * w[2 * k] + w[2 * k + 1] * w[2 * k + 1]) * cnt[k];
    if (vc) {
      const int f = dagger_h(k, n);
      a[k] += (w[2 * f] * w[2 * f] + w[2 * f + 1] * w[2 * f + 1]) * cnt[f];
    }
  }
  return a;
}

// Spectrum of the weighted adjoint of an all-(-1/beta) lifted matrix (the
// first RHS, Z = 0, D = 1: proj/src/solvers.cpp:128-139):
// -(conj(wc) counts (+ vc: wc[fl] counts[fl])) / beta.
inline std::vector<float2> initial_weighted_adjoint_h(const std::vector<double>& w,
                                                      const std::vector<double>& cnt, int n,
                                                      bool vc, double beta) {
  std::vector<float2> h(n);
  for (int k = 0; k < n; ++k) {
    double re = w[2 * k] * cnt[k], im = -w[2 * k + 1] * cnt[k];
    if (vc) {
      const int f = dagger_h(k, n);
      re += w[2 * f] * cnt[f];
      im += w[2 * f + 1] * cnt[f];
    }
    h[k] = make_float2((float)(-re / beta), (float)(-im / beta));
  }
  return h;
}

}  // namespace util
}  // namespace shlr_b200
