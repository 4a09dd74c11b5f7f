// Image-quality metrics on the device: the sum-of-squares
// coil combination ssos (proj/src/io.cpp:105-117), RLNE and mean SSIM
// (proj/src/metrics.cpp:9-75).  FP64 throughout.  Per-pixel / per-window
// arithmetic follows the reference's operation order with round-to-nearest
// intrinsics (no FMA contraction), so ssos and every window's SSIM are
// bitwise the reference's; the final sums are deterministic tree reductions
// (a different summation order than the reference's sequential loop: ~1e-16
// relative).
#include <cmath>
#include <vector>

#include "common.cuh"
#include "metrics.cuh"

namespace shlr_b200 {

namespace {

constexpr int kWin = 11;
constexpr int kMetricThreads = 256;

__constant__ double c_win[kWin * kWin];  // normalised Gaussian window (metrics.cpp:31-41)

// out[r][c] = sqrt(sum_k |x[r][c][k]|^2), k ascending (io.cpp:109-115)
__global__ void k_ssos(const double2* __restrict__ x, size_t pixels, int j, double* __restrict__ out) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pixels) return;
  double s = 0.0;
  for (int k = 0; k < j; ++k) {
    const double2 v = x[p * j + k];
    s = __dadd_rn(s, __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)));  // std::norm
  }
  out[p] = __dsqrt_rn(s);
}

// Deterministic block reduction of two FP64 partial sums.
__device__ __forceinline__ void block_sum2(double& a, double& b, double* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) {
    sh[w] = a;
    sh[nw + w] = b;
  }
  __syncthreads();
  if (w == 0) {
    a = l < nw ? sh[l] : 0.0;
    b = l < nw ? sh[nw + l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
  }
}

// Per block: sum (ref - rec)^2 and sum ref^2 over a grid-stride range.
__global__ void k_rlne_partial(const double* __restrict__ ref, const double* __restrict__ rec, size_t count,
                               double2* __restrict__ part) {
  __shared__ double sh[2 * (kMetricThreads / 32)];
  double num = 0.0, den = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const double d = __dsub_rn(ref[i], rec[i]);
    num = __dadd_rn(num, __dmul_rn(d, d));
    den = __dadd_rn(den, __dmul_rn(ref[i], ref[i]));
  }
  block_sum2(num, den, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = make_double2(num, den);
}

// Sum of the per-block partials (one block, fixed order).
__global__ void k_sum_partials(const double2* __restrict__ part, int n, double2* __restrict__ out) {
  __shared__ double sh[2 * (kMetricThreads / 32)];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    a += part[i].x;
    b += part[i].y;
  }
  block_sum2(a, b, sh);
  if (threadIdx.x == 0) *out = make_double2(a, b);
}

// max(ref) (metrics.cpp:43-45; max is order-independent): per block, then one block
__global__ void k_max_partial(const double* __restrict__ ref, size_t count, double* __restrict__ part) {
  __shared__ double sh[kMetricThreads / 32];
  double m = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    m = fmax(m, ref[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    part[blockIdx.x] = m;
  }
}

// SSIM of the 11 x 11 window at (r, c), the reference's loop order
// (metrics.cpp:49-70): means, then variances and covariance about them.
__device__ double window_ssim(const double* __restrict__ a, const double* __restrict__ b, size_t cols, size_t r,
                              size_t c, double c1, double c2) {
  double mu_a = 0.0, mu_b = 0.0;
  for (int i = 0; i < kWin; ++i)
    for (int jj = 0; jj < kWin; ++jj) {
      const double w = c_win[i * kWin + jj];
      const size_t o = (r + i) * cols + c + jj;
      mu_a = __dadd_rn(mu_a, __dmul_rn(w, a[o]));
      mu_b = __dadd_rn(mu_b, __dmul_rn(w, b[o]));
    }
  double var_a = 0.0, var_b = 0.0, cov = 0.0;
  for (int i = 0; i < kWin; ++i)
    for (int jj = 0; jj < kWin; ++jj) {
      const double w = c_win[i * kWin + jj];
      const size_t o = (r + i) * cols + c + jj;
      const double da = __dsub_rn(a[o], mu_a), db = __dsub_rn(b[o], mu_b);
      var_a = __dadd_rn(var_a, __dmul_rn(__dmul_rn(w, da), da));
      var_b = __dadd_rn(var_b, __dmul_rn(__dmul_rn(w, db), db));
      cov = __dadd_rn(cov, __dmul_rn(__dmul_rn(w, da), db));
    }
  const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_a), mu_b), c1),
                               __dadd_rn(__dmul_rn(2.0, cov), c2));
  const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu_a, mu_a), __dmul_rn(mu_b, mu_b)), c1),
                               __dadd_rn(__dadd_rn(var_a, var_b), c2));
  return __ddiv_rn(num, den);
}

// Per block: sum of the window SSIMs over a grid-stride range of windows.
__global__ void k_ssim_partial(const double* __restrict__ a, const double* __restrict__ b, size_t rows, size_t cols,
                               const double* __restrict__ maxref, double2* __restrict__ part) {
  __shared__ double sh[2 * (kMetricThreads / 32)];
  const double mx = *maxref;
  const double c1 = __dmul_rn(__dmul_rn(0.01, mx), __dmul_rn(0.01, mx));
  const double c2 = __dmul_rn(__dmul_rn(0.03, mx), __dmul_rn(0.03, mx));
  const size_t wr = rows - kWin + 1, wc = cols - kWin + 1, nwin = wr * wc;
  double s = 0.0, unused = 0.0;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < nwin; t += (size_t)gridDim.x * blockDim.x)
    s += window_ssim(a, b, cols, t / wc, t % wc, c1, c2);
  block_sum2(s, unused, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = make_double2(s, 0.0);
}

int grid_of(size_t n) { return (int)std::min<size_t>(592, std::max<size_t>(1, (n + kMetricThreads - 1) / kMetricThreads)); }

template <typename T>
T* dev_copy(const T* h, size_t n, cudaStream_t s) {
  T* d = nullptr;
  SHLR_CUDA(cudaMallocAsync(&d, std::max<size_t>(n, 1) * sizeof(T), s));
  if (n) SHLR_CUDA(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  return d;
}

}  // namespace

void ssos_host(const double* x, size_t m, size_t n, size_t j, double* out) {
  if (m == 0 || n == 0 || j == 0) throw InvalidArg("ssos: expected an M x N x J tensor");
  cudaStream_t s;
  SHLR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t pixels = m * n;
  double2* dx = dev_copy(reinterpret_cast<const double2*>(x), pixels * j, s);
  double* dout = nullptr;
  SHLR_CUDA(cudaMallocAsync(&dout, pixels * sizeof(double), s));
  k_ssos<<<(int)((pixels + kMetricThreads - 1) / kMetricThreads), kMetricThreads, 0, s>>>(dx, pixels, (int)j, dout);
  SHLR_LAUNCH_CHECK();
  SHLR_CUDA(cudaMemcpyAsync(out, dout, pixels * sizeof(double), cudaMemcpyDeviceToHost, s));
  SHLR_CUDA(cudaFreeAsync(dx, s));
  SHLR_CUDA(cudaFreeAsync(dout, s));
  SHLR_CUDA(cudaStreamSynchronize(s));
  SHLR_CUDA(cudaStreamDestroy(s));
}

double rlne_host(const double* ref, const double* rec, size_t count) {
  cudaStream_t s;
  SHLR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double* da = dev_copy(ref, count, s);
  double* db = dev_copy(rec, count, s);
  const int g = grid_of(count);
  double2 *part = nullptr, *tot = nullptr;
  SHLR_CUDA(cudaMallocAsync(&part, g * sizeof(double2), s));
  SHLR_CUDA(cudaMallocAsync(&tot, sizeof(double2), s));
  k_rlne_partial<<<g, kMetricThreads, 0, s>>>(da, db, count, part);
  SHLR_LAUNCH_CHECK();
  k_sum_partials<<<1, kMetricThreads, 0, s>>>(part, g, tot);
  SHLR_LAUNCH_CHECK();
  double2 h;
  SHLR_CUDA(cudaMemcpyAsync(&h, tot, sizeof(double2), cudaMemcpyDeviceToHost, s));
  for (void* p : {(void*)da, (void*)db, (void*)part, (void*)tot}) SHLR_CUDA(cudaFreeAsync(p, s));
  SHLR_CUDA(cudaStreamSynchronize(s));
  SHLR_CUDA(cudaStreamDestroy(s));
  if (h.y == 0.0) throw InvalidArg("rlne: reference image is identically zero");
  return std::sqrt(h.x / h.y);
}

double mssim_host(const double* ref, const double* rec, size_t rows, size_t cols) {
  if (rows < (size_t)kWin || cols < (size_t)kWin)
    throw InvalidArg("mssim: image smaller than the 11x11 window");
  // the window exactly as metrics.cpp:31-41 builds it (host FP64)
  double w[kWin * kWin], wsum = 0.0;
  for (int i = 0; i < kWin; ++i)
    for (int j = 0; j < kWin; ++j) {
      const double di = (double)i - 5.0, dj = (double)j - 5.0;
      w[i * kWin + j] = std::exp(-(di * di + dj * dj) / (2.0 * 1.5 * 1.5));
      wsum += w[i * kWin + j];
    }
  for (double& v : w) v /= wsum;
  cudaStream_t s;
  SHLR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  SHLR_CUDA(cudaMemcpyToSymbolAsync(c_win, w, sizeof(w), 0, cudaMemcpyHostToDevice, s));
  const size_t count = rows * cols;
  double* da = dev_copy(ref, count, s);
  double* db = dev_copy(rec, count, s);
  const int gm = grid_of(count);
  double *mpart = nullptr, *mx = nullptr;
  SHLR_CUDA(cudaMallocAsync(&mpart, gm * sizeof(double), s));
  SHLR_CUDA(cudaMallocAsync(&mx, sizeof(double), s));
  k_max_partial<<<gm, kMetricThreads, 0, s>>>(da, count, mpart);
  SHLR_LAUNCH_CHECK();
  k_max_partial<<<1, kMetricThreads, 0, s>>>(mpart, gm, mx);
  SHLR_LAUNCH_CHECK();
  const size_t nwin = (rows - kWin + 1) * (cols - kWin + 1);
  const int g = grid_of(nwin);
  double2 *part = nullptr, *tot = nullptr;
  SHLR_CUDA(cudaMallocAsync(&part, g * sizeof(double2), s));
  SHLR_CUDA(cudaMallocAsync(&tot, sizeof(double2), s));
  k_ssim_partial<<<g, kMetricThreads, 0, s>>>(da, db, rows, cols, mx, part);
  SHLR_LAUNCH_CHECK();
  k_sum_partials<<<1, kMetricThreads, 0, s>>>(part, g, tot);
  SHLR_LAUNCH_CHECK();
  double2 h;
  SHLR_CUDA(cudaMemcpyAsync(&h, tot, sizeof(double2), cudaMemcpyDeviceToHost, s));
  for (void* p : {(void*)da, (void*)db, (void*)mpart, (void*)mx, (void*)part, (void*)tot})
    SHLR_CUDA(cudaFreeAsync(p, s));
  SHLR_CUDA(cudaStreamSynchronize(s));
  SHLR_CUDA(cudaStreamDestroy(s));
  return h.x / (double)nwin;
}

}  // namespace shlr_b200
