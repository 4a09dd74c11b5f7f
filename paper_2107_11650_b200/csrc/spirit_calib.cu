// SPIRiT kernel calibration on the device, FP64.
//
// Reference: spirit_calibrate (proj/src/spirit.cpp:22-94).  Per target coil
// dst it solves the Tikhonov-filtered least-squares problem on the
// (a-k+1)(b-k+1) x (k^2 J - 1) patch matrix with the self centre tap
// removed,  w = V diag(s / (s^2 + mu^2)) U^H b,  mu = tikhonov * s_max,
// which is algebraically the ridge solution (A^H A + mu^2 I) w = A^H b.  The
// same restatement runs on the host in host_spirit.cpp; here:
//   1. k_cal_gram: the Hermitian Gram of the augmented patch matrix
//      [features | centres] (nf + J columns) in 16 x 16 tiles, rows staged
//      through shared memory, one thread per entry (fixed summation order);
//   2. k_cal_solve, one CTA per target coil: the reduced Gram (column
//      centre_block + dst removed), s_max^2 by power iteration (the host's
//      stopping rule), the ridge shift, a left-looking Cholesky with the
//      factor stored column-major in HBM, column-oriented triangular solves,
//      and the scatter into SpiritKernels::raw() order (spirit.hpp:21-29).
// All reductions are CTA-local with a fixed order: deterministic.
#include "common.cuh"

#include <vector>

namespace shlr_b200 {

namespace {

constexpr int kGT = 16;       // Gram tile edge
constexpr int kGR = 32;       // rows per staged chunk
constexpr int kSolveNT = 512;

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__device__ __forceinline__ double2 zmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

struct CalGeom {
  int a, b, J, k, h, nf, nfa, nr, wc;  // wc = b - k + 1 windows per row
};

// Element (row, col) of the augmented patch matrix: col < nf is the
// neighbour (di, dj, src) of window row, col >= nf the centre of coil col - nf
// (spirit.cpp:45-60 ordering).
__device__ __forceinline__ double2 cal_elem(const double2* __restrict__ x, const CalGeom& g, int row, int col) {
  const int r = g.h + row / g.wc, c = g.h + row % g.wc;
  if (col >= g.nf) return __ldg(x + ((long long)r * g.b + c) * g.J + (col - g.nf));
  const int s = col % g.J, tap = col / g.J;
  const int di = tap / g.k, dj = tap % g.k;
  return __ldg(x + ((long long)(r + di - g.h) * g.b + (c + dj - g.h)) * g.J + s);
}

__global__ void __launch_bounds__(kGT * kGT) k_cal_gram(const double2* __restrict__ x, CalGeom g,
                                                        double2* __restrict__ gram) {
  __shared__ double2 sp[kGR][kGT + 1], sq[kGR][kGT + 1];
  const int tx = threadIdx.x % kGT, ty = threadIdx.x / kGT;
  const int p0 = blockIdx.y * kGT, q0 = blockIdx.x * kGT;
  if (q0 + kGT <= p0) return;  // lower tiles: filled by symmetry
  double2 acc = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < g.nr; r0 += kGR) {
    for (int t = threadIdx.x; t < kGR * kGT; t += blockDim.x) {
      const int rr = t / kGT, cc = t % kGT;
      const int row = r0 + rr;
      const bool ok = row < g.nr;
      sp[rr][cc] = ok && p0 + cc < g.nfa ? cal_elem(x, g, row, p0 + cc) : make_double2(0.0, 0.0);
      sq[rr][cc] = ok && q0 + cc < g.nfa ? cal_elem(x, g, row, q0 + cc) : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < kGR; ++rr) {
      const double2 u = sp[rr][ty], v = sq[rr][tx];
      acc.x += u.x * v.x + u.y * v.y;  // conj(u) v
      acc.y += u.x * v.y - u.y * v.x;
    }
    __syncthreads();
  }
  const int p = p0 + ty, q = q0 + tx;
  if (p < g.nfa && q < g.nfa && q >= p) {
    gram[(long long)p * g.nfa + q] = acc;
    gram[(long long)q * g.nfa + p] = make_double2(acc.x, -acc.y);
  }
}

__device__ double block_sum_d(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

// One CTA per target coil.  M (n x n, column-major: M[j * n + i]) is this
// target's scratch for the reduced Gram and then its Cholesky factor.
__global__ void __launch_bounds__(kSolveNT) k_cal_solve(const double2* __restrict__ gram, CalGeom g,
                                                        double tikhonov, double2* __restrict__ scratch,
                                                        double2* __restrict__ weights, int* __restrict__ status) {
  extern __shared__ double2 sm_cal[];
  __shared__ double sh[33];
  __shared__ double s_scal[2];
  const int dst = blockIdx.x, tid = threadIdx.x, NT = blockDim.x;
  const int nfa = g.nfa, n = g.nf - 1;
  const int drop = (g.h * g.k + g.h) * g.J + dst;  // self centre tap column
  double2* M = scratch + (long long)dst * n * n;
  double2* v = sm_cal;          // n
  double2* rhs = v + n;         // n
  auto full = [&](int c) { return c < drop ? c : c + 1; };
  // reduced Gram (column-major == conj of row-major for a Hermitian matrix)
  for (long long t = tid; t < (long long)n * n; t += NT) {
    const int j = (int)(t / n), i = (int)(t % n);
    M[t] = gram[(long long)full(i) * nfa + full(j)];
  }
  for (int i = tid; i < n; i += NT) {
    rhs[i] = gram[(long long)full(i) * nfa + g.nf + dst];  // F^H centres
    v[i] = make_double2(1.0, 0.0);
  }
  __syncthreads();
  // s_max^2: power iteration with the host's rule (host_spirit.cpp)
  double lam = 0.0;
  double2* w = rhs + n;  // n
  for (int it = 0; it < 20000; ++it) {
    for (int i = tid; i < n; i += NT) {
      double2 s = make_double2(0.0, 0.0);
      for (int kk = 0; kk < n; ++kk) {
        const double2 mv = M[(long long)kk * n + i];  // = g[i][kk] (column kk of M, row i)
        s.x += mv.x * v[kk].x - mv.y * v[kk].y;
        s.y += mv.x * v[kk].y + mv.y * v[kk].x;
      }
      w[i] = s;
    }
    __syncthreads();
    double nv = 0.0, num = 0.0, nw = 0.0;
    for (int i = tid; i < n; i += NT) {
      nv += v[i].x * v[i].x + v[i].y * v[i].y;
      num += v[i].x * w[i].x + v[i].y * w[i].y;
      nw += w[i].x * w[i].x + w[i].y * w[i].y;
    }
    nv = block_sum_d(nv, sh);
    num = block_sum_d(num, sh);
    nw = sqrt(block_sum_d(nw, sh));
    const double rq = num / nv;
    if (nw == 0.0) {
      lam = 0.0;
      break;
    }
    for (int i = tid; i < n; i += NT) v[i] = make_double2(w[i].x / nw, w[i].y / nw);
    __syncthreads();
    if (it > 10 && fabs(rq - lam) <= 1e-15 * fabs(rq)) {
      lam = rq;
      break;
    }
    lam = rq;
  }
  const double mu2 = tikhonov * tikhonov * lam;
  for (int i = tid; i < n; i += NT) M[(long long)i * n + i].x += mu2;
  __syncthreads();
  // left-looking Cholesky: column j of L (rows i >= j) into M[j * n + i]
  for (int j = 0; j < n; ++j) {
    double dpart = 0.0;
    for (int kk = tid; kk < j; kk += NT) {
      const double2 l = M[(long long)kk * n + j];
      dpart += l.x * l.x + l.y * l.y;
    }
    const double dsum = block_sum_d(dpart, sh);
    if (tid == 0) {
      const double d = M[(long long)j * n + j].x - dsum;
      s_scal[0] = d > 0.0 ? sqrt(d) : -1.0;
    }
    __syncthreads();
    const double ljj = s_scal[0];
    if (!(ljj > 0.0)) {
      if (tid == 0) status[dst] = 1;
      return;
    }
    for (int i = j + 1 + tid; i < n; i += NT) {
      double2 s = M[(long long)j * n + i];
      for (int kk = 0; kk < j; ++kk) {
        const double2 a = M[(long long)kk * n + i], bj = M[(long long)kk * n + j];
        s.x -= a.x * bj.x + a.y * bj.y;  // a conj(bj)
        s.y -= a.y * bj.x - a.x * bj.y;
      }
      M[(long long)j * n + i] = make_double2(s.x / ljj, s.y / ljj);
    }
    if (tid == 0) M[(long long)j * n + j] = make_double2(ljj, 0.0);
    __syncthreads();
  }
  // L y = rhs (column-oriented), then L^H x = y
  for (int kk = 0; kk < n; ++kk) {
    const double lkk = M[(long long)kk * n + kk].x;
    const double2 yk = make_double2(rhs[kk].x / lkk, rhs[kk].y / lkk);
    __syncthreads();
    for (int i = kk + 1 + tid; i < n; i += NT) {
      const double2 l = M[(long long)kk * n + i];
      rhs[i].x -= l.x * yk.x - l.y * yk.y;
      rhs[i].y -= l.x * yk.y + l.y * yk.x;
    }
    if (tid == 0) rhs[kk] = yk;
    __syncthreads();
  }
  for (int i = n - 1; i >= 0; --i) {
    const double lii = M[(long long)i * n + i].x;
    const double2 xi = make_double2(rhs[i].x / lii, rhs[i].y / lii);
    __syncthreads();
    for (int kk = tid; kk < i; kk += NT) {
      const double2 l = M[(long long)kk * n + i];  // L[i][kk]; L^H[kk][i] = conj(l)
      rhs[kk].x -= l.x * xi.x + l.y * xi.y;
      rhs[kk].y -= l.x * xi.y - l.y * xi.x;
    }
    if (tid == 0) rhs[i] = xi;
    __syncthreads();
  }
  for (int c = tid; c < n; c += NT) {
    const int f = full(c);
    const int tap = f / g.J, src = f % g.J;
    weights[((long long)tap * g.J + src) * g.J + dst] = rhs[c];
  }
}

}  // namespace

// Host entry (C-ABI wrapper in capi.cu): returns false when a reduced Gram is
// not positive definite (the host path's failure mode).
bool spirit_calibrate_device(const double* acs, size_t a, size_t b, size_t j, size_t k, double tikhonov,
                             double* weights_out) {
  CalGeom g;
  g.a = (int)a;
  g.b = (int)b;
  g.J = (int)j;
  g.k = (int)k;
  g.h = (int)k / 2;
  g.nf = (int)(k * k * j);
  g.nfa = g.nf + (int)j;
  g.wc = (int)(b - k + 1);
  g.nr = (int)((a - k + 1) * (b - k + 1));
  const int n = g.nf - 1;
  cudaStream_t st;
  SHLR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double2 *x = nullptr, *gram = nullptr, *scr = nullptr, *w = nullptr;
  int* status = nullptr;
  const size_t nx = a * b * j, nw = k * k * j * j;
  SHLR_CUDA(cudaMallocAsync(&x, nx * sizeof(double2), st));
  SHLR_CUDA(cudaMallocAsync(&gram, (size_t)g.nfa * g.nfa * sizeof(double2), st));
  SHLR_CUDA(cudaMallocAsync(&scr, (size_t)j * n * n * sizeof(double2), st));
  SHLR_CUDA(cudaMallocAsync(&w, nw * sizeof(double2), st));
  SHLR_CUDA(cudaMallocAsync(&status, j * sizeof(int), st));
  SHLR_CUDA(cudaMemcpyAsync(x, acs, nx * sizeof(double2), cudaMemcpyHostToDevice, st));
  SHLR_CUDA(cudaMemsetAsync(w, 0, nw * sizeof(double2), st));
  SHLR_CUDA(cudaMemsetAsync(status, 0, j * sizeof(int), st));
  const int tiles = (g.nfa + kGT - 1) / kGT;
  k_cal_gram<<<dim3(tiles, tiles), kGT * kGT, 0, st>>>(x, g, gram);
  SHLR_LAUNCH_CHECK();
  const size_t smem = 3ull * n * sizeof(double2);
  if (smem > 48 * 1024)
    SHLR_CUDA(cudaFuncSetAttribute(k_cal_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_cal_solve<<<(unsigned)j, kSolveNT, smem, st>>>(gram, g, tikhonov, scr, w, status);
  SHLR_LAUNCH_CHECK();
  std::vector<int> hs(j);
  SHLR_CUDA(cudaMemcpyAsync(weights_out, w, nw * sizeof(double2), cudaMemcpyDeviceToHost, st));
  SHLR_CUDA(cudaMemcpyAsync(hs.data(), status, j * sizeof(int), cudaMemcpyDeviceToHost, st));
  SHLR_CUDA(cudaFreeAsync(x, st));
  SHLR_CUDA(cudaFreeAsync(gram, st));
  SHLR_CUDA(cudaFreeAsync(scr, st));
  SHLR_CUDA(cudaFreeAsync(w, st));
  SHLR_CUDA(cudaFreeAsync(status, st));
  SHLR_CUDA(cudaStreamSynchronize(st));
  SHLR_CUDA(cudaStreamDestroy(st));
  for (int s : hs)
    if (s) return false;
  return true;
}

}  // namespace shlr_b200
