// Microbenchmark of the subspace solver's in-CTA Householder QR (profiling
// helper, not product code): one CTA per 120 x 48 block, clock64 per phase,
// orthogonality check of Q.   nvcc ... -o qr_bench scripts/qr_bench.cu
#include "../paper_2107_11650_b200/csrc/hankel_svt.cu"
#include <cstdio>
#include <vector>

namespace shlr_b200 {
template <int KB, int KS, int DP>
__device__ void qr_exp(float2* M, float2* Q, int d, float* tau, int mode, long long* ck) {
  constexpr int T = DP / 8;
  const int g = threadIdx.x >> 3, s = threadIdx.x & 7;
  const int k = g;
  const bool act = k < KB;
  float2 col[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int row = s + 8 * t;
    col[t] = (act && row < d) ? M[row * KS + k] : make_float2(0.f, 0.f);
  }
  // every group computes the reflector of its own column at pivot j (uniform
  // control flow, full-mask shuffles); only the owner (k == j) stores it
  auto reflect = [&](int j) {
    float ss = 0.f;
    float2 x0 = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + 8 * t;
      const float2 c = row >= j ? col[t] : make_float2(0.f, 0.f);
      ss = fmaf(c.x, c.x, fmaf(c.y, c.y, ss));
      if (row == j) x0 = col[t];
    }
    ss = group8_sum(ss);
    x0.x = group8_sum(x0.x);  // only one lane of the group holds row j
    x0.y = group8_sum(x0.y);
    const float nrm = sqrtf(ss);
    const float ax0 = sqrtf(x0.x * x0.x + x0.y * x0.y);
    float tj = 0.f;
    float2 inv_v0 = make_float2(0.f, 0.f);
    if (nrm > 0.f) {
      const float r0 = ax0 > 0.f ? __frcp_rn(ax0) : 0.f;
      const float2 ph = ax0 > 0.f ? make_float2(x0.x * r0, x0.y * r0) : make_float2(1.f, 0.f);
      const float rn0 = __frcp_rn(ax0 + nrm);
      inv_v0 = make_float2(ph.x * rn0, -ph.y * rn0);
      tj = 1.f + ax0 * __frcp_rn(nrm);
    }
    if (k == j) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int row = s + 8 * t;
        if (row > j && row < d) M[row * KS + j] = cmul(col[t], inv_v0);
      }
      if (s == 0) tau[j] = tj;
    }
  };
  reflect(0);
  __syncthreads();
  for (int j = 0; j < KB; ++j) {
    float2 part = make_float2(0.f, 0.f);
    float2 v[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + 8 * t;
      v[t] = (row > j && row < d) ? M[row * KS + j] : make_float2(row == j ? 1.f : 0.f, 0.f);
      cfmac(part, v[t], col[t]);
    }
    part.x = group8_sum(part.x);
    part.y = group8_sum(part.y);
    const float2 tw = (act && k > j) ? cscale(part, tau[j]) : make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < T; ++t) col[t] = csub(col[t], cmul(v[t], tw));
    if (j + 1 < KB) reflect(j + 1);
    __syncthreads();
  }
  if (threadIdx.x == 0) ck[0] = clock64();
  if (mode & 1) return;
#pragma unroll
  for (int t = 0; t < T; ++t) col[t] = make_float2(s + 8 * t == k ? 1.f : 0.f, 0.f);
  for (int j = KB - 1; j >= 0; --j) {
    float2 part = make_float2(0.f, 0.f);
    float2 v[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + 8 * t;
      v[t] = (row > j && row < d) ? M[row * KS + j] : make_float2(row == j ? 1.f : 0.f, 0.f);
      cfmac(part, v[t], col[t]);
    }
    part.x = group8_sum(part.x);
    part.y = group8_sum(part.y);
    const float2 tw = (act && k >= j) ? cscale(part, tau[j]) : make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < T; ++t) col[t] = csub(col[t], cmul(v[t], tw));
  }
  if (act) {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + 8 * t;
      if (row < DP) Q[row * KS + k] = row < d ? col[t] : make_float2(0.f, 0.f);
    }
  }
}

template <int DP, int KB>
__global__ void __launch_bounds__(kSubNT, 1) qr_kernel(const float2* in, float2* out, long long* clk, int d, int mode) {
  constexpr int KS = KB + 1;
  extern __shared__ __align__(16) unsigned char sm[];
  float2* M = reinterpret_cast<float2*>(sm);
  float2* Q = M + DP * KS;
  float* tau = reinterpret_cast<float*>(Q + DP * KS);
  const float2* src = in + (long long)blockIdx.x * DP * KB;
  for (int t = threadIdx.x; t < DP * KB; t += kSubNT) M[(t / KB) * KS + t % KB] = src[t];
  __syncthreads();
  long long t0 = clock64();
  __shared__ long long ck[1];
  if (mode < 0) householder_qr<KB, KS, DP>(M, Q, d, tau); else qr_exp<KB, KS, DP>(M, Q, d, tau, mode, ck);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { clk[2 * blockIdx.x] = t1 - t0; clk[2 * blockIdx.x + 1] = mode < 0 ? 0 : ck[0] - t0; }
  for (int t = threadIdx.x; t < DP * KB; t += kSubNT) out[(long long)blockIdx.x * DP * KB + t] = Q[(t / KB) * KS + t % KB];
}
}  // namespace shlr_b200

int main() {
  using namespace shlr_b200;
  constexpr int DP = 120, KB = 48, NB = 148;
  const int d = 120;
  std::vector<float2> h((size_t)NB * DP * KB);
  unsigned s = 1;
  for (auto& v : h) {
    s = s * 1664525u + 1013904223u; v.x = (s >> 8) / 16777216.f - 0.5f;
    s = s * 1664525u + 1013904223u; v.y = (s >> 8) / 16777216.f - 0.5f;
  }
  float2 *din, *dout; long long* dclk;
  cudaMalloc(&din, h.size() * 8); cudaMalloc(&dout, h.size() * 8); cudaMalloc(&dclk, 2 * NB * 8);
  cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = 2 * DP * (KB + 1) * 8 + KB * 4 + 64;
  cudaFuncSetAttribute(qr_kernel<DP, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode : {-1}) {
    for (int rep = 0; rep < 3; ++rep) qr_kernel<DP, KB><<<NB, kSubNT, smem>>>(din, dout, dclk, d, mode);
    cudaDeviceSynchronize();
    std::vector<long long> cc(2 * NB); cudaMemcpy(cc.data(), dclk, 2 * NB * 8, cudaMemcpyDeviceToHost);
    double m0 = 0, m1 = 0; for (int i = 0; i < NB; ++i) { m0 += cc[2 * i]; m1 += cc[2 * i + 1]; }
    printf("mode %d: total %.0f  factor-part %.0f cycles\n", mode, m0 / NB, m1 / NB);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<long long> c(NB, 0);
  std::vector<float2> q(h.size()); cudaMemcpy(q.data(), dout, q.size() * 8, cudaMemcpyDeviceToHost);
  double mean = 0; for (auto v : c) mean += v; mean /= NB;
  double err = 0;  // ||Q^H Q - I||_max of block 0
  for (int a = 0; a < KB; ++a) for (int b = 0; b < KB; ++b) {
    double re = 0, im = 0;
    for (int i = 0; i < d; ++i) { float2 x = q[i * KB + a], y = q[i * KB + b]; re += x.x * y.x + x.y * y.y; im += x.x * y.y - x.y * y.x; }
    re -= (a == b); err = std::max(err, std::sqrt(re * re + im * im));
  }
  // span check: || M - Q Q^H M ||_F / ||M||_F for block 0
  double num = 0, den = 0;
  for (int k = 0; k < KB; ++k) {
    std::vector<double> pr(KB * 2, 0.0);
    for (int a = 0; a < KB; ++a) for (int i = 0; i < d; ++i) { float2 x = q[i * KB + a], m = h[i * KB + k]; pr[2*a] += x.x * m.x + x.y * m.y; pr[2*a+1] += x.x * m.y - x.y * m.x; }
    for (int i = 0; i < d; ++i) {
      double re = h[i * KB + k].x, im = h[i * KB + k].y; den += re * re + im * im;
      for (int a = 0; a < KB; ++a) { float2 x = q[i * KB + a]; re -= x.x * pr[2*a] - x.y * pr[2*a+1]; im -= x.x * pr[2*a+1] + x.y * pr[2*a]; }
      num += re * re + im * im;
    }
  }
  (void)mean; printf("qr %d x %d: %.0f  orth err %.2e  span err %.2e\n", d, KB, mean, err, std::sqrt(num / den));
  return 0;
}
