// Microbenchmark + accuracy check of the subspace solver's Rayleigh-Ritz
// eigensolver (hermitian_eig_tridiag) on random 48 x 48 Hermitian matrices
// with a spread spectrum (profiling helper, not product code).
#include "../paper_2107_11650_b200/csrc/hankel_svt.cu"
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <vector>

namespace shlr_b200 {
template <int KB>
__global__ void __launch_bounds__(kSubNT, 1) eig_kernel(const float2* in, float2* uout, double* ev,
                                                       long long* clk, float care) {
  constexpr int KS = KB + 1;
  extern __shared__ __align__(16) unsigned char sm[];
  float2* H = reinterpret_cast<float2*>(sm);
  float2* C = H + KB * KS;              // 3 KB^2 floats of work (>= KB x KS float2)
  float* scr = reinterpret_cast<float*>(C + 2 * KB * KS);
  double* evs = reinterpret_cast<double*>(scr + 16 * KB);
  for (int t = threadIdx.x; t < KB * KB; t += kSubNT) H[(t / KB) * KS + t % KB] = in[(long long)blockIdx.x * KB * KB + t];
  __syncthreads();
  long long t0 = clock64();
  __shared__ long long ck[8];
  hermitian_eig_tridiag<KB, KS>(H, scr, reinterpret_cast<float*>(C), C, evs, care, ck);
  long long t1 = clock64();
  if (threadIdx.x == 0) { clk[blockIdx.x * 8] = t1 - t0; for (int i = 1; i < 7; ++i) clk[blockIdx.x * 8 + i] = ck[i] - ck[i - 1]; }
  for (int t = threadIdx.x; t < KB * KB; t += kSubNT) uout[(long long)blockIdx.x * KB * KB + t] = C[(t / KB) * KS + t % KB];
  for (int t = threadIdx.x; t < KB; t += kSubNT) ev[blockIdx.x * KB + t] = evs[t];
}
}  // namespace shlr_b200

int main() {
  using namespace shlr_b200;
  constexpr int KB = 48, NB = 148;
  // H = Q diag(lam) Q^H with Q from Gram-Schmidt of a random matrix, lam spread over 1e-6..1
  std::vector<double> hre((size_t)NB * KB * KB), him(hre.size());
  unsigned s = 7;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) / 16777216.0 - 0.5; };
  std::vector<float2> h(hre.size());
  for (int b = 0; b < NB; ++b) {
    std::vector<double> qr(KB * KB), qi(KB * KB);
    for (auto& v : qr) v = rnd();
    for (auto& v : qi) v = rnd();
    for (int c = 0; c < KB; ++c) {  // MGS on columns
      for (int p = 0; p < c; ++p) {
        double dr = 0, di = 0;
        for (int i = 0; i < KB; ++i) { dr += qr[i*KB+p]*qr[i*KB+c] + qi[i*KB+p]*qi[i*KB+c]; di += qr[i*KB+p]*qi[i*KB+c] - qi[i*KB+p]*qr[i*KB+c]; }
        for (int i = 0; i < KB; ++i) { qr[i*KB+c] -= dr*qr[i*KB+p] - di*qi[i*KB+p]; qi[i*KB+c] -= dr*qi[i*KB+p] + di*qr[i*KB+p]; }
      }
      double nn = 0; for (int i = 0; i < KB; ++i) nn += qr[i*KB+c]*qr[i*KB+c] + qi[i*KB+c]*qi[i*KB+c];
      nn = 1 / std::sqrt(nn); for (int i = 0; i < KB; ++i) { qr[i*KB+c] *= nn; qi[i*KB+c] *= nn; }
    }
    std::vector<double> lam(KB);
    for (int k = 0; k < KB; ++k) lam[k] = std::pow(10.0, -6.0 * k / (KB - 1)) * (b % 3 == 0 && k == 5 ? 0 : 1) + (b % 3 == 1 && k == 7 ? lam[k-1] : 0);
    if (b % 3 == 1) lam[7] = lam[6] * (1 + 1e-7);   // a near-degenerate pair
    for (int i = 0; i < KB; ++i) for (int j = 0; j < KB; ++j) {
      double r = 0, im = 0;
      for (int k = 0; k < KB; ++k) { r += lam[k] * (qr[i*KB+k]*qr[j*KB+k] + qi[i*KB+k]*qi[j*KB+k]); im += lam[k] * (qi[i*KB+k]*qr[j*KB+k] - qr[i*KB+k]*qi[j*KB+k]); }
      hre[(size_t)b*KB*KB + i*KB+j] = r; him[(size_t)b*KB*KB + i*KB+j] = im;
      h[(size_t)b*KB*KB + i*KB+j] = make_float2((float)r, (float)im);
    }
  }
  float2 *din, *dout; double* dev; long long* dclk;
  cudaMalloc(&din, h.size() * 8); cudaMalloc(&dout, h.size() * 8); cudaMalloc(&dev, NB * KB * 8); cudaMalloc(&dclk, NB * 64);
  cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)3 * KB * (KB + 1) * 8 + 16 * KB * 4 + KB * 8 + 64;
  cudaFuncSetAttribute(eig_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const float care = getenv("CARE") ? atof(getenv("CARE")) : 0.f;
  for (int rep = 0; rep < 3; ++rep) eig_kernel<KB><<<NB, kSubNT, smem>>>(din, dout, dev, dclk, care);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float2> u(h.size()); std::vector<double> ev(NB * KB); std::vector<long long> c(NB * 8);
  cudaMemcpy(u.data(), dout, u.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(ev.data(), dev, ev.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), dclk, NB * 64, cudaMemcpyDeviceToHost);
  double mc = 0, ph[8] = {0}; for (int b = 0; b < NB; ++b) { mc += c[b * 8]; for (int i = 1; i < 7; ++i) ph[i] += c[b * 8 + i]; } mc /= NB;
  printf("phases: tridiag %.0f  similarity %.0f  bisection %.0f  twisted %.0f  mgs %.0f  backtransform %.0f\n", ph[1]/NB, ph[2]/NB, ph[3]/NB, ph[4]/NB, ph[5]/NB, ph[6]/NB);
  double worst_res = 0, worst_orth = 0; int unsorted = 0, bad = 0;
  for (int b = 0; b < NB; ++b) {
    const double* Hr = &hre[(size_t)b*KB*KB]; const double* Hi = &him[(size_t)b*KB*KB];
    const float2* U = &u[(size_t)b*KB*KB];
    for (int k = 0; k < KB; ++k) {
      if (k && ev[b*KB+k] > ev[b*KB+k-1]) ++unsorted;
      double rn = 0;
      for (int i = 0; i < KB; ++i) {
        double r = 0, im = 0;
        for (int j = 0; j < KB; ++j) { r += Hr[i*KB+j]*U[j*KB+k].x - Hi[i*KB+j]*U[j*KB+k].y; im += Hr[i*KB+j]*U[j*KB+k].y + Hi[i*KB+j]*U[j*KB+k].x; }
        r -= ev[b*KB+k] * U[i*KB+k].x; im -= ev[b*KB+k] * U[i*KB+k].y; rn += r*r + im*im;
      }
      if (ev[b*KB+k] < care) continue;  // tail below `care`: any orthonormal basis
      if (std::sqrt(rn) > 1e-4 && bad < 6) { printf("bad: mat %d (class %d) k %d res %.2e ev %.3e\n", b, b % 3, k, std::sqrt(rn), ev[b*KB+k]); ++bad; }
      worst_res = std::max(worst_res, std::sqrt(rn));   // relative to ||H|| = 1
      for (int l = 0; l < KB; ++l) {
        double r = 0, im = 0;
        for (int i = 0; i < KB; ++i) { r += U[i*KB+k].x*U[i*KB+l].x + U[i*KB+k].y*U[i*KB+l].y; im += U[i*KB+k].x*U[i*KB+l].y - U[i*KB+k].y*U[i*KB+l].x; }
        r -= (k == l); worst_orth = std::max(worst_orth, std::sqrt(r*r + im*im));
      }
    }
  }
  printf("eig %d: %.0f cycles/CTA  max residual ||Hu - lam u|| %.2e (||H||=1)  max |U^H U - I| %.2e  unsorted %d  ev0 %.6f ev1 %.6f\n",
         KB, mc, worst_res, worst_orth, unsorted, ev[0], ev[1]);
  return 0;
}
