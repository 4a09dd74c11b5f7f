// Centered unitary DFT on the device (proj/src/fft.cpp:91-140 semantics).
//
// The reference transform is fftshift(F(ifftshift(v)))/sqrt(N) with DC at
// floor(N/2) (fft.cpp:100-106).  For even N this equals
//   out[k] = (-1)^{N/2} (-1)^k / sqrt(N) * FFT((-1)^n v[n])[k],
// so power-of-two lengths run a Stockham radix-4/2 FFT in shared memory with
// the (-1)^n modulation folded into the load and the (-1)^k scale into the
// store.  Other lengths use a direct O(N^2) centered DFT (twiddle index
// (k - c)(n - c) mod N), which is what the reference's Bluestein path
// computes (fft.cpp:39-71).
//
// Data layout of a tile: buf[k * F + f], k in [0, N) along the transform,
// f in [0, F) the fibre -- the fibre index is the contiguous (inner) memory
// dimension, so tile loads/stores are coalesced.
#pragma once

#include "common.cuh"

namespace shlr_b200 {

struct FftTwiddles {
  const float2* tw = nullptr;  // tw[k] = exp(-2 pi i k / n), k < n (fp64-rounded)
  int n = 0;
  int logn = -1;               // >= 0 iff n is a power of two
};

// t -> (fibre f, row k) of an [n][F] tile; shifts when F is a power of two
// (lf = log2 F, or -1).
__device__ __forceinline__ int fib_log2(int F) { return (F & (F - 1)) == 0 ? __ffs(F) - 1 : -1; }
__device__ __forceinline__ void tile_idx(int t, int F, int lf, int& f, int& k) {
  if (lf >= 0) {
    f = t & (F - 1);
    k = t >> lf;
  } else {
    f = t % F;
    k = t / F;
  }
}

// Radix-4 butterfly on v[0..3]; forward uses w = -i.
template <bool INV>
__device__ __forceinline__ void dft4(float2& a, float2& b, float2& c, float2& d) {
  const float2 s0 = cadd(a, c), s1 = csub(a, c);
  const float2 s2 = cadd(b, d), s3 = csub(b, d);
  // forward: X1 = s1 - i s3, X3 = s1 + i s3 ; inverse swaps.
  const float2 is3 = make_float2(-s3.y, s3.x);  // i * s3
  a = cadd(s0, s2);
  c = csub(s0, s2);
  if (INV) {
    b = cadd(s1, is3);
    d = csub(s1, is3);
  } else {
    b = csub(s1, is3);
    d = cadd(s1, is3);
  }
}

__device__ __forceinline__ float2 twiddle(const float2* __restrict__ tw, int idx, bool inv) {
  float2 w = __ldg(tw + idx);
  return inv ? cconj(w) : w;
}

// In-smem Stockham FFT of F fibres of length n (power of two) held in `a`
// ([n][F]); `b` is scratch of the same size.  All threads of the block take
// part; returns the buffer that holds the (natural-order) result.  Starts
// and ends with the caller's __syncthreads() discipline: the caller must
// sync after filling `a`; this routine syncs after every stage.
template <bool INV>
__device__ float2* smem_fft_pow2(float2* a, float2* b, int n, int logn, int F,
                                 const float2* __restrict__ tw) {
  float2* in = a;
  float2* out = b;
  // fibre counts are powers of two in every caller: index math by shifts
  const bool fpow2 = (F & (F - 1)) == 0;
  const int lf = fpow2 ? __ffs(F) - 1 : 0;
  int lns = 0;  // log2 of the current span ns
  int rem = logn;
  while (rem > 0) {
    const int ns = 1 << lns;
    if (rem >= 2) {
      const int nb = n >> 2;
      const int sshift = logn - lns - 2;  // n / (ns * 4) = 1 << sshift
      for (int t = threadIdx.x; t < nb * F; t += blockDim.x) {
        const int f = fpow2 ? (t & (F - 1)) : t % F;
        const int j = fpow2 ? (t >> lf) : t / F;
        const int k = j & (ns - 1);
        const int step = k << sshift;
        float2 v0 = in[(j)*F + f];
        float2 v1 = in[(j + nb) * F + f];
        float2 v2 = in[(j + 2 * nb) * F + f];
        float2 v3 = in[(j + 3 * nb) * F + f];
        if (ns > 1) {
          v1 = cmul(v1, twiddle(tw, step, INV));
          v2 = cmul(v2, twiddle(tw, 2 * step, INV));
          v3 = cmul(v3, twiddle(tw, 3 * step, INV));
        }
        dft4<INV>(v0, v1, v2, v3);
        const int d0 = ((j >> lns) << (lns + 2)) + k;
        out[(d0)*F + f] = v0;
        out[(d0 + ns) * F + f] = v1;
        out[(d0 + 2 * ns) * F + f] = v2;
        out[(d0 + 3 * ns) * F + f] = v3;
      }
      lns += 2;
      rem -= 2;
    } else {
      const int nb = n >> 1;
      const int sshift = logn - lns - 1;
      for (int t = threadIdx.x; t < nb * F; t += blockDim.x) {
        const int f = fpow2 ? (t & (F - 1)) : t % F;
        const int j = fpow2 ? (t >> lf) : t / F;
        const int k = j & (ns - 1);
        const int step = k << sshift;
        float2 v0 = in[(j)*F + f];
        float2 v1 = in[(j + nb) * F + f];
        if (ns > 1) v1 = cmul(v1, twiddle(tw, step, INV));
        const int d0 = ((j >> lns) << (lns + 1)) + k;
        out[(d0)*F + f] = cadd(v0, v1);
        out[(d0 + ns) * F + f] = csub(v0, v1);
      }
      lns += 1;
      rem -= 1;
    }
    __syncthreads();
    float2* t = in;
    in = out;
    out = t;
  }
  return in;
}

// Direct centered DFT (any n): out[k] = sum_m in[m] w^{(k-c)(m-c)}, no scale.
template <bool INV>
__device__ float2* smem_dft_direct(float2* a, float2* b, int n, int F,
                                   const float2* __restrict__ tw) {
  const int c = n / 2;
  for (int t = threadIdx.x; t < n * F; t += blockDim.x) {
    const int f = t % F, k = t / F;
    float2 acc = make_float2(0.f, 0.f);
    const int kc = ((k - c) % n + n) % n;
    int idx = (int)(((long long)kc * (long long)((n - c) % n)) % n);  // m = 0
    for (int m = 0; m < n; ++m) {
      cfma(acc, a[m * F + f], twiddle(tw, idx, INV));
      idx += kc;
      if (idx >= n) idx -= n;
    }
    b[k * F + f] = acc;
  }
  __syncthreads();
  return b;
}

// Scale applied on the store side of a centered unitary transform.
__device__ __forceinline__ float centered_out_scale(int k, int n, int logn, float inv_sqrt_n) {
  if (logn < 0) return inv_sqrt_n;
  // (-1)^{n/2} (-1)^k / sqrt(n)
  const int sgn = ((n >> 1) + k) & 1;
  return sgn ? -inv_sqrt_n : inv_sqrt_n;
}
__device__ __forceinline__ float centered_in_sign(int m, int logn) {
  if (logn < 0) return 1.f;
  return (m & 1) ? -1.f : 1.f;
}

// Full centered transform of a tile that the caller has loaded RAW into `a`
// (the caller need not modulate): applies the input modulation in place,
// transforms, and returns the result buffer; the caller multiplies element k
// by centered_out_scale(k, ...) on the way out.
template <bool INV>
__device__ float2* smem_centered_dft(float2* a, float2* b, const FftTwiddles& tw, int F) {
  const int n = tw.n;
  if (tw.logn >= 0) {
    const bool fpow2 = (F & (F - 1)) == 0;
    const int lf = fpow2 ? __ffs(F) - 1 : 0;
    for (int t = threadIdx.x; t < n * F; t += blockDim.x) {
      const int m = fpow2 ? (t >> lf) : t / F;
      if (m & 1) a[t] = make_float2(-a[t].x, -a[t].y);
    }
    __syncthreads();
    return smem_fft_pow2<INV>(a, b, n, tw.logn, F, tw.tw);
  }
  __syncthreads();
  return smem_dft_direct<INV>(a, b, n, F, tw.tw);
}

// ------------------------------------------------------------ generic kernel
// Transform along the middle axis of a tensor viewed as [outer][n][inner]
// with a user Op providing load(o, k, i) and store(o, k, i, v).  Grid:
// x = inner tiles of F fibres, y = outer.  Dynamic smem: 2 * n * F float2.
// Threads of the smem-FFT kernels: 512 gives one radix-4 butterfly per
// thread for an 8-fibre tile of length 256 and doubles the resident warps
// per SM over 256 (these kernels are latency-bound, their data L2-resident).
constexpr int kFftThreads = 512;

template <class Op, bool INV>
__global__ void __launch_bounds__(kFftThreads) fft_axis_kernel(Op op, FftTwiddles tw, int outer,
                                                       int inner, int F) {
  extern __shared__ float2 fft_smem[];
  if (op.skip()) return;
  const int n = tw.n;
  float2* a = fft_smem;
  float2* b = fft_smem + (size_t)n * F;
  const int o = blockIdx.y;
  const int i0 = blockIdx.x * F;
  const int lf = fib_log2(F);
#pragma unroll 4
  for (int t = threadIdx.x; t < n * F; t += blockDim.x) {
    int f, k;
    tile_idx(t, F, lf, f, k);
    const int i = i0 + f;
    a[t] = (i < inner) ? op.load(o, k, i) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float2* r = smem_centered_dft<INV>(a, b, tw, F);
  const float isn = rsqrtf((float)n);
  for (int t = threadIdx.x; t < n * F; t += blockDim.x) {
    int f, k;
    tile_idx(t, F, lf, f, k);
    const int i = i0 + f;
    if (i < inner) op.store(o, k, i, cscale(r[t], centered_out_scale(k, n, tw.logn, isn)));
  }
}

// Plain strided op: in/out element (o, k, i) at base + o*so + k*sk + i*si.
struct StridedCopyOp {
  const float2* in;
  float2* out;
  long long so, sk, si;
  __device__ bool skip() const { return false; }
  __device__ float2 load(int o, int k, int i) const { return in[o * so + k * sk + i * si]; }
  __device__ void store(int o, int k, int i, float2 v) const { out[o * so + k * sk + i * si] = v; }
};

// Host-side: twiddle table (fp64 computed, rounded to fp32).
FftTwiddles make_twiddles(int n, float2** dev_storage, cudaStream_t stream);

template <class Op, bool INV>
void launch_fft_axis(const Op& op, const FftTwiddles& tw, int outer, int inner, int F,
                     cudaStream_t stream) {
  const size_t smem = 2 * (size_t)tw.n * F * sizeof(float2);
  static bool configured = false;
  if (!configured) {
    SHLR_CUDA(cudaFuncSetAttribute(fft_axis_kernel<Op, INV>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  dim3 grid((inner + F - 1) / F, outer);
  fft_axis_kernel<Op, INV><<<grid, kFftThreads, smem, stream>>>(op, tw, outer, inner, F);
  SHLR_LAUNCH_CHECK();
}

// Pick the fibre count of a tile: at least `min_f`, a multiple of `mult`,
// keeping 2*n*F*8 bytes under ~64 KB.
inline int pick_fibres(int n, int inner, int mult) {
  int f = mult;
  while (f * 2 <= 32 && 2LL * n * (f * 2) * 8 <= 64 * 1024 && f * 2 <= ((inner + mult - 1) / mult) * mult)
    f *= 2;
  return f;
}

}  // namespace shlr_b200
