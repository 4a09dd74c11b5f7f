// Subspace Hankel-SVT solver (see hankel_svt.cuh): block subspace iteration
// with Householder QR, Rayleigh-Ritz by tridiagonalisation + multisection,
// the fused Z / dual / adjoint epilogue, the large-d variants and the
// deflation chain.  The kernel template is instantiated per dimension class
// in svt_sub_small.cu (d <= 128), svt_sub_big.cu (128 < d <= 248) and
// svt_sub_huge.cu (248 < d <= 496) so the three build in parallel.
#pragma once
#include "svt_device.cuh"
#include "svt_mma.cuh"

namespace shlr_b200 {

// ============================================================================
// Subspace SVT solver
// ============================================================================
namespace {

constexpr int kSubNT = 512;  // threads of the subspace kernel (16 warps)

__device__ __forceinline__ float hash_unit(unsigned int x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return (float)(x >> 8) * (2.0f / 16777216.0f) - 1.0f;
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Householder vector of column j of M (rows j..d-1): v_j = 1 implicit, rows
// > j overwritten by v, tau[j] set.  Executed by one warp.
template <int KS>
__device__ __forceinline__ void householder_prep(float2* M, int d, int j, float* tau) {
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  for (int i = j + lane; i < d; i += 32) {
    const float2 x = M[i * KS + j];
    s = fmaf(x.x, x.x, fmaf(x.y, x.y, s));
  }
  s = warp_sum_f(s);
  const float nrm = sqrtf(s);
  const float2 x0 = M[j * KS + j];
  const float ax0 = hypotf(x0.x, x0.y);
  float t = 0.f;
  float2 inv_v0 = make_float2(0.f, 0.f);
  if (nrm > 0.f) {
    const float2 ph = ax0 > 0.f ? make_float2(x0.x / ax0, x0.y / ax0) : make_float2(1.f, 0.f);
    const float2 alpha = make_float2(-ph.x * nrm, -ph.y * nrm);
    const float2 v0 = csub(x0, alpha);        // = ph (|x0| + nrm)
    const float n0 = ax0 + nrm;
    inv_v0 = make_float2(ph.x / n0, -ph.y / n0);  // 1 / v0
    t = 1.f + ax0 / nrm;                      // (alpha - x0) / alpha, real
    (void)v0;
  }
  __syncwarp();
  for (int i = j + 1 + lane; i < d; i += 32) M[i * KS + j] = cmul(M[i * KS + j], inv_v0);
  if (lane == 0) tau[j] = t;
  __syncwarp();
}

__device__ __forceinline__ float group8_sum(float v, unsigned mask = 0xffffffffu) {
  v += __shfl_xor_sync(mask, v, 4);
  v += __shfl_xor_sync(mask, v, 2);
  v += __shfl_xor_sync(mask, v, 1);
  return v;
}
// sum over aligned groups of GS lanes (GS = 8 or 16)
template <int GS>
__device__ __forceinline__ float group_sum(float v) {
  if (GS >= 16) v += __shfl_xor_sync(0xffffffffu, v, 8);
  return group8_sum(v);
}

// Yc (R x ncols, row stride KS) = C B (scaled by column), one output per
// thread (the HUGE variant's 16-row chunk, no room for split-k buffers): a
// warp holds one row and 32 consecutive columns, so C[r][k] is a broadcast
// and B[k][c..c+31] one conflict-free row.  Ends with a barrier.
template <int CS, int KS, int R>
__device__ __forceinline__ void chunk_block_huge(const float2* C, const float2* Bm, float2* Yc, int d, int ncols,
                                                 const float* scale) {
  static_assert(kSubNT % R == 0, "threads per row");
  constexpr int TPR = kSubNT / R;
  const int r = threadIdx.x / TPR, c0 = threadIdx.x % TPR;
  for (int c = c0; c < ncols; c += TPR) {
    float2 y0 = make_float2(0.f, 0.f), y1 = make_float2(0.f, 0.f);
    const float2* cr = C + r * CS;
    int k = 0;
#pragma unroll 4
    for (; k + 1 < d; k += 2) {
      cfma(y0, cr[k], Bm[k * KS + c]);
      cfma(y1, cr[k + 1], Bm[(k + 1) * KS + c]);
    }
    if (k < d) cfma(y0, cr[k], Bm[k * KS + c]);
    Yc[r * KS + c] = cscale(cadd(y0, y1), scale ? scale[c] : 1.f);
  }
  __syncthreads();
}

// Q (rows < d, KB orthonormal columns, stride KS) of the Householder QR of M
// (DP x KB, rows >= d zero); M is destroyed: column j receives the full
// reflector v_j (0 above row j, 1 at row j), so the apply loops carry no
// per-row predicates.
//
// Each column is owned by a group of 8 threads for the whole factorisation
// and held in registers (rows s + 8t); warp w owns columns 4w..4w+3, so warps
// whose columns are finished (or do not exist) skip a step as a whole.  Step
// j: every owner of a column k > j applies reflector j; the warp owning
// column j+1 then forms reflector j+1 from its registers -- one CTA barrier
// per column.  Forming Q applies the stored reflectors backwards to
// register-resident columns of the identity, with no barrier at all.
template <int KB, int KS, int DP, int GS = 8>
__device__ void householder_qr(float2* M, float2* Q, int d, float* tau) {
  constexpr int T = DP / GS;       // rows per thread
  constexpr int CPW = 32 / GS;     // columns per warp
  const int g = threadIdx.x / GS, s = threadIdx.x % GS;
  static_assert(kSubNT / GS >= KB, "one GS-thread group per column");
  static_assert(DP % GS == 0, "DP multiple of GS");
  const int w = g / CPW;
  const int k = g;                 // this group's column
  const bool act = k < KB;
  const bool warp_act = CPW * w < KB;
  float2 col[T];
#pragma unroll
  for (int t = 0; t < T; ++t) col[t] = act ? M[(s + GS * t) * KS + k] : make_float2(0.f, 0.f);
  // executed by a whole warp (full-mask shuffles); the group owning column j
  // stores reflector j
  auto reflect = [&](int j) {
    float ss = 0.f;
    float2 x0 = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + GS * t;
      if (row >= j) ss = fmaf(col[t].x, col[t].x, fmaf(col[t].y, col[t].y, ss));
      if (row == j) x0 = col[t];
    }
    ss = group_sum<GS>(ss);
    x0.x = group_sum<GS>(x0.x);  // one lane of the group holds row j
    x0.y = group_sum<GS>(x0.y);
    const float nrm = sqrtf(ss);
    const float ax0 = sqrtf(fmaf(x0.x, x0.x, x0.y * x0.y));
    float tj = 0.f;
    float2 inv_v0 = make_float2(0.f, 0.f);
    if (nrm > 0.f) {
      const float2 ph = ax0 > 0.f ? make_float2(x0.x / ax0, x0.y / ax0) : make_float2(1.f, 0.f);
      const float rn0 = 1.f / (ax0 + nrm);          // v0 = x0 - alpha = ph (|x0| + nrm)
      inv_v0 = make_float2(ph.x * rn0, -ph.y * rn0);  // 1 / v0
      tj = 1.f + ax0 / nrm;                           // (alpha - x0) / alpha, real
    }
    if (k == j) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int row = s + GS * t;
        M[row * KS + j] = row > j ? cmul(col[t], inv_v0) : make_float2(row == j ? 1.f : 0.f, 0.f);
      }
      if (s == 0) tau[j] = tj;
    }
  };
  if (w == 0) reflect(0);
  __syncthreads();
  for (int j = 0; j < KB; ++j) {
    if (warp_act && CPW * w + CPW - 1 > j) {  // warp-uniform: some column k > j in this warp
      float2 part = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < T; ++t) cfmac(part, M[(s + GS * t) * KS + j], col[t]);  // sum conj(v) col
      part.x = group_sum<GS>(part.x);
      part.y = group_sum<GS>(part.y);
      const float2 tw = (act && k > j) ? cscale(part, tau[j]) : make_float2(0.f, 0.f);
      // the reflector is read again rather than kept: half the registers
      // (two CTAs per SM at 64 registers need it)
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float2 v = M[(s + GS * t) * KS + j];
        col[t].x -= v.x * tw.x - v.y * tw.y;
        col[t].y -= v.x * tw.y + v.y * tw.x;
      }
      if (j + 1 < KB && w == (j + 1) / CPW) reflect(j + 1);
    }
    __syncthreads();
  }
  // explicit Q = H_0 ... H_{KB-1} [I; 0]: column k of the identity, reflectors
  // backwards (H_j leaves e_k alone for j > k)
#pragma unroll
  for (int t = 0; t < T; ++t) col[t] = make_float2(s + GS * t == k ? 1.f : 0.f, 0.f);
  if (warp_act) {
    for (int j = min(CPW * w + CPW - 1, KB - 1); j >= 0; --j) {
      float2 part = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < T; ++t) cfmac(part, M[(s + GS * t) * KS + j], col[t]);
      part.x = group_sum<GS>(part.x);
      part.y = group_sum<GS>(part.y);
      const float2 tw = (act && k >= j) ? cscale(part, tau[j]) : make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float2 v = M[(s + GS * t) * KS + j];
        col[t].x -= v.x * tw.x - v.y * tw.y;
        col[t].y -= v.x * tw.y + v.y * tw.x;
      }
    }
  }
  if (M == Q) __syncthreads();  // in place: every warp is done reading the reflectors
  if (act) {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + GS * t;
      Q[row * KS + k] = row < d ? col[t] : make_float2(0.f, 0.f);
    }
  }
}

// Eigen-decomposition of the n x n Hermitian Rayleigh-Ritz matrix H (full
// storage in smem, stride KS, destroyed) for the subspace solver:
//   1. Householder tridiagonalisation H = Q T Q^H (one reflector per column,
//      3 CTA barriers per column; reflectors kept in H's columns);
//   2. a diagonal phase similarity makes T real symmetric tridiagonal;
//   3. eigenvalues by multisection on Sturm counts, 8 threads per eigenvalue
//      (9 sub-intervals per step, 8 steps: FP32 resolution);
//   4. eigenvectors of T by the twisted factorisation (one thread per
//      eigenvalue); members of clusters above `care` rebuilt by inverse
//      iteration with reorthogonalisation; modified Gram-Schmidt in
//      descending order;
//   5. back-transform through the phases and the stored reflectors, one
//      8-thread group per eigenvector held in registers (no barriers).
// Out: evals[k] descending, U[i * KS + k] the matching unit eigenvectors.
// scr: >= 12 n floats; work: >= 3 n n floats, may alias U (dead before U is
// written).  Runs on kSubNT threads; ~ (3 n + 60) barriers in total.
template <int n, int KS>
__device__ void hermitian_eig_tridiag(float2* H, float* scr, float* work, float2* U, double* evals,
                                      float care = 0.f, long long* clk = nullptr, int orth_mode = 0) {
#define EIG_STAMP(k) \
  if (clk && threadIdx.x == 0) clk[k] = clock64()
  EIG_STAMP(0);
  static_assert(n % 8 == 0 && n <= 64, "n must be a multiple of 8, <= 64");
  constexpr int NT = kSubNT;
  constexpr int CU = n / 8;  // columns (rows) per thread in the 8-thread-group mappings
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float2* vbuf = reinterpret_cast<float2*>(scr);  // n: current reflector
  float2* pbuf = vbuf + n;                         // n: p = tau A v
  float2* ph = pbuf + n;                           // n: phases of the real similarity
  float2* ee = ph + n;                             // n: complex subdiagonal of T
  float* dd = reinterpret_cast<float*>(ee + n);    // n: diagonal of T
  float* bb = dd + n;                              // n: |subdiagonal|
  float* b2 = bb + n;                              // n: |subdiagonal|^2
  float* th = b2 + n;                              // n: reflector tau

  // ---------------------------------------------------------- 1. tridiagonalise
  const int gi = tid >> 3, gs = tid & 7;  // row-group mapping: row j+1+gi, columns j+1+gs+8u
  for (int j = 0; j < n - 2; ++j) {
    if (warp == 0) {
      const int i0 = j + 1 + lane, i1 = i0 + 32;
      const float2 xa = i0 < n ? H[i0 * KS + j] : make_float2(0.f, 0.f);
      const float2 xb = i1 < n ? H[i1 * KS + j] : make_float2(0.f, 0.f);
      float ss = fmaf(xa.x, xa.x, fmaf(xa.y, xa.y, fmaf(xb.x, xb.x, xb.y * xb.y)));
      ss = warp_sum_f(ss);
      const float2 x0 = make_float2(__shfl_sync(0xffffffffu, xa.x, 0), __shfl_sync(0xffffffffu, xa.y, 0));
      const float nrm = sqrtf(ss);
      const float ax0 = sqrtf(fmaf(x0.x, x0.x, x0.y * x0.y));
      float tj = 0.f;
      float2 alpha = make_float2(0.f, 0.f), inv_v0 = make_float2(0.f, 0.f);
      if (nrm > 0.f) {
        const float2 phs = ax0 > 0.f ? make_float2(x0.x / ax0, x0.y / ax0) : make_float2(1.f, 0.f);
        alpha = make_float2(-phs.x * nrm, -phs.y * nrm);
        const float rn0 = 1.f / (ax0 + nrm);
        inv_v0 = make_float2(phs.x * rn0, -phs.y * rn0);
        tj = 1.f + ax0 / nrm;
      }
      if (i0 < n) {
        const float2 v = i0 == j + 1 ? make_float2(1.f, 0.f) : cmul(xa, inv_v0);
        vbuf[i0] = v;
        H[i0 * KS + j] = v;
      }
      if (i1 < n) {
        const float2 v = cmul(xb, inv_v0);
        vbuf[i1] = v;
        H[i1 * KS + j] = v;
      }
      if (lane == 0) {
        th[j] = tj;
        ee[j] = alpha;
      }
    }
    __syncthreads();
    const float tj = th[j];
    {  // p = tau A v, A = H[j+1:, j+1:]
      const int i = j + 1 + gi;
      float2 part = make_float2(0.f, 0.f);
      if (i < n) {
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int c = j + 1 + gs + 8 * u;
          if (c < n) cfma(part, H[i * KS + c], vbuf[c]);
        }
      }
      part.x = group8_sum(part.x);
      part.y = group8_sum(part.y);
      if (i < n && gs == 0) pbuf[i] = cscale(part, tj);
    }
    __syncthreads();
    float kk;  // K = (tau / 2) v^H p (real for Hermitian A)
    {
      float t = 0.f;
      for (int i = j + 1 + lane; i < n; i += 32) {
        const float2 v = vbuf[i], pv = pbuf[i];
        t = fmaf(v.x, pv.x, fmaf(v.y, pv.y, t));
      }
      kk = 0.5f * tj * warp_sum_f(t);
    }
    {  // A -= v w^H + w v^H, w = p - K v
      const int i = j + 1 + gi;
      if (i < n) {
        const float2 vi = vbuf[i];
        const float2 wi = csub(pbuf[i], cscale(vi, kk));
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int c = j + 1 + gs + 8 * u;
          if (c < n) {
            const float2 vc = vbuf[c];
            const float2 wc = csub(pbuf[c], cscale(vc, kk));
            float2 a = H[i * KS + c];
            // a -= vi conj(wc) + wi conj(vc)
            a.x -= vi.x * wc.x + vi.y * wc.y + wi.x * vc.x + wi.y * vc.y;
            a.y -= vi.y * wc.x - vi.x * wc.y + wi.y * vc.x - wi.x * vc.y;
            H[i * KS + c] = a;
          }
        }
      }
    }
    __syncthreads();
  }
  if (tid < n) dd[tid] = H[tid * KS + tid].x;
  if (tid == 0) ee[n - 2] = H[(n - 1) * KS + (n - 2)];
  __syncthreads();
  // reflector columns j <= n-3: zero above row j+1 (row j+1 already holds 1)
  for (int t = tid; t < n * n; t += NT) {
    const int i = t / n, c = t - i * n;
    if (c <= n - 3 && i <= c) H[i * KS + c] = make_float2(0.f, 0.f);
  }
  EIG_STAMP(1);
  // ---------------------------------------------------------- 2. real similarity
  if (tid < n) {  // |e_j| and the unit factors e_j / |e_j| in parallel
    const float2 e = tid < n - 1 ? ee[tid] : make_float2(0.f, 0.f);
    const float a = sqrtf(fmaf(e.x, e.x, e.y * e.y));
    bb[tid] = a;
    b2[tid] = a * a;
    const float ia = a > 0.f ? 1.f / a : 0.f;
    ee[tid] = a > 0.f ? make_float2(e.x * ia, e.y * ia) : make_float2(1.f, 0.f);
  }
  __syncthreads();
  if (tid == 0) {  // phases: prefix products of the unit factors
    float2 p = make_float2(1.f, 0.f);
    ph[0] = p;
    for (int j = 0; j < n - 1; ++j) {
      p = cmul(p, ee[j]);
      ph[j + 1] = p;
    }
  }
  __syncthreads();
  EIG_STAMP(2);
  // ---------------------------------------------------------- 3. eigenvalues (multisection)
  float maxb2 = 0.f;
  for (int i = 0; i < n - 1; ++i) maxb2 = fmaxf(maxb2, b2[i]);
  const float pivmin = 1.0e-30f * fmaxf(1.f, maxb2);
  {
    const int g = gi, s = gs, l = g & 3;
    const bool act = g < n;
    float lo = 3.0e38f, hi = -3.0e38f;
    for (int i = s; i < n; i += 8) {
      const float r = (i > 0 ? bb[i - 1] : 0.f) + bb[i];
      lo = fminf(lo, dd[i] - r);
      hi = fmaxf(hi, dd[i] + r);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const float pad = 1e-6f * fmaxf(fabsf(lo), fabsf(hi)) + pivmin;
    lo -= pad;
    hi += pad;
    const int mrank = n - 1 - g;  // ascending index of the g-th largest eigenvalue
    for (int it = 0; it < 8; ++it) {  // 9^8 = 4.3e7: FP32 resolution of the interval
      const float h = (hi - lo) * (1.f / 9.f);
      const float x = lo + (float)(s + 1) * h;
      int c = 0;
      if (act) {
        float q = dd[0] - x;
        if (fabsf(q) < pivmin) q = -pivmin;
        c = q < 0.f;
#pragma unroll 8
        for (int i = 1; i < n; ++i) {
          q = (dd[i] - x) - __fdividef(b2[i - 1], q);
          if (fabsf(q) < pivmin) q = -pivmin;
          c += q < 0.f;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, act && c > mrank);
      const unsigned gb = (bal >> (8 * l)) & 0xffu;
      if (gb) {
        const int f = __ffs(gb) - 1;
        const float nhi = lo + (float)(f + 1) * h;
        lo = f > 0 ? lo + (float)f * h : lo;
        hi = nhi;
      } else {
        lo = lo + 8.f * h;
      }
    }
    if (act && s == 0) evals[g] = 0.5 * ((double)lo + (double)hi);
  }
  __syncthreads();
  EIG_STAMP(3);
  // ---------------------------------------------------------- 4. eigenvectors of T (twisted)
  float* Dp = work;
  float* Dm = work + n * n;
  float* Y = work + 2 * n * n;  // [i * n + k]
  if (tid < n) {
    const int k = tid;
    const float lam = (float)evals[k];
    float q = dd[0] - lam;
    if (fabsf(q) < pivmin) q = -pivmin;
    Dp[k] = q;
    for (int i = 1; i < n; ++i) {
      q = (dd[i] - lam) - b2[i - 1] / q;
      if (fabsf(q) < pivmin) q = -pivmin;
      Dp[i * n + k] = q;
    }
    q = dd[n - 1] - lam;
    if (fabsf(q) < pivmin) q = -pivmin;
    Dm[(n - 1) * n + k] = q;
    for (int i = n - 2; i >= 0; --i) {
      q = (dd[i] - lam) - b2[i] / q;
      if (fabsf(q) < pivmin) q = -pivmin;
      Dm[i * n + k] = q;
    }
    int r = 0;
    float best = 3.0e38f;
    for (int i = 0; i < n; ++i) {
      const float gm = fabsf(Dp[i * n + k] + Dm[i * n + k] - (dd[i] - lam));
      if (gm < best) {
        best = gm;
        r = i;
      }
    }
    float z = 1.f, nrm2 = 1.f;
    Y[r * n + k] = 1.f;
    for (int i = r - 1; i >= 0; --i) {
      z = -(bb[i] / Dp[i * n + k]) * z;
      Y[i * n + k] = z;
      nrm2 = fmaf(z, z, nrm2);
    }
    z = 1.f;
    for (int i = r + 1; i < n; ++i) {
      z = -(bb[i - 1] / Dm[i * n + k]) * z;
      Y[i * n + k] = z;
      nrm2 = fmaf(z, z, nrm2);
    }
    const float inv = rsqrtf(nrm2);
    for (int i = 0; i < n; ++i) Y[i * n + k] *= inv;
  }
  __syncthreads();
  // clusters (gap < 2e-6 of the spectral radius): the twisted vectors of the
  // members nearly coincide; rebuild members 2.. by inverse iteration
  // (T - lam_k) x = y with reorthogonalisation against the earlier members
  // (LAPACK stein-style).  One warp: rows lane and lane + 32, dot products by
  // warp reduction, the tridiagonal solve by lane 0.  At most 24 members per
  // matrix are rebuilt (clusters are rare: bound the worst case).
  if (warp == 0) {
    static_assert(n <= 64, "two rows per lane");
    const float tnorm = fmaxf(fabsf((float)evals[0]), fabsf((float)evals[n - 1]));
    const float ctol = 2e-6f * tnorm, dfloor = 1e-7f * tnorm + pivmin;
    const int r0 = lane, r1 = lane + 32;
    const bool h1 = r1 < n;
    int cs = 0, budget = 24;
    for (int k = 1; k < n && budget > 0; ++k) {
      if ((float)(evals[k - 1] - evals[k]) > ctol) {
        cs = k;
        continue;
      }
      // clusters below `care` (shrink factor 0) keep their MGS-orthonormalised
      // twisted vectors: any orthonormal basis of that tail will do
      if ((float)evals[cs] < care) continue;
      --budget;
      float y0 = Y[r0 * n + k], y1 = h1 ? Y[r1 * n + k] : 0.f;
      for (int it = 0; it < 3; ++it) {
        for (int p = cs; p < k; ++p) {
          const float p0 = Y[r0 * n + p], p1 = h1 ? Y[r1 * n + p] : 0.f;
          const float dt = warp_sum_f(fmaf(y0, p0, y1 * p1));
          y0 = fmaf(-dt, p0, y0);
          y1 = fmaf(-dt, p1, y1);
        }
        const float nn = warp_sum_f(fmaf(y0, y0, y1 * y1));
        if (!(nn > 1e-30f)) {  // fully dependent: restart from a fixed pseudo-random vector
          y0 = hash_unit(0x9E3779B9u * (unsigned)(r0 + 1) + (unsigned)k);
          y1 = h1 ? hash_unit(0x9E3779B9u * (unsigned)(r1 + 1) + (unsigned)k) : 0.f;
          continue;
        }
        const float inn = rsqrtf(nn);
        y0 *= inn;
        y1 *= inn;
        if (it == 2) break;
        // one inverse-iteration step with the stored L D L^T of T - lam (D floored)
        Y[r0 * n + k] = y0;
        if (h1) Y[r1 * n + k] = y1;
        __syncwarp();
        if (lane == 0) {
          auto dfl = [&](float dv) { return fabsf(dv) < dfloor ? copysignf(dfloor, dv) : dv; };
          float w = Y[k];
          for (int i = 1; i < n; ++i) {
            const float dv = dfl(Dp[(i - 1) * n + k]);
            const float wi = Y[i * n + k] - (bb[i - 1] / dv) * w;
            Y[(i - 1) * n + k] = w / dv;
            w = wi;
          }
          float x = w / dfl(Dp[(n - 1) * n + k]);
          Y[(n - 1) * n + k] = x;
          for (int i = n - 2; i >= 0; --i) {
            x = Y[i * n + k] - (bb[i] / dfl(Dp[i * n + k])) * x;
            Y[i * n + k] = x;
          }
        }
        __syncwarp();
        y0 = Y[r0 * n + k];
        y1 = h1 ? Y[r1 * n + k] : 0.f;
        float mx = fmaxf(fabsf(y0), fabsf(y1));  // keep the iterate in range
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (mx > 0.f) {
          y0 /= mx;
          y1 /= mx;
        }
      }
      Y[r0 * n + k] = y0;
      if (h1) Y[r1 * n + k] = y1;
      __syncwarp();
    }
  }
  __syncthreads();
  EIG_STAMP(4);
  // ---------------------------------------------------------- 5. MGS, phases, back-transform
  {
    const int g = gi, s = gs;
    const bool act = g < n;
    float y[CU];
#pragma unroll
    for (int t = 0; t < CU; ++t) y[t] = act ? Y[(s + 8 * t) * n + g] : 0.f;
    // Gram-Schmidt over the eigenvectors whose eigenvalue is >= care (the
    // only ones that enter the thresholded spectral function; the rest are a
    // warm-start basis that the next QR re-orthonormalises) plus one
    int nh = 1;
    for (int k = 1; k < n; ++k) nh += (float)evals[k] >= care;
    nh = min(n, nh + 1);
    // orth_mode 0 (default): one symmetric first-order correction of the head,
    // Y_h <- Y_h (I - E / 2), E = Y_h^T Y_h - I -- the twisted / cluster vectors
    // are orthonormal to ~1e-4 at worst (close, unclustered pairs in early
    // iterations), which the correction squares -- in two barrier-separated
    // steps instead of nh; the Gram-Schmidt sweep below stays as the fallback
    // when some |E| exceeds 1e-3.  2: Gram-Schmidt only; 1: neither (experiment).
    if (orth_mode == 1) nh = 0;
    if (orth_mode == 0) {
      float* E = Dp;  // n x n floats, dead after the twisted factorisations
      bool big = false;
      for (int idx = tid; idx < nh * nh; idx += NT) {
        const int a = idx / nh, b = idx - a * nh;
        if (a <= b) {
          float dot = 0.f;
#pragma unroll 8
          for (int i = 0; i < n; ++i) dot = fmaf(Y[i * n + a], Y[i * n + b], dot);
          const float e = dot - (a == b ? 1.f : 0.f);
          E[a * n + b] = e;
          E[b * n + a] = e;
          big = big || !(fabsf(e) <= 1e-3f);
        }
      }
      if (!__syncthreads_or(big)) {
        if (act && g < nh) {
#pragma unroll
          for (int t = 0; t < CU; ++t) {
            float acc = 0.f;
            for (int b = 0; b < nh; ++b) acc = fmaf(Y[(s + 8 * t) * n + b], E[b * n + g], acc);
            y[t] = fmaf(-0.5f, acc, y[t]);
          }
        }
        nh = 0;
      }
    }
    for (int k = 0; k < nh; ++k) {
      float ss = 0.f;
#pragma unroll
      for (int t = 0; t < CU; ++t) ss = fmaf(y[t], y[t], ss);
      ss = group8_sum(ss);
      if (g == k) {
        const float inv = rsqrtf(ss);
#pragma unroll
        for (int t = 0; t < CU; ++t) {
          y[t] *= inv;
          Y[(s + 8 * t) * n + k] = y[t];
        }
      }
      __syncthreads();
      float dot = 0.f;
      float yk[CU];
#pragma unroll
      for (int t = 0; t < CU; ++t) {
        yk[t] = Y[(s + 8 * t) * n + k];
        dot = fmaf(y[t], yk[t], dot);
      }
      dot = group8_sum(dot);
      if (act && g > k) {
#pragma unroll
        for (int t = 0; t < CU; ++t) y[t] = fmaf(-dot, yk[t], y[t]);
      }
    }
    EIG_STAMP(5);
    float2 u[CU];
#pragma unroll
    for (int t = 0; t < CU; ++t) u[t] = cscale(ph[s + 8 * t], y[t]);
    for (int j = n - 3; j >= 0; --j) {
      float2 part = make_float2(0.f, 0.f);
      float2 v[CU];
#pragma unroll
      for (int t = 0; t < CU; ++t) {
        v[t] = H[(s + 8 * t) * KS + j];
        cfmac(part, v[t], u[t]);
      }
      part.x = group8_sum(part.x);
      part.y = group8_sum(part.y);
      const float2 tw = cscale(part, th[j]);
#pragma unroll
      for (int t = 0; t < CU; ++t) u[t] = csub(u[t], cmul(v[t], tw));
    }
    __syncthreads();  // Y / Dp / Dm (aliasing U) are dead
    if (act) {
#pragma unroll
      for (int t = 0; t < CU; ++t) U[(s + 8 * t) * KS + g] = u[t];
    }
  }
  __syncthreads();
  EIG_STAMP(6);
#undef EIG_STAMP
}

}  // namespace

// M (d x KB in smem, row stride KS) <- (I - V1 V1^H) M, V1 = the first k1
// columns of a global d x ld block (orthonormal), coefficients staged in
// `coef` (k1 x KB smem).  Two barriers; called by the whole CTA.
template <int KB, int KS>
__device__ void project_out(float2* M, const float2* __restrict__ V1, int ld, int k1, int d, float2* coef) {
  for (int t = threadIdx.x; t < k1 * KB; t += blockDim.x) {
    const int i = t % k1, j = t / k1;
    float2 a = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int k = 0; k < d; ++k) cfmac(a, __ldg(V1 + (long long)k * ld + i), M[k * KS + j]);
    coef[i * KB + j] = a;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < d * KB; t += blockDim.x) {
    const int k = t / KB, j = t - k * KB;
    float2 m = M[k * KS + j];
#pragma unroll 4
    for (int i = 0; i < k1; ++i) {
      const float2 v = __ldg(V1 + (long long)k * ld + i), c = coef[i * KB + j];
      m.x -= v.x * c.x - v.y * c.y;
      m.y -= v.x * c.y + v.y * c.x;
    }
    M[k * KS + j] = m;
  }
  __syncthreads();
}

template <int DP, int KB, int R, bool BIG, bool L2, int MINB = 1, bool MMA = false>
__global__ void __launch_bounds__(kSubNT, MINB) svt_subspace_kernel(const SvtParams prm) {
  constexpr int NT = kSubNT;
  constexpr int KS = KB + 1;       // row stride of the d x KB blocks (conflict-free column walks)
  constexpr int CS = DP + 1;       // row stride of the R x d chunk (odd: conflict-free anti-diagonal walks)
  constexpr int NC = KB / 16;      // 16-column groups
  constexpr int MR = (DP + 31) / 32;
  // the large-d fallback block (KB > 48) has no room for the split-k buffer
  // solver levels: level 1 (KB1 columns) for every matrix, level 2 (KB2) for
  // the ones whose rank above the threshold came too close to KB1; d <= 128
  // has the full solver behind level 2, d > 128 (BIG) has nothing
  // (d <= 128 level 1 runs with kSubspaceKB1 or kSubspaceKB columns; only
  // the former has a level 2 behind it)
  // HUGE (248 < d <= 496): 16-row chunks, a 32-column block for every level
  // (level 1, then the deflation chain), one-output-per-thread chunk GEMM
  constexpr bool HUGE = BIG && R == 16;
  // SMALLD (40 <= d < 72): 16-column level 1, 32-column level 2
  constexpr bool SMALLD = !BIG && DP < 72;
  // COLOC: the large-d *layout* used at d <= 128 so that two CTAs share an SM
  // (MINB = 2); its levels are those of d <= 128 (level 2 and the full solver
  // behind it run in the resident layout)
  constexpr bool COLOC = BIG && MINB == 2;
  constexpr bool BIGLV = BIG && !COLOC;
  constexpr int KB1 = HUGE ? kSubspaceKBHuge : BIGLV ? kSubspaceKB : SMALLD ? kSubspaceKBSmall : (L2 ? kSubspaceKB1 : KB);
  constexpr int KB2 = HUGE ? kSubspaceKBHuge : BIGLV ? kSubspaceKBBig : SMALLD ? kSubspaceKB1 : kSubspaceKB;
  static_assert(HUGE     ? KB == kSubspaceKBHuge
                : SMALLD ? KB == (L2 ? KB2 : KB1)
                : L2     ? KB == KB2
                         : (BIGLV ? KB == kSubspaceKB : (KB == kSubspaceKB1 || KB == kSubspaceKB)),
                "block size of the level");
  static_assert(!COLOC || !L2, "the co-located layout is a level-1 variant");
  // the chunk buffer doubles as the eigen-solver's work area (3 KB^2 floats)
  // and the Cholesky QR's Gram matrix (KB x KS); in the large-d layout the
  // Rayleigh-Ritz matrix sits right behind it, so the co-located layout pads
  // the chunk buffer to CROWS >= R rows when R x CS is too small for the work
  // area (d = 72 with a 48-column block, config 1: 48 rows)
  constexpr int CROWS = (COLOC && 2 * R * CS < 3 * KB * KB) ? (3 * KB * KB / 2 + CS - 1) / CS : R;
  static_assert(!COLOC || (2 * CROWS * CS >= 3 * KB * KB && CROWS * CS >= KB * KS),
                "chunk buffer too small for this block");
  constexpr bool NOSPLIT = BIG && L2 && !HUGE;
  // MMA: the chunk contractions run as 3xTF32 on the tensor cores (svt_mma.cuh)
  static_assert(!MMA || (R == 32 && (KB == 48 || KB == 32) && !NOSPLIT && !HUGE && DP <= 128 && DP % 8 == 0),
                "the mma.sync mappings cover 32- and 48-column blocks with d <= 128");
  static_assert(KB % 16 == 0 && KB % 8 == 0, "KB must be a multiple of 16");
  static_assert(R == 32 || HUGE, "the thread mappings assume 32-row chunks (HUGE: 16)");
  // Ritz pairs one deflation step keeps, and the margin below the block edge
  constexpr int DSTEP = HUGE ? KB - kSubspaceMargin : kDeflateK;
  // epilogue mapping: Z row zr, columns zc + ZC m
  constexpr int ZC = kSubNT / R;

  if (prm.skip && *prm.skip) return;
  int mat;
  const SvtFamily& F = family_of(prm, blockIdx.x, mat);
  if (F.halt && F.halt[mat / F.halt_div]) return;
  if (prm.only_flagged && (prm.only_flag_value ? F.fallback[mat] != prm.only_flag_value : !F.fallback[mat]))
    return;
  // per-matrix level flag (fallback): 0 level 1, kLevelHanded handed to
  // level 2 by level 1 in this launch, kLevelStay2 kept at level 2 from the
  // previous iteration, kLevelDeflate split between level 2 and the deflated
  // level 3, kLevelOverflow beyond that; level 1 skips the matrices that are
  // not at level 1
  if (!L2 && !HUGE && F.fallback &&
      (F.fallback[mat] == kLevelStay2 || F.fallback[mat] == kLevelOverflow || F.fallback[mat] == kLevelDeflate ||
       F.fallback[mat] == kLevelDeflDone))
    return;
  // level 3 (large d): SVT of the part of the matrix orthogonal to level 2's
  // leading kDeflateK Ritz vectors, plus level 2's Z1 on that part
  const bool defl3 = BIG && L2 && prm.deflate;
  const int tid = threadIdx.x;
  const int d = F.d, e = F.e, len = F.len, B = F.B, J = F.J;
  const bool admm = prm.mode != SVT_PLAIN;
  const bool weighted = prm.mode == SVT_ADMM_WEIGHTED;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  // BIG (d > 128): one d x KB block V (the pass output, the QR and the Ritz
  // rotation work in place; X aliases V), no resident spectra / adjoint
  // accumulators (wl holds wc (len), acc the two carried partial adjoint
  // blocks (2 x len)), no dual staging (duals read from L2 per chunk), and
  // the Rayleigh-Ritz matrix H in the Yc | Yc2 pair.
  float2* V = reinterpret_cast<float2*>(smem_raw);  // DP x KS
  float2* X = BIG ? V : V + DP * KS;                 // DP x KS (non-BIG: also H for the Ritz solve)
  float2* C = BIG ? V + DP * KS : X + DP * KS;       // R x CS  (Ahat chunk / U / T)
  float2* Yc = C + CROWS * CS;                       // R x KS
  float2* Yc2;                                       // R x KS (second k-half of the chunk GEMM)
  float2* wl;                                        // B x len  (BIG: len)
  float2* acc;                                       // B x len  (BIG: 2 x len)
  float2* tail;
  // NOSPLIT: the Rayleigh-Ritz matrix sits behind the eigen-solver's work
  // area (3 KB^2 floats at C), spilling from C into the Y region
  constexpr int YREG = HUGE ? R * KS : NOSPLIT ? (KB * KS + 3 * KB * KB / 2 - R * CS > R * KS ? KB * KS + 3 * KB * KB / 2 - R * CS
                                                                              : R * KS)
                               : 2 * R * KS;
  if (BIG) {
    Yc2 = NOSPLIT ? nullptr : Yc + R * KS;
    wl = Yc + YREG;
    acc = wl + len;
    tail = acc + 2 * len;
  } else {
    wl = Yc + R * KS;
    acc = wl + B * len;
    Yc2 = acc + B * len;
    tail = Yc2 + R * KS;
  }
  float2* Hm = BIG ? ((NOSPLIT || HUGE) ? C + 3 * KB * KB / 2 : Yc) : X;  // KB x KS Rayleigh-Ritz matrix
  Smem<KB> S;                                        // Rayleigh-Ritz Jacobi workspace
  S.G = Hm;
  S.rec = reinterpret_cast<SlotRec*>(tail);
  S.dgr = reinterpret_cast<double2*>(S.rec + KB);
  S.dg = reinterpret_cast<double*>(S.dgr + KB);
  S.f = reinterpret_cast<float*>(S.dg + KB);
  float* tau = S.f + KB;
  S.flags = reinterpret_cast<int*>(tau + KB);
  S.scal = reinterpret_cast<float*>(S.flags + 4);
  int* cnt = reinterpret_cast<int*>(S.scal + 4);
  int* perm = cnt + 4;                               // KB: descending-order position
  int* lofs = perm + KB;                             // max(d, e): lift offsets (lift_tab)

  float2* Dg = admm ? F.D + (long long)mat * e * d : nullptr;
  // Ahat V of the Rayleigh-Ritz pass (e x KB), reused by the Z pass
  float2* ycg = (MMA && prm.ycache) ? prm.ycache + (long long)blockIdx.x * e * KB : nullptr;
  float2* Vsg = F.Vs + (long long)mat * DP * KB1;  // level-1 store: KB1 columns
  float2* Vsg2 = L2 && F.Vs2 ? F.Vs2 + (long long)mat * DP * KB : nullptr;  // level-2 store
  // level 2 starts warm (from its own store) only for matrices it kept from
  // the previous iteration; the ones level 1 just handed over start from
  // level 1's fresh block (+ random columns)
  const int lvl_in = F.fallback ? F.fallback[mat] : 0;
  const bool warm = !defl3 && prm.warm && *prm.warm &&
                    (!L2 || (Vsg2 && (lvl_in == kLevelStay2 || lvl_in == kLevelOverflow || lvl_in == kLevelDeflate ||
                                      lvl_in == kLevelDeflDone)));
  const bool seeded = L2 && !defl3 && !warm && lvl_in == kLevelHanded;
  // deflation chain: Ritz vectors already solved (level 2's leading block and
  // every earlier level-3 step's), kept orthonormal in Vd
  const bool chain = BIG && (L2 || HUGE) && F.Z1 && F.Vd && F.ndefl;
  float2* Vdg = chain ? F.Vd + (long long)mat * DP * DP : nullptr;
  const int nd_in = defl3 ? F.ndefl[mat] : 0;
  // M <- (I - Vd Vd^H) M over the deflated columns, in blocks of kDeflateK
  // (block classical Gram-Schmidt, repeated: CGS2)
  auto project_defl = [&](float2* M) {
    for (int rep = 0; rep < 2; ++rep)
      for (int b0 = 0; b0 < nd_in; b0 += DSTEP)
        project_out<KB, KS>(M, Vdg + b0, DP, min(DSTEP, nd_in - b0), d, C);
  };
  const bool stg = Dg != nullptr && !BIG;  // duals staged by cp.async (non-BIG)

  // ---------------------------------------------------------- spectra
  const float2* spg = F.spec + (long long)mat * F.s_mat;
  if (BIG) {
    for (int t = tid; t < len; t += NT) wl[t] = weighted ? F.wc[t] : make_float2(1.f, 0.f);
    for (int t = tid; t < 2 * len; t += NT) acc[t] = make_float2(0.f, 0.f);
    // block/shift of the lifted index: rows of Ahat (wide) or its columns (tall)
    build_lofs(lofs, F, true, tid, NT);
    // tall: the adjoint accumulates into this matrix's own output region
    // across chunks (every chunk touches every block); the output must not
    // alias the spectra (read again in every pass)
    if (!F.wide) {
      float2* op = F.out + (long long)mat * F.o_mat;
      for (int t = tid; t < J * len; t += NT) {
        const int j = t / len, n = t - j * len;
        op[(long long)n * F.o_n + (long long)j * F.o_j] = make_float2(0.f, 0.f);
      }
    }
    if (tid < 4) S.flags[tid] = 0;
    if (tid == 0) *cnt = 0;
  } else {
    stage_spectra(wl, F, spg, weighted, tid, NT);
    for (int t = tid; t < B * len; t += NT) acc[t] = make_float2(0.f, 0.f);
    build_lofs(lofs, F, false, tid, NT);
    if (tid < 4) S.flags[tid] = 0;
    if (tid == 0) *cnt = 0;
  }
  int ns_steps = 0;  // Newton-Schulz steps taken (diagnostics)
  if (BIG && Dg) prefetch_l2(Dg, min(R, e) * d);  // first chunk of the first pass
  long long clk_qr = 0, clk_pass = 0, clk_t = clock64();
  long long clk_wait = 0, clk_build = 0, clk_g1 = 0, clk_sum = 0, clk_g2 = 0, clk_u = 0;
#define SUB_ACC(v) \
  if (prm.phase_clk) { const long long nw_ = clock64(); v += nw_ - clk_u; clk_u = nw_; }
#define SUB_STAMP(k) \
  if (prm.phase_clk && tid == 0) prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + (k)] = clock64()
  SUB_STAMP(0);

  // ---------------------------------------------------------- starting block
  if (warm) {
    for (int t = tid; t < DP * KB; t += NT) {
      const int k = t / KB, j = t - k * KB;
      V[k * KS + j] = Vsg2 ? Vsg2[t] : (j < KB1 ? Vsg[k * KB1 + j] : make_float2(0.f, 0.f));
    }
    __syncthreads();
  } else {
    for (int t = tid; t < DP * KB; t += NT) {
      const int k = t / KB, j = t - k * KB;
      const unsigned int h = (unsigned int)(mat * 0x9E3779B1u) ^ (unsigned int)(t * 0x85EBCA77u);
      float2 v = k < d ? make_float2(hash_unit(h), hash_unit(h ^ 0x5bd1e995u)) : make_float2(0.f, 0.f);
      if (seeded && j < KB1) v = Vsg[k * KB1 + j];
      X[k * KS + j] = v;
    }
    __syncthreads();
    if (defl3) project_defl(X);  // start orthogonal to the deflated columns
    householder_qr<KB, KS, DP, (HUGE ? 16 : 8)>(X, V, d, tau);
    // a remainder narrower than the block: the QR's extra columns leave the
    // remainder, projecting them out makes them ~0 (Ritz values ~0, f = 0)
    if (defl3 && d - nd_in < KB) project_defl(V);
  }

  // large-d chunk build; the tensor variants have the split buffer Yc2 free
  // during the passes and stage the chunk's lift sources there
  auto build_big = [&](int i0, int rows) {
    if constexpr (BIG && MMA) {
      const ChunkSources cs = stage_chunk_sources(Yc2, R * KS, F, spg, wl, weighted, i0, rows);
      if (cs.ok) {
        __syncthreads();
        build_chunk_staged<DP, CS, R>(C, F, Yc2, cs, lofs, Dg, i0, rows, prm.inv_beta);
        return;
      }
    }
    if constexpr (BIG) build_chunk_big<DP, CS, R>(C, F, spg, wl, weighted, lofs, Dg, i0, rows, prm.inv_beta);
  };
  // mappings: Yc rows yi / X rows k0 + 32m, columns c + 16n
  const int yi = tid >> 4, c16 = tid & 15;
  int iters = warm ? prm.q_warm : prm.q_cold;
  if (warm && prm.relc) {  // adaptive warm passes: the iterate moved a lot last iteration
    const double rc = *prm.relc;
    if (rc > (double)prm.relc_q3) iters = max(iters, 3);
    else if (rc > (double)prm.relc_q2) iters = max(iters, 2);
  }
  // large-d level 2 (41 to 62 of its 64 columns above the threshold): the
  // block has little margin over the rank, which is what sets the accuracy of
  // a warm pass -- two passes (config 3 against the reference's own run at
  // iteration 50, all 512 matrices at level 2 or in the chain: 1.04e-4 with
  // one pass; more passes for the chain matrices alone changed nothing)
  if (BIGLV && L2 && warm && prm.l2_warm_passes > 1) {
    // (with the previous rank known: only where the margin is small)
    const int r_prev = (F.rank_prev && prm.l2_pass_margin > 0) ? F.rank_prev[mat] : KB;
    if (r_prev > KB - prm.l2_pass_margin || prm.l2_pass_margin <= 0) iters = max(iters, prm.l2_warm_passes);
  }
  // inner passes are only normalised when the warm block is already near the
  // subspace (the default single pass); extra adaptive passes are QR'd
  const bool inner_norm = prm.inner_norm && iters == prm.q_warm;

  // ---------------------------------------------------------- subspace iteration
  // Duals are staged chunk by chunk with cp.async into a buffer that is free
  // during the pass (X here, V in the epilogue pass): the copy of chunk c+1
  // overlaps the GEMMs of chunk c.
  for (int it = 0; it < iters; ++it) {
    float2 xa[MMA ? 1 : MR][MMA ? 1 : NC];
    XAccMma<KB / 16> xm;
    if constexpr (MMA) {
      xm.zero();
    } else {
#pragma unroll
      for (int m = 0; m < MR; ++m)
#pragma unroll
        for (int n = 0; n < NC; ++n) xa[m][n] = make_float2(0.f, 0.f);
    }
    __syncthreads();  // X (reflectors of the last QR) is free from here
    if (stg) stage_d_async(X, Dg, 0, min(R, e), d);
    if (prm.phase_clk) clk_u = clock64();
    for (int i0 = 0; i0 < e; i0 += R) {
      const int rows = min(R, e - i0);
      if (stg) stage_d_wait();
      SUB_ACC(clk_wait);
      if (BIG && Dg && i0 + R < e) prefetch_l2(Dg + (long long)(i0 + R) * d, min(R, e - i0 - R) * d);
      if (BIG) build_big(i0, rows);
      else build_chunk<DP, CS, R>(C, wl, lofs, F, Dg ? X : nullptr, i0, rows, prm.inv_beta);
      __syncthreads();
      SUB_ACC(clk_build);
      if (stg && i0 + R < e) stage_d_async(X, Dg, i0 + R, min(R, e - i0 - R), d);
      if constexpr (HUGE) chunk_block_huge<CS, KS, R>(C, V, Yc, d, KB, nullptr);  // Yc = C V
      else if constexpr (MMA) chunk_block_mma<CS, KS, NC, R>(C, V, Yc, Yc2, d, nullptr);
      else chunk_block<CS, KS, NC, R, NOSPLIT>(C, V, Yc, Yc2, d, nullptr);
      SUB_ACC(clk_g1);
      if constexpr (MMA) {
        xacc_mma<CS, KS>(xm, C, Yc);  // X += C^H Yc (rows beyond the chunk are zero)
      } else {
#pragma unroll 4
        for (int i = 0; i < rows; ++i) {  // X += C^H Yc
          float2 yv[NC];
#pragma unroll
          for (int n = 0; n < NC; ++n) yv[n] = Yc[i * KS + c16 + 16 * n];
#pragma unroll
          for (int m = 0; m < MR; ++m) {
            const int k = yi + 32 * m;
            if (k < DP) {
              const float2 a = C[i * CS + k];
#pragma unroll
              for (int n = 0; n < NC; ++n) cfmac(xa[m][n], a, yv[n]);
            }
          }
        }
      }
      if (!stg) __syncthreads();  // with staged duals the next stage_d_wait() is the barrier
      SUB_ACC(clk_g2);
    }
    if (stg) __syncthreads();
    if constexpr (MMA) {
      xacc_store<DP, KS>(xm, X);
    } else {
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        const int k = yi + 32 * m;
        if (k < DP)
#pragma unroll
          for (int n = 0; n < NC; ++n) X[k * KS + c16 + 16 * n] = xa[m][n];
      }
    }
    __syncthreads();
    clk_pass += clock64() - clk_t;
    clk_t = clock64();
    if (BIG && Dg) prefetch_l2(Dg, min(R, e) * d);  // first chunk of the next pass (behind the QR)
    if (defl3) project_defl(X);
    if (warm && inner_norm && it + 1 < iters) {
      // warm inner pass: X ~ V0 Lambda with V0 the previous (sorted) Ritz
      // vectors, so unit columns are already a well-conditioned basis; the
      // last pass is orthonormalised before the Rayleigh-Ritz projection
      const int g = tid >> 3, s8 = tid & 7;
      float ss = 0.f;
      if (g < KB)
        for (int row = s8; row < d; row += 8) {
          const float2 x = X[row * KS + g];
          ss = fmaf(x.x, x.x, fmaf(x.y, x.y, ss));
        }
      ss = group8_sum(ss);
      const float inv = ss > 1e-30f ? rsqrtf(ss) : 0.f;
      if (g < KB)
        for (int row = s8; row < DP; row += 8) V[row * KS + g] = cscale(X[row * KS + g], inv);
    } else {
      int ns = 0;
      if constexpr (MMA) {
        // warm pass: Cholesky QR on the tensor cores (ns_orth 1), or the
        // Newton-Schulz trial (2: the tail columns of a warm block are too far
        // from orthogonal for it, ||E||_F ~ 3)
        if (warm && prm.ns_orth == 1)
          ns = cholesky_qr_mma<KB, KS, DP>(X, V, C, BIG ? Yc : V, tau, S.flags + 3, 1e-3f,
                                           prm.phase_clk ? prm.phase_clk + (long long)blockIdx.x * kPhaseSlots + 13
                                                         : nullptr);  // slots 13, 14, 15, 23
        else if (warm && prm.ns_orth == 2)
          ns = newton_schulz_orth<KB, KS, DP>(X, V, C, tau);
        ns_steps += ns;
      }
      if (ns == 0) householder_qr<KB, KS, DP, (HUGE ? 16 : 8)>(X, V, d, tau);
      if (defl3 && d - nd_in < KB) project_defl(V);
    }
    clk_qr += clock64() - clk_t;
    clk_t = clock64();
  }
  if (prm.phase_clk && tid == 0) {
    prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + 1] = clk_pass;
    prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + 2] = clk_qr;
    prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + 8] = clk_wait;
    prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + 9] = clk_build;
    prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + 10] = clk_g1;
    prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + 11] = clk_sum;
    prm.phase_clk[(long long)blockIdx.x * kPhaseSlots + 12] = clk_g2;
  }
  SUB_STAMP(3);

  // ---------------------------------------------------------- Rayleigh-Ritz: H = (Ahat V)^H (Ahat V)
  {
    constexpr int HM = (KB + 31) / 32;
    float2 h[MMA ? 1 : HM][MMA ? 1 : NC];
    HAccMma hm;
    if constexpr (MMA) {
      hm.zero();
    } else {
#pragma unroll
      for (int m = 0; m < HM; ++m)
#pragma unroll
        for (int n = 0; n < NC; ++n) h[m][n] = make_float2(0.f, 0.f);
    }
    __syncthreads();  // X is free from here
    if (stg) stage_d_async(X, Dg, 0, min(R, e), d);
    for (int i0 = 0; i0 < e; i0 += R) {
      const int rows = min(R, e - i0);
      if (stg) stage_d_wait();
      if (BIG && Dg && i0 + R < e) prefetch_l2(Dg + (long long)(i0 + R) * d, min(R, e - i0 - R) * d);
      if (BIG) build_big(i0, rows);
      else build_chunk<DP, CS, R>(C, wl, lofs, F, Dg ? X : nullptr, i0, rows, prm.inv_beta);
      __syncthreads();
      if (stg && i0 + R < e) stage_d_async(X, Dg, i0 + R, min(R, e - i0 - R), d);
      if constexpr (HUGE) chunk_block_huge<CS, KS, R>(C, V, Yc, d, KB, nullptr);
      else if constexpr (MMA) chunk_block_mma<CS, KS, NC, R>(C, V, Yc, Yc2, d, nullptr);
      else chunk_block<CS, KS, NC, R, NOSPLIT>(C, V, Yc, Yc2, d, nullptr);
      if constexpr (MMA) {
        if (ycg)  // Ahat V rows of this chunk, kept for the Z pass
          for (int t = tid; t < rows * KB; t += NT) {
            const int i = t / KB, j = t - i * KB;
            ycg[(long long)(i0 + i) * KB + j] = Yc[i * KS + j];
          }
        hacc_mma<KS>(hm, Yc);  // rows beyond the chunk are zero
      } else {
        for (int i = 0; i < rows; ++i) {
#pragma unroll
          for (int m = 0; m < HM; ++m) {
            const int a = yi + 32 * m;
            if (a < KB) {
              const float2 ya = Yc[i * KS + a];
#pragma unroll
              for (int n = 0; n < NC; ++n) cfmac(h[m][n], ya, Yc[i * KS + c16 + 16 * n]);
            }
          }
        }
      }
      if (!stg) __syncthreads();
    }
    if (stg) __syncthreads();
    // H (full Hermitian, stride KB+1 = KS) into Hm, diagonal to S.dg
    if constexpr (MMA) {
      hacc_store<KS>(hm, Hm);  // upper block triangle
      __syncthreads();
      // mirror into the lower triangle (the diagonal blocks hold both
      // triangles, equal only to the last bits of the split products)
      for (int t = tid; t < KB * KB; t += NT) {
        const int a = t / KB, b = t - a * KB;
        if (a < b) {
          Hm[b * KS + a] = cconj(Hm[a * KS + b]);
        } else if (a == b) {
          const float2 v = Hm[a * KS + a];
          Hm[a * KS + a] = make_float2(v.x, 0.f);
          S.dg[a] = v.x;
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < HM; ++m) {
        const int a = yi + 32 * m;
        if (a < KB)
#pragma unroll
          for (int n = 0; n < NC; ++n) {
            const int b = c16 + 16 * n;
            if (a == b) S.dg[a] = h[m][n].x;
            Hm[a * KS + b] = h[m][n];
          }
      }
    }
  }
  __syncthreads();
  if (BIG && Dg) prefetch_l2(Dg, min(R, e) * d);  // first chunk of the Z pass (behind the Rayleigh-Ritz solve)
  if (!prm.rr_jacobi) {
    SUB_STAMP(4);
    hermitian_eig_tridiag<KB, KS>(Hm, reinterpret_cast<float*>(S.rec), reinterpret_cast<float*>(C), C, S.dg,
                                  0.25f * prm.thresh * prm.thresh,
                                  prm.phase_clk ? prm.phase_clk + (long long)blockIdx.x * kPhaseSlots + 16 : nullptr,
                                  prm.rr_orth_mode);
    SUB_STAMP(5);
    if (prm.sweeps_out && tid == 0) prm.sweeps_out[blockIdx.x] = ns_steps;
  } else {
  if (tid < 32) {  // absolute rotation floor relative to the largest Ritz value
    double mx = 0.0;
    for (int u = tid; u < KB; u += 32) mx = fmax(mx, S.dg[u]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (tid == 0) S.scal[0] = (float)((prm.rr_tol_abs > 0.f ? prm.rr_tol_abs : kTolAbsRR) * mx);
  }
  __syncthreads();
  {
    constexpr int WK = KB / 8;
    float2 ut[WK], ub[WK];
    if (tid < 4 * KB) {
      const int vrow = tid >> 2, vg = tid & 3;
#pragma unroll
      for (int w = 0; w < WK; ++w) {
        const int s = vg * WK + w;
        ut[w] = make_float2(vrow == top0(s, KB) ? 1.f : 0.f, 0.f);
        ub[w] = make_float2(vrow == bot0(s, KB) ? 1.f : 0.f, 0.f);
      }
    }
    SUB_STAMP(4);
    // Ritz pairs both well below the threshold only mix the tail (shrink
    // factor 0 either way) and are not rotated
    // (a pair straddling the boundary can keep re-coupling through the
    // unrotated tail: the sweep cap bounds that; such vectors have f ~ 0)
    const float tail = prm.rr_tail * prm.thresh * prm.thresh;
    const int sw = jacobi<KB, WK>(S, ut, ub, prm.rr_tol_rel > 0.f ? prm.rr_tol_rel : kTolRel2, S.scal[0],
                                 min(prm.max_sweeps, kRitzMaxSweeps), tail);
    SUB_STAMP(5);
    if (prm.sweeps_out && tid == 0) prm.sweeps_out[blockIdx.x] = sw;
    if (tid < 4 * KB) store_v<KB, WK>(C, KS, ut, ub);  // U (KB x KB) into the chunk buffer
  }
  __syncthreads();
  }
  // descending order of the Ritz values: the stored block stays sorted, so the
  // next warm-started QR processes dominant directions first
  for (int j = tid; j < KB; j += NT) {
    const double lj = S.dg[j];
    int rank = 0;
    for (int i = 0; i < KB; ++i) {
      const double li = S.dg[i];
      rank += (li > lj) || (li == lj && i < j);
    }
    perm[j] = rank;
  }
  __syncthreads();
  // V <- V U (Ritz vectors, sorted) into X
  if constexpr (MMA) {
    XAccMma<KB / 16> vm;
    vm.zero();
    vu_mma<KS, KB>(vm, V, C);
    if (BIG) __syncthreads();  // in place: all reads of V are done
    xacc_store_perm<DP, KS>(vm, X, perm);
  } else {
    float2 va[MR][NC];
#pragma unroll
    for (int m = 0; m < MR; ++m)
#pragma unroll
      for (int n = 0; n < NC; ++n) va[m][n] = make_float2(0.f, 0.f);
    for (int j = 0; j < KB; ++j) {
      float2 u[NC];
#pragma unroll
      for (int n = 0; n < NC; ++n) u[n] = C[j * KS + c16 + 16 * n];
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        const int k = yi + 32 * m;
        if (k < DP) {
          const float2 v = V[k * KS + j];
#pragma unroll
          for (int n = 0; n < NC; ++n) cfma(va[m][n], v, u[n]);
        }
      }
    }
    if (BIG) __syncthreads();  // in place: all reads of V are done
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int k = yi + 32 * m;
      if (k < DP)
#pragma unroll
        for (int n = 0; n < NC; ++n) X[k * KS + perm[c16 + 16 * n]] = va[m][n];
    }
  }
  for (int j = tid; j < KB; j += NT) {
    const double lam = S.dg[j];
    float f = 0.f;
    if (lam > (double)prm.thresh * prm.thresh && lam > 0.0) {
      f = (float)(1.0 - prm.thresh / sqrt(lam));
      atomicAdd(cnt, 1);
    }
    S.f[perm[j]] = f;
  }
  __syncthreads();
  float2* Vf = X;  // final Ritz vectors (d x KB)
  const int r = *cnt;
  // diagnostics: Ritz values above the threshold (x1000) + Rayleigh-Ritz sweeps
  if (prm.sweeps_out && tid == 0) prm.sweeps_out[blockIdx.x] += 1000 * r;
  if (F.rank_prev && !defl3 && tid == 0) F.rank_prev[mat] = r;
  // the last level accepts Ritz pairs up to KB - kSubspaceMarginLast: pairs
  // that close to the block edge converge slowest but sit near the threshold,
  // where the shrink factor 1 - tau / sigma is ~0.  It keeps a matrix until
  // its rank falls well inside level 1's range (hysteresis).
  constexpr int kMarginHere = (BIG && L2 && !HUGE) ? kSubspaceMarginLast : kSubspaceMargin;
  // level 2 (large d) with too many values above the threshold and a Z1
  // buffer: keep the leading kDeflateK Ritz pairs (Z1 = Ahat V1 f1 V1^H to
  // HBM) and hand the rest to the deflated level 3
  // (level 3 again while the remainder is wider than its block; a remainder
  // the block spans is solved exactly, so the chain always finishes)
  const bool to_defl = chain && r > KB - kMarginHere && d - nd_in > KB;
  if (F.fallback && tid == 0) {
    if (defl3)
      F.fallback[mat] = to_defl ? kLevelDeflate : kLevelDeflDone;
    else if (HUGE)  // level 1 is the last level: the chain, or finishing with what it has
      F.fallback[mat] = to_defl ? kLevelDeflate : r > KB - kSubspaceMarginLast ? kLevelOverflow : 0;
    else if (L2)
      F.fallback[mat] = to_defl ? kLevelDeflate
                        : r > KB - kMarginHere ? kLevelOverflow
                        : r <= KB1 - 2 * kSubspaceMargin ? 0 : kLevelStay2;
    else
      F.fallback[mat] = (r > KB - kSubspaceMargin) ? kLevelHanded : 0;
  }
  if (to_defl) {  // append the leading DSTEP Ritz vectors to the deflated basis
    for (int t = tid; t < DP * DSTEP; t += NT) {
      const int k = t / DSTEP, j = t - k * DSTEP;
      Vdg[(long long)k * DP + nd_in + j] = Vf[k * KS + j];
    }
    if (tid == 0) F.ndefl[mat] = nd_in + DSTEP;
  }
  if (Vsg2 && !defl3)
    for (int t = tid; t < DP * KB; t += NT) {
      const int k = t / KB, j = t - k * KB;
      Vsg2[t] = Vf[k * KS + j];
    }
  // warm start of the next ADMM iteration at level 1: the leading KB1 Ritz
  // vectors (sorted), stored even when this matrix is handed to a fallback
  for (int t = tid; t < (defl3 ? 0 : DP * KB1); t += NT) {
    const int k = t / KB1, j = t - k * KB1;
    Vsg[t] = Vf[k * KS + j];
  }
  // too many singular values above the threshold: the fallback redoes this
  // matrix from its untouched duals (d <= 128: the full solver; d > 128: this
  // kernel with the larger block).  The last level finishes with the Ritz
  // pairs it has and the host reports the flag.
  // handed on: the next level redoes this matrix from its untouched duals
  // (the last level, BIG level 2, finishes with what it has; the host
  // reports its overflow flag)
  if (!(BIG && (L2 || HUGE)) && r > KB - kMarginHere) return;

  // ---------------------------------------------------------- Z = (Ahat V) f V^H, duals, adjoint
  SUB_STAMP(6);
  float2* Ds = V;  // the old basis is dead: stage the duals there (non-BIG)
  // cached Z pass (tensor-core variants): Ahat Vf = (Ahat V) U comes from the
  // Rayleigh-Ritz pass's Ahat V (ycg) and the rotation U (sorted, scaled by
  // the shrink factors) instead of rebuilding the chunk and multiplying by Vf
  constexpr int US = 32;  // row stride of the scaled rotation (its first 16 nb <= 32 sorted columns)
  constexpr bool CACHE_OK = MMA;
  static_assert(!MMA || R * KS >= KB * US, "the scaled rotation fits the split buffer");
  const bool cached = CACHE_OK && ycg != nullptr && r <= 32;
  float2* Us = Yc2;  // the split-k buffer the tensor path does not use
  const int nbz = (r + 15) >> 4;
  constexpr int YPT = MMA ? R * KB / kSubNT : 1;  // cached elements per thread
  float2 ypre[YPT];
  auto ycache_fetch = [&](int i0) {
#pragma unroll
    for (int q = 0; q < YPT; ++q) {
      const int t = tid + NT * q, i = t / KB, j = t - i * KB;
      ypre[q] = (i0 + i < e) ? __ldcg(ycg + (long long)(i0 + i) * KB + j) : make_float2(0.f, 0.f);
    }
  };
  if (cached) {
    static_assert(!MMA || R * KB == YPT * kSubNT, "whole cached elements per thread");
    for (int t = tid; t < KB * KB; t += NT) {
      const int j = t / KB, c = t - j * KB;
      const int pc = perm[c];
      if (pc < US) Us[j * US + pc] = cscale(C[j * KS + c], S.f[pc]);
    }
    ycache_fetch(0);
  }
  __syncthreads();
  if (stg) stage_d_async(Ds, Dg, 0, min(R, e), d);
  for (int i0 = 0; i0 < e; i0 += R) {
    const int rows = min(R, e - i0);
    if (cached) {  // Yc is free (the previous chunk's Z GEMM is behind a barrier)
#pragma unroll
      for (int q = 0; q < YPT; ++q) {
        const int t = tid + NT * q, i = t / KB, j = t - i * KB;
        Yc[i * KS + j] = ypre[q];
      }
    }
    if (BIG && Dg && i0 + R < e) prefetch_l2(Dg + (long long)(i0 + R) * d, min(R, e - i0 - R) * d);
    if (stg) stage_d_wait();
    else if (cached) __syncthreads();
    if (cached) {
      if constexpr (MMA) {
        if (i0 + R < e) ycache_fetch(i0 + R);
        ycache_rotate_mma<KS, US>(Yc, Us, nbz);
      }
    } else {
    if (BIG) build_chunk_big<DP, CS, R>(C, F, spg, wl, weighted, lofs, Dg, i0, rows, prm.inv_beta);
    else build_chunk<DP, CS, R>(C, wl, lofs, F, Dg ? Ds : nullptr, i0, rows, prm.inv_beta);
    __syncthreads();
    }
    if (!cached) {
      // only the first r (sorted) Ritz columns have f > 0 (Z1 mode: the
      // leading kDeflateK)
      static_assert(NC <= 4, "NC > 4 needs more cases");
      const int nb = ((to_defl ? DSTEP : r) + 15) >> 4;
      if constexpr (HUGE) chunk_block_huge<CS, KS, R>(C, Vf, Yc, d, min(KB, 16 * nb), S.f);
      else if constexpr (MMA) {
        if (nb <= 1) chunk_block_mma<CS, KS, 1, R>(C, Vf, Yc, Yc2, d, S.f);
        else if (nb == 2 || NC == 2) chunk_block_mma<CS, KS, 2, R>(C, Vf, Yc, Yc2, d, S.f);
        else chunk_block_mma<CS, KS, (NC >= 3 ? 3 : 2), R>(C, Vf, Yc, Yc2, d, S.f);
      }
      else if (nb <= 1) chunk_block<CS, KS, 1, R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
      else if (nb == 2 || NC == 2) chunk_block<CS, KS, (NC >= 2 ? 2 : 1), R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
      else if (nb == 3 || NC == 3) chunk_block<CS, KS, (NC >= 3 ? 3 : 1), R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
      else chunk_block<CS, KS, NC, R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
    }
    {
      // Z[zr][k] = sum_{j < r} Yc[zr][j] conj(Vf[k][j]), then the dual update
      // and T = Z - D/beta into the chunk buffer for the adjoint
      const int rz = to_defl ? DSTEP : r;
      // dpre: the dual element, when the caller already loaded it (large-d layout)
      auto finish = [&](int zr, int k, float2 z, const float2* dpre = nullptr) {
        if (!(zr < rows && k < d)) return;
        if (to_defl) {  // Z1 only (accumulated along the chain): level 3 finishes this matrix
          float2* z1p = F.Z1 + (long long)mat * e * d + (long long)(i0 + zr) * d + k;
          *z1p = defl3 ? cadd(__ldcg(z1p), z) : z;
          return;
        }
        if (defl3) {
          const float2 z1 = __ldcg(F.Z1 + (long long)mat * e * d + (long long)(i0 + zr) * d + k);
          z.x += z1.x;
          z.y += z1.y;
        }
        float2 tv = z;
        if (admm) {
          const float2 L = BIG ? (F.wide ? lift_global(F, spg, wl, weighted, lofs[i0 + zr], k)
                                         : cconj(lift_global(F, spg, wl, weighted, lofs[k], i0 + zr)))
                               : lift_tab(wl, lofs, F.wide, i0 + zr, k);
          const long long gi = (long long)(i0 + zr) * d + k;
          float2 dn = BIG ? (dpre ? *dpre : __ldcg(Dg + gi)) : Ds[zr * d + k];
          dn.x = fmaf(prm.tau_dual, L.x - z.x, dn.x);
          dn.y = fmaf(prm.tau_dual, L.y - z.y, dn.y);
          Dg[gi] = dn;
          tv.x = fmaf(-dn.x, prm.inv_beta, z.x);
          tv.y = fmaf(-dn.y, prm.inv_beta, z.y);
        }
        C[zr * CS + k] = tv;
      };
      if constexpr (MMA) {
        // all reads of the chunk (the GEMM above) are behind chunk_block_mma's barrier
        ZAccMma zm;
        zgemm_mma<DP, KS>(zm, Yc, Vf, (rz + 7) >> 3);
        // through the chunk buffer, so the dual update below walks rows
        // contiguously (coalesced dual stores, conflict-free lifts)
        zm.for_each<DP>([&](int zr, int k, float2 z) {
          if (k < DP) C[zr * CS + k] = z;
        });
        __syncthreads();
        if (BIG && admm) {
          // duals straight from HBM / L2: four loads in flight per thread
          for (int t0 = tid; t0 < rows * d; t0 += 4 * NT) {
            float2 dp4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int t = t0 + q * NT;
              dp4[q] = t < rows * d ? __ldcg(Dg + (long long)i0 * d + t) : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int t = t0 + q * NT;
              if (t < rows * d) {
                const int zr = t / d, k = t - zr * d;
                finish(zr, k, C[zr * CS + k], &dp4[q]);
              }
            }
          }
        } else {
          for (int t = tid; t < rows * d; t += NT) {
            const int zr = t / d, k = t - zr * d;
            finish(zr, k, C[zr * CS + k]);
          }
        }
      } else {
        constexpr int MZ = (DP + ZC - 1) / ZC;
        const int zr = tid / ZC, zc = tid % ZC;
        float2 z[MZ];
#pragma unroll
        for (int m = 0; m < MZ; ++m) z[m] = make_float2(0.f, 0.f);
        for (int j = 0; j < rz; ++j) {
          const float2 yv = Yc[zr * KS + j];
#pragma unroll
          for (int m = 0; m < MZ; ++m) {
            const int k = zc + ZC * m;
            if (k < DP) cfmac(z[m], Vf[k * KS + j], yv);  // yv * conj(V[k][j])
          }
        }
#pragma unroll
        for (int m = 0; m < MZ; ++m) finish(zr, zc + ZC * m, z[m]);
      }
    }
    __syncthreads();
    if (stg && i0 + R < e) stage_d_async(Ds, Dg, i0 + R, min(R, e - i0 - R), d);  // overlaps the adjoint
    if (to_defl) {
      // Z1 mode: no duals, no adjoint (level 3 finishes the matrix)
    } else if (BIG && !F.wide) {
      // tall: out_b[n] += sum_i T[i][b q + n - i] over this chunk's rows,
      // read-modify-write of the CTA's own output region.  Weighted lifts
      // apply the adjoint weighting to the chunk's partial sums (it is linear
      // per n): regular block b adds conj(wc[n]) s at (n, coil b); after a
      // barrier, virtual-coil block b adds wc[n] conj(s) at (dagger(n), coil
      // b - J), the same output slots (adjoint_lift_weighted,
      // operators.cpp:60-91)
      const int q = F.q;
      float2* op = F.out + (long long)mat * F.o_mat;
      const int nlo = i0, nhi = min(len - 1, i0 + rows - 1 + q - 1);
      const int span = nhi - nlo + 1;
      const int npass = (weighted && F.vc) ? 2 : 1;
      for (int pass = 0; pass < npass; ++pass) {
        for (int o = tid; o < B * span; o += NT) {
          const int b = o / span, n = nlo + o % span;
          const bool vcb = weighted && F.vc && b >= J;
          if (vcb != (pass == 1)) continue;
          const int ilo = max(i0, n - q + 1), ihi = min(i0 + rows - 1, n);
          float2 sacc = make_float2(0.f, 0.f);
          for (int i = ilo; i <= ihi; ++i) sacc = cadd(sacc, C[(i - i0) * CS + b * q + (n - i)]);
          if (!weighted) {
            float2* dst = op + (long long)n * F.o_n + (long long)b * F.o_j;
            *dst = cadd(*dst, sacc);
          } else if (!vcb) {
            float2* dst = op + (long long)n * F.o_n + (long long)b * F.o_j;
            *dst = cadd(*dst, cmulc(wl[n], sacc));
          } else {
            float2* dst = op + (long long)dagger_src(n, len) * F.o_n + (long long)(b - J) * F.o_j;
            *dst = cadd(*dst, cmul(wl[n], cconj(sacc)));
          }
        }
        __syncthreads();
      }
    } else if (BIG) {
      // blocks b_lo..b_hi touch this chunk; a block whose rows continue into
      // the next chunk is carried (acc[par]), the one carried in from the
      // previous chunk is acc[par ^ 1]; complete blocks are weighted and
      // stored -- regular blocks first, then (after a barrier) the
      // virtual-coil blocks, which add into the regular blocks' output
      // (adjoint_lift_weighted, operators.cpp:60-91)
      const int q = F.q, P = F.P;
      const int b_lo = i0 / q, b_hi = (i0 + rows - 1) / q;
      const int par = (i0 / R) & 1;
      const bool carried_in = i0 > 0 && (i0 % q) != 0;  // block b_lo started in the previous chunk
      float2* op = F.out + (long long)mat * F.o_mat;
      for (int pass = 0; pass < 2; ++pass) {
        for (int o = tid; o < (b_hi - b_lo + 1) * len; o += NT) {
          const int b = b_lo + o / len, n = o % len;
          const bool vcb = weighted && F.vc && b >= J;
          if (vcb != (pass == 1)) continue;
          float2 sacc = (b == b_lo && carried_in) ? acc[(par ^ 1) * len + n] : make_float2(0.f, 0.f);
          const int tlo = max(max(0, i0 - b * q), n - P + 1);
          const int thi = min(min(q - 1, i0 + rows - 1 - b * q), n);
          for (int t = tlo; t <= thi; ++t) sacc = cadd(sacc, cconj(C[(b * q + t - i0) * CS + (n - t)]));
          if ((b + 1) * q - 1 > i0 + rows - 1) {  // continues into the next chunk
            acc[par * len + n] = sacc;
          } else if (!weighted) {
            op[(long long)n * F.o_n + (long long)b * F.o_j] = sacc;
          } else if (!vcb) {
            op[(long long)n * F.o_n + (long long)b * F.o_j] = cmulc(wl[n], sacc);
          } else {
            const int fl = dagger_src(n, len);
            float2* dst = op + (long long)fl * F.o_n + (long long)(b - J) * F.o_j;
            *dst = cadd(*dst, cmul(wl[n], cconj(sacc)));
          }
        }
        __syncthreads();
      }
    } else {
    for (int o = tid; o < B * len; o += NT) {
      const int b = o / len, n = o - b * len;
      float2 s = acc[o];
      if (!F.wide) {
        const int ilo = max(i0, n - F.q + 1), ihi = min(i0 + rows - 1, n);
        for (int i = ilo; i <= ihi; ++i) s = cadd(s, C[(i - i0) * CS + b * F.q + (n - i)]);
      } else {
        const int tlo = max(max(0, i0 - b * F.q), n - F.P + 1);
        const int thi = min(min(F.q - 1, i0 + rows - 1 - b * F.q), n);
        for (int t = tlo; t <= thi; ++t) s = cadd(s, cconj(C[(b * F.q + t - i0) * CS + (n - t)]));
      }
      acc[o] = s;
    }
    __syncthreads();
    }
  }
  SUB_STAMP(7);
#undef SUB_STAMP

  // ---------------------------------------------------------- weighting + store
  if (!BIG) {
    float2* op = F.out + (long long)mat * F.o_mat;
    for (int t = tid; t < J * len; t += NT) {
      const int j = t / len, n = t - j * len;
      float2 v = acc[j * len + n];
      if (weighted) {
        v = cmulc(F.wc[n], v);
        if (F.vc) {
          const int fl = dagger_src(n, len);
          v = cadd(v, cmul(F.wc[fl], cconj(acc[(J + j) * len + fl])));
        }
      }
      op[n * F.o_n + j * F.o_j] = v;
    }
  }
}


namespace {
template <int DP, int KB, bool BIG, bool L2, int MINB = 1, bool MMA = false>
void launch_sub(const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    SHLR_CUDA(cudaFuncSetAttribute(svt_subspace_kernel<DP, KB, 32, BIG, L2, MINB, MMA>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = true;
  }
  svt_subspace_kernel<DP, KB, 32, BIG, L2, MINB, MMA><<<total, kSubNT, smem, stream>>>(prm);
  SHLR_LAUNCH_CHECK();
}
}  // namespace

}  // namespace shlr_b200
