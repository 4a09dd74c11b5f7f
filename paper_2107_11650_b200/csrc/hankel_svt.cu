// Fused batched Hankel-SVT kernel (see hankel_svt.cuh for the algorithm).
//
// Eigen-solver: cyclic parallel two-sided Jacobi on the d x d Gram in smem
// (Brent-Luk ring ordering), in two stages:
//   stage 1 (cold start only)  G  = Ahat^H Ahat               -> V1
//   stage 2 (always)           G2 = (Ahat V1)^H (Ahat V1)      -> V = V1 V2
// Stage 2 recovers the accuracy the FP32 Gram loses on small singular values
// (G2's entries are accurate relative to sigma_i sigma_j) and is also the
// ADMM warm start: V1 = the eigenvectors this matrix had in the previous
// outer iteration (kept in HBM), so a warm launch skips the Gram and stage 1.
// The Gram diagonal is carried in FP64 (it is updated once per round).
#include <algorithm>
#include <type_traits>
#include <string>

#include <cuda_pipeline.h>

#include "hankel_svt.cuh"

#include <cstdlib>

namespace shlr_b200 {

namespace {

// Stage 1 (loose: stage 2 refines) and stage 2 (tight) rotation thresholds:
// rotate iff |g_ab| > tol_rel sqrt(g_aa g_bb) and |g_ab| > tol_abs max_u g_uu.
constexpr float kTolRel1 = 1.0e-5f;
constexpr float kTolAbs1 = 1.0e-7f;
constexpr float kTolAbsRR = 1.0e-6f;  // Rayleigh-Ritz absolute floor (x max Ritz value)
constexpr float kTolRel2 = 2.0e-6f;
constexpr int kRitzMaxSweeps = 8;  // Rayleigh-Ritz Jacobi sweep cap (subspace solver)

struct __align__(16) SlotRec {
  int a, b, flag, pad;  // storage indices of the pair, 1 = non-identity rotation
  float c, sn;          // cos, sin
  float2 cw;            // c * conj(phase)
  float2 sw;            // s * conj(phase)
  float pad2[2];
};

__device__ __forceinline__ int ring_idx(int k, int r, int DP) {
  const int v = k - r;
  return v < 0 ? v + DP - 1 : v;
}
__device__ __forceinline__ int top_of(int s, int r, int DP) {
  return s == 0 ? DP - 1 : ring_idx(s - 1, r, DP);
}
__device__ __forceinline__ int bot_of(int s, int r, int DP) { return ring_idx(DP - 2 - s, r, DP); }
// storage column held by slot s at round 0 (the arrangement after a sweep)
__device__ __forceinline__ int top0(int s, int DP) { return s == 0 ? DP - 1 : s - 1; }
__device__ __forceinline__ int bot0(int s, int DP) { return DP - 2 - s; }

__device__ __forceinline__ const SvtFamily& family_of(const SvtParams& p, int blk, int& local) {
  if (p.nfam > 1 && blk >= p.fam[0].count) {
    local = blk - p.fam[0].count;
    return p.fam[1];
  }
  local = blk;
  return p.fam[0];
}

// Lifted element L at (row i of Ahat, storage column u) from the staged
// weighted spectra wl[b * len + n].
__device__ __forceinline__ float2 lift_elem(const float2* wl, const SvtFamily& F, int i, int u) {
  if (!F.wide) {
    const int b = u / F.q, t = u - b * F.q;
    return wl[b * F.len + i + t];
  } else {
    const int b = i / F.q, t = i - b * F.q;
    return cconj(wl[b * F.len + u + t]);
  }
}

// Shared state of one CTA.
template <int DP>
struct Smem {
  float2* G;     // DP x (DP+1): Gram / V1 / G2 / W (off-diagonal upper repr. in Jacobi)
  double* dg;    // DP: diagonal of G (fp64)
  float2* wl;    // B x len weighted spectra
  float2* acc;   // B x len adjoint accumulators
  float2* A;     // R x DP chunk of Ahat (also V panel staging)
  float2* X;     // R x DP chunk of D / B = Ahat V1 / T
  SlotRec* rec;  // 2 x S (current / next round)
  double2* dgr;  // 2 x S diagonal entries (a, b) of each slot after its rotation
  float* f;      // DP shrink factors
  int* flags;    // 4
  float* scal;   // 4
};

// Ahat chunk rows [i0, i0 + rows) into S.A (zero padded to R x DP); with
// want_d the raw D rows go to S.X.
template <int DP, int R>
__device__ __forceinline__ void load_chunk(const Smem<DP>& S, const SvtFamily& F, const float2* Dg,
                                           int i0, int rows, float inv_beta, bool want_d) {
  const int d = F.d;
  for (int t = threadIdx.x; t < R * DP; t += blockDim.x) {
    const int r = t / DP, u = t - r * DP;
    float2 v = make_float2(0.f, 0.f), dd = make_float2(0.f, 0.f);
    if (r < rows && u < d) {
      v = lift_elem(S.wl, F, i0 + r, u);
      if (Dg) {
        dd = Dg[(long long)(i0 + r) * d + u];
        v.x = fmaf(dd.x, inv_beta, v.x);
        v.y = fmaf(dd.y, inv_beta, v.y);
      }
    }
    S.A[t] = v;
    if (want_d) S.X[t] = dd;
  }
}

// Same as load_chunk, into an explicit R x DP buffer (no D copy).
template <int DP, int R>
__device__ __forceinline__ void load_chunk_to(float2* dst, const float2* wl, const SvtFamily& F,
                                              const float2* Dg, int i0, int rows, float inv_beta) {
  const int d = F.d;
  for (int t = threadIdx.x; t < R * DP; t += blockDim.x) {
    const int r = t / DP, u = t - r * DP;
    float2 v = make_float2(0.f, 0.f);
    if (r < rows && u < d) {
      v = lift_elem(wl, F, i0 + r, u);
      if (Dg) {
        const float2 dd = Dg[(long long)(i0 + r) * d + u];
        v.x = fmaf(dd.x, inv_beta, v.x);
        v.y = fmaf(dd.y, inv_beta, v.y);
      }
    }
    dst[t] = v;
  }
}

// Asynchronous copy (cp.async, L2 -> smem) of the dual rows [i0, i0 + rows)
// of one matrix -- rows * d contiguous complex64 in HBM -- into `stage`.
// The caller waits with stage_d_wait() before reading it.
__device__ __forceinline__ void stage_d_async(float2* stage, const float2* Dg, int i0, int rows, int d) {
  const float2* src = Dg + (long long)i0 * d;
  const int cnt = rows * d;
  const bool al16 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(stage)) & 15) == 0;
  if (al16) {
    const int n16 = cnt >> 1;
    for (int t = threadIdx.x; t < n16; t += blockDim.x) __pipeline_memcpy_async(stage + 2 * t, src + 2 * t, 16);
    if ((cnt & 1) && threadIdx.x == 0) __pipeline_memcpy_async(stage + cnt - 1, src + cnt - 1, 8);
  } else {
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) __pipeline_memcpy_async(stage + t, src + t, 8);
  }
  __pipeline_commit();
}
__device__ __forceinline__ void stage_d_wait() {
  __pipeline_wait_prior(0);
  __syncthreads();
}

// Ahat chunk rows [i0, i0 + rows) into dst (R x DP, zero padded) from the
// smem spectra and the staged duals (row stride d), or without duals.
// lofs: per-index spectrum offsets (b * len + t of index = b * q + t) over the
// lifted matrix's block index (columns of A when tall, rows of A^H when wide).
__device__ __forceinline__ float2 lift_tab(const float2* wl, const int* lofs, bool wide, int i, int u) {
  return wide ? cconj(wl[lofs[i] + u]) : wl[lofs[u] + i];
}

template <int DP, int CS, int R>
__device__ __forceinline__ void build_chunk(float2* dst, const float2* wl, const int* lofs, const SvtFamily& F,
                                            const float2* dstage, int i0, int rows, float inv_beta) {
  const int d = F.d;
  const bool wide = F.wide;
  for (int t = threadIdx.x; t < R * DP; t += blockDim.x) {
    const int r = t / DP, u = t - r * DP;
    float2 v = make_float2(0.f, 0.f);
    if (r < rows && u < d) {
      v = lift_tab(wl, lofs, wide, i0 + r, u);
      if (dstage) {
        const float2 dd = dstage[r * d + u];
        v.x = fmaf(dd.x, inv_beta, v.x);
        v.y = fmaf(dd.y, inv_beta, v.y);
      }
    }
    dst[r * CS + u] = v;
  }
}

// Large-d (BIG) subspace variant, wide families only (Ahat = A^H): the lifted
// spectra are not staged in shared memory -- element (c, u) of Ahat is
// conj(wl_b[t + u]) with (b, t) = lofs[c] (packed b << 16 | t), read from
// the global spectra (L2-resident) with the weighting wc (smem copy `wcs`)
// and the virtual-coil dagger applied on the fly (lift_weighted,
// operators.cpp:36-56).
__device__ __forceinline__ float2 lift_global(const SvtFamily& F, const float2* __restrict__ sp,
                                              const float2* wcs, bool weighted, int bt, int u) {
  const int b = bt >> 16, n = (bt & 0xffff) + u;
  float2 v;
  if (b < F.J) {
    v = __ldg(sp + (long long)n * F.s_n + (long long)b * F.s_j);
    if (weighted) v = cmul(wcs[n], v);
  } else {
    const int fl = dagger_src(n, F.len);
    v = cmul(wcs[n], cconj(__ldg(sp + (long long)fl * F.s_n + (long long)(b - F.J) * F.s_j)));
  }
  return cconj(v);
}

template <int DP, int CS, int R>
__device__ __forceinline__ void build_chunk_big(float2* dst, const SvtFamily& F, const float2* __restrict__ sp,
                                                const float2* wcs, bool weighted, const int* lofs,
                                                const float2* __restrict__ Dg, int i0, int rows, float inv_beta) {
  const int d = F.d;
  for (int t = threadIdx.x; t < R * DP; t += blockDim.x) {
    const int r = t / DP, u = t - r * DP;
    float2 v = make_float2(0.f, 0.f);
    if (r < rows && u < d) {
      v = F.wide ? lift_global(F, sp, wcs, weighted, lofs[i0 + r], u)
                 : cconj(lift_global(F, sp, wcs, weighted, lofs[u], i0 + r));  // tall: Ahat = A
      if (Dg) {  // duals straight from HBM/L2 (coalesced rows)
        const float2 dd = __ldcg(Dg + (long long)(i0 + r) * d + u);
        v.x = fmaf(dd.x, inv_beta, v.x);
        v.y = fmaf(dd.y, inv_beta, v.y);
      }
    }
    dst[r * CS + u] = v;
  }
}

// Yc = C B over all 512 threads: the k range is split in two halves (threads
// 0-255 -> Yc, 256-511 -> Yc2), each half a 2 x NB register tile per thread
// (2 + NB shared loads per 2 NB complex FMAs).  The caller sums the halves
// (sum_halves) after a barrier.
template <int DP, int KS, int NB>
__device__ __forceinline__ void chunk_times_block_split(const float2* C, const float2* Bm, float2* Yc,
                                                        float2* Yc2, int d) {
  const int h = threadIdx.x >> 8, t = threadIdx.x & 255;
  const int r2 = (t >> 4) * 2, c16 = t & 15;
  const int dh = (d + 1) >> 1;
  const int kb = h ? dh : 0, ke = h ? d : dh;
  float2 y0[NB], y1[NB];
#pragma unroll
  for (int n = 0; n < NB; ++n) y0[n] = y1[n] = make_float2(0.f, 0.f);
  const float2* c0 = C + r2 * DP;
  const float2* c1 = c0 + DP;
#pragma unroll 4
  for (int k = kb; k < ke; ++k) {
    const float2 a0 = c0[k], a1 = c1[k];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      const float2 b = Bm[k * KS + c16 + 16 * n];
      cfma(y0[n], a0, b);
      cfma(y1[n], a1, b);
    }
  }
  float2* out = h ? Yc2 : Yc;
#pragma unroll
  for (int n = 0; n < NB; ++n) {
    out[r2 * KS + c16 + 16 * n] = y0[n];
    out[(r2 + 1) * KS + c16 + 16 * n] = y1[n];
  }
}
template <int KS, int R>
__device__ __forceinline__ void sum_halves(float2* Yc, const float2* Yc2, int ncols, const float* scale) {
  for (int t = threadIdx.x; t < R * ncols; t += blockDim.x) {
    const int r = t / ncols, c = t - r * ncols;
    const float sc = scale ? scale[c] : 1.f;
    Yc[r * KS + c] = cscale(cadd(Yc[r * KS + c], Yc2[r * KS + c]), sc);
  }
}

// Chunk GEMM Yc = C B (columns 16 NB), optionally column-scaled; the split-k
// form needs the second buffer Yc2, the NOSPLIT form (large block, no room
// for Yc2) runs on the first 256 threads.  Ends with a barrier.
template <int CS, int KS, int NB, int R, bool NOSPLIT>
__device__ __forceinline__ void chunk_block(const float2* C, const float2* Bm, float2* Yc, float2* Yc2, int d,
                                            const float* scale);

// Yc (rows r2, r2+1 of the chunk; columns c16 + 16 n, n < NB) = C B for the
// first 256 threads (2 x NB register tiles: 2 + NB shared loads per 2 NB
// complex FMAs), optionally column-scaled.
template <int DP, int KS, int NB>
__device__ __forceinline__ void chunk_times_block(const float2* C, const float2* Bm, float2* Yc, int d,
                                                  const float* scale) {
  const int tid = threadIdx.x;
  if (tid >= 256) return;
  const int r2 = (tid >> 4) * 2, c16 = tid & 15;
  float2 y0[NB], y1[NB];
#pragma unroll
  for (int n = 0; n < NB; ++n) y0[n] = y1[n] = make_float2(0.f, 0.f);
  const float2* c0 = C + r2 * DP;
  const float2* c1 = c0 + DP;
#pragma unroll 2
  for (int k = 0; k < d; ++k) {
    const float2 a0 = c0[k], a1 = c1[k];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      const float2 b = Bm[k * KS + c16 + 16 * n];
      cfma(y0[n], a0, b);
      cfma(y1[n], a1, b);
    }
  }
#pragma unroll
  for (int n = 0; n < NB; ++n) {
    const float sc = scale ? scale[c16 + 16 * n] : 1.f;
    Yc[r2 * KS + c16 + 16 * n] = cscale(y0[n], sc);
    Yc[(r2 + 1) * KS + c16 + 16 * n] = cscale(y1[n], sc);
  }
}

template <int CS, int KS, int NB, int R, bool NOSPLIT>
__device__ __forceinline__ void chunk_block(const float2* C, const float2* Bm, float2* Yc, float2* Yc2, int d,
                                            const float* scale) {
  if constexpr (NOSPLIT) {
    chunk_times_block<CS, KS, NB>(C, Bm, Yc, d, scale);
    __syncthreads();
  } else {
    chunk_times_block_split<CS, KS, NB>(C, Bm, Yc, Yc2, d);
    __syncthreads();
    sum_halves<KS, R>(Yc, Yc2, 16 * NB, scale);
    __syncthreads();
  }
}

// Gram-type accumulation acc[m][c] += sum_r conj(src[r][kq+8m]) src[r][l0+c].
template <int DP, int W>
__device__ __forceinline__ void gram_accumulate(const float2* src, int rows, int kq, int l0,
                                                float2 (&g0)[W], float2 (&g1)[W]) {
  for (int r = 0; r < rows; ++r) {
    const float2* row = src + r * DP;
    const float2 b0 = row[l0], b1 = row[l0 + 1];
#pragma unroll
    for (int m = 0; m < W; ++m) {
      const float2 a = row[kq + 8 * m];
      cfmac(g0[m], a, b0);
      cfmac(g1[m], a, b1);
    }
  }
}

// Gram tile entries (k, l0) and (k, l0+1) into the full Hermitian storage:
// the upper-triangle value is written to both (k, l) and conj to (l, k), the
// real diagonal to S.dg.
template <int DP>
__device__ __forceinline__ void store_gram_pair(const Smem<DP>& S, int k, int l0, float2 g0, float2 g1) {
  constexpr int GS = DP + 1;
  if (k < l0) {
    S.G[k * GS + l0] = g0;
    S.G[l0 * GS + k] = cconj(g0);
  }
  if (k < l0 + 1) {
    S.G[k * GS + l0 + 1] = g1;
    S.G[(l0 + 1) * GS + k] = cconj(g1);
  }
  if (k == l0) S.dg[k] = g0.x;
  if (k == l0 + 1) S.dg[k] = g1.x;
}

// out[kq+8m][l0..l0+1] = sum_k A[kq+8m][k] * Bm[k][l0..l0+1], k < kmax.
template <int DP, int RM>
__device__ __forceinline__ void chunk_gemm(const float2* A, const float2* Bm, int kmax, int kq, int l0,
                                           float2 (&z0)[RM], float2 (&z1)[RM]) {
  constexpr int GS = DP + 1;
#pragma unroll
  for (int m = 0; m < RM; ++m) z0[m] = z1[m] = make_float2(0.f, 0.f);
  for (int k = 0; k < kmax; ++k) {
    const float2 w0 = Bm[k * GS + l0], w1 = Bm[k * GS + l0 + 1];
#pragma unroll
    for (int m = 0; m < RM; ++m) {
      const float2 a = A[(kq + 8 * m) * DP + k];
      cfma(z0[m], a, w0);
      cfma(z1[m], a, w1);
    }
  }
}

// Rotation that annihilates g = G[a][b] given the current diagonal entries
// (al, be): rotate iff |g| > tol_rel sqrt(al be), |g| > tol_abs and not both
// al, be < tail (pairs inside a tail whose shrink factor is 0 either way).
__device__ __forceinline__ bool make_rotation(SlotRec& rc, double2& nd, int a, int b, double al,
                                              double be, float2 gm, float tol_rel, float tol_abs,
                                              float tail) {
  rc.a = a;
  rc.b = b;
  rc.flag = 0;
  rc.c = 1.f;
  rc.sn = 0.f;
  rc.cw = make_float2(1.f, 0.f);
  rc.sw = make_float2(0.f, 0.f);
  nd = make_double2(al, be);
  const float g = hypotf(gm.x, gm.y);
  const float alf = (float)al, bef = (float)be;
  if (!(g > 0.f && g > tol_abs && g > tol_rel * sqrtf(fmaxf(alf * bef, 0.f)))) return false;
  if (alf < tail && bef < tail) return false;
  // fp64 angle: with fp32 the accumulated diagonal/angle mismatch costs ~10x
  // in the final singular values (measured)
  const double zeta = (be - al) / (2.0 * (double)g);
  const double az = fabs(zeta);
  double t = 1.0 / (az + sqrt(1.0 + az * az));
  t = zeta < 0.0 ? -t : t;
  const double ci = 1.0 / sqrt(1.0 + t * t);
  const float2 ph = make_float2(gm.x / g, -gm.y / g);  // conj(g)/|g|
  rc.c = (float)ci;
  rc.sn = (float)(t * ci);
  rc.cw = cscale(ph, rc.c);
  rc.sw = cscale(ph, rc.sn);
  nd = make_double2(al - t * (double)g, be + t * (double)g);
  rc.flag = 1;
  return true;
}

// Parallel cyclic Jacobi on S.G (off-diagonal, upper representation) and
// S.dg (diagonal, fp64) with V held in registers (vt/vb, 4 threads per row).
//
// One barrier per round: the rotation of slot s for round r+1 pairs
// (top_r(s-1), bot_r(s+1)) -- an element of block (s-1, s+1) of round r --
// so the thread that updates that block computes the next rotation on the
// spot (diagonal entries come from the round-r rotation records).  Special
// cases: slot 0 <- block (0,1) element (top0, bot1); slot 1 <- block (0,2)
// element (bot0, bot2); slot S-1 <- block (S-2,S-1) element (top, top).
// Returns the number of sweeps; the final diagonal is written to S.dg.
template <int DP, int W>
__device__ int jacobi(const Smem<DP>& S, float2 (&vt)[W], float2 (&vb)[W], float tol_rel,
                      float tol_abs, int max_sweeps, float tail = 0.f) {
  constexpr int NT = 4 * DP;
  constexpr int S_ = DP / 2;
  constexpr int GS = DP + 1;
  const int tid = threadIdx.x;
  const int vg = tid & 3;
  // Work items q = tid + k*NT: items 0..S-1 are the S rotation-carrying
  // blocks (threads 0..S-1, i.e. the first warps only, so the rotation math
  // does not diverge every warp); the remaining off-diagonal blocks follow in
  // row-major order (consecutive lanes -> consecutive s2 -> conflict-free).
  constexpr int NOFF = S_ * (S_ - 1) / 2;
  constexpr int NBT = (NOFF + NT - 1) / NT;
  int blk_code[NBT];  // s1 | s2 << 8 | (carrier + 1) << 16, or -1
#pragma unroll
  for (int k = 0; k < NBT; ++k) {
    const int q = tid < NT ? tid + k * NT : NOFF;  // threads >= 4*DP only join barriers
    int s1 = -1, s2 = -1, cr = -1;
    if (q < S_) {
      const int s = q;
      if (s == 0) {
        s1 = 0; s2 = 1; cr = 0;
      } else if (s == 1) {
        s1 = 0; s2 = 2; cr = (1 << 2) | 1;
      } else if (s == S_ - 1) {
        s1 = S_ - 2; s2 = S_ - 1; cr = ((S_ - 1) << 2) | 2;
      } else {
        s1 = s - 1; s2 = s + 1; cr = s << 2;
      }
    } else if (q < NOFF) {
      // j-th non-carrying block in row-major order
      int j = q - S_;
      for (int row = 0; row < S_ - 2; ++row) {
        const int first = row == 0 ? 3 : row + 1;             // row 0 skips (0,1),(0,2)
        const int cnt = row == 0 ? S_ - 3 : S_ - 2 - row;      // rows >= 1 skip (row,row+2)
        if (j < cnt) {
          s1 = row;
          s2 = first + j;
          if (row >= 1 && s2 >= row + 2) ++s2;
          break;
        }
        j -= cnt;
      }
    }
    blk_code[k] = s1 < 0 ? -1 : (s1 | (s2 << 8) | ((cr + 1) << 16));
  }
  // rotations of round 0 of the first sweep
  if (tid < S_) {
    const int a = top_of(tid, 0, DP), b = bot_of(tid, 0, DP);
    const int lo = min(a, b), hi = max(a, b);
    float2 gm = S.G[lo * GS + hi];
    if (a > b) gm.y = -gm.y;
    SlotRec rc;
    double2 nd;
    if (make_rotation(rc, nd, a, b, S.dg[a], S.dg[b], gm, tol_rel, tol_abs, tail)) {
      S.G[lo * GS + hi] = make_float2(0.f, 0.f);
      S.flags[0] = 1;
    }
    S.rec[tid] = rc;
    S.dgr[tid] = nd;
  }
  __syncthreads();
  int cur = 0;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int r = 0; r < DP - 1; ++r) {
      const SlotRec* rc = S.rec + cur * S_;
      SlotRec* rn = S.rec + (cur ^ 1) * S_;
      int* next_flag = &S.flags[(r == DP - 2) ? ((sweep + 1) & 1) : (sweep & 1)];
#pragma unroll
      for (int k = 0; k < NBT; ++k) {
        const int code = blk_code[k];
        if (code < 0) continue;
        const int s1 = code & 0xff, s2 = (code >> 8) & 0xff, cr = (code >> 16) - 1;
        const SlotRec& p1 = rc[s1];
        const SlotRec& p2 = rc[s2];
        if (cr < 0 && !(p1.flag | p2.flag)) continue;
        const int x0 = p1.a, x1 = p1.b, y0 = p2.a, y1 = p2.b;
        // upper-representation addresses and conjugation signs
        const int i00 = min(x0, y0) * GS + max(x0, y0), i01 = min(x0, y1) * GS + max(x0, y1);
        const int i10 = min(x1, y0) * GS + max(x1, y0), i11 = min(x1, y1) * GS + max(x1, y1);
        const float s00 = x0 > y0 ? -1.f : 1.f, s01 = x0 > y1 ? -1.f : 1.f;
        const float s10 = x1 > y0 ? -1.f : 1.f, s11 = x1 > y1 ? -1.f : 1.f;
        float2 a00 = S.G[i00], a01 = S.G[i01], a10 = S.G[i10], a11 = S.G[i11];
        a00.y *= s00; a01.y *= s01; a10.y *= s10; a11.y *= s11;
        {  // X J2 (columns); identity parameters are exact
          const float2 n00 = csub(cscale(a00, p2.c), cmul(p2.sw, a01));
          const float2 n01 = cadd(cscale(a00, p2.sn), cmul(p2.cw, a01));
          const float2 n10 = csub(cscale(a10, p2.c), cmul(p2.sw, a11));
          const float2 n11 = cadd(cscale(a10, p2.sn), cmul(p2.cw, a11));
          a00 = n00; a01 = n01; a10 = n10; a11 = n11;
        }
        {  // J1^H X (rows)
          const float2 n00 = csub(cscale(a00, p1.c), cmulc(p1.sw, a10));
          const float2 n10 = cadd(cscale(a00, p1.sn), cmulc(p1.cw, a10));
          const float2 n01 = csub(cscale(a01, p1.c), cmulc(p1.sw, a11));
          const float2 n11 = cadd(cscale(a01, p1.sn), cmulc(p1.cw, a11));
          a00 = n00; a01 = n01; a10 = n10; a11 = n11;
        }
        if (cr >= 0) {  // next-round rotation carried by this block
          const int kind = cr & 3, slot = cr >> 2;
          const double2 d1 = S.dgr[cur * S_ + s1], d2 = S.dgr[cur * S_ + s2];
          const int ra = kind == 1 ? x1 : x0;
          const int rb = kind == 2 ? y0 : y1;
          const double al = kind == 1 ? d1.y : d1.x;
          const double be = kind == 2 ? d2.x : d2.y;
          const float2 gm = kind == 0 ? a01 : (kind == 1 ? a11 : a00);
          SlotRec nr;
          double2 nd;
          if (make_rotation(nr, nd, ra, rb, al, be, gm, tol_rel, tol_abs, tail)) {
            const float2 z = make_float2(0.f, 0.f);
            if (kind == 0) a01 = z;
            if (kind == 1) a11 = z;
            if (kind == 2) a00 = z;
            *next_flag = 1;
          }
          rn[slot] = nr;
          S.dgr[(cur ^ 1) * S_ + slot] = nd;
        }
        a00.y *= s00; a01.y *= s01; a10.y *= s10; a11.y *= s11;
        S.G[i00] = a00; S.G[i01] = a01; S.G[i10] = a10; S.G[i11] = a11;
      }
      // V <- V J on this thread's slots
      if (tid < NT) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const SlotRec& p = rc[vg * W + w];
          if (p.flag) {
            const float2 a = vt[w], b = vb[w];
            vt[w] = csub(cscale(a, p.c), cmul(p.sw, b));
            vb[w] = cadd(cscale(a, p.sn), cmul(p.cw, b));
          }
        }
      }
      __syncthreads();
      cur ^= 1;
      // ring shift of the V columns: tops move right, bottoms move left
      if (tid < NT) {  // whole warps: 4*DP is a multiple of 32
        const float2 up_t = make_float2(__shfl_up_sync(0xffffffffu, vt[W - 1].x, 1, 4),
                                        __shfl_up_sync(0xffffffffu, vt[W - 1].y, 1, 4));
        const float2 up_b = make_float2(__shfl_up_sync(0xffffffffu, vb[0].x, 1, 4),
                                        __shfl_up_sync(0xffffffffu, vb[0].y, 1, 4));
        const float2 dn_b = make_float2(__shfl_down_sync(0xffffffffu, vb[0].x, 1, 4),
                                        __shfl_down_sync(0xffffffffu, vb[0].y, 1, 4));
        float2 nt[W], nb[W];
        if constexpr (W == 1) {
          nt[0] = vg == 0 ? vt[0] : (vg == 1 ? up_b : up_t);
        } else {
          nt[0] = vg == 0 ? vt[0] : up_t;
          nt[1] = vg == 0 ? vb[0] : vt[0];
#pragma unroll
          for (int w = 2; w < W; ++w) nt[w] = vt[w - 1];
        }
#pragma unroll
        for (int w = 0; w < W - 1; ++w) nb[w] = vb[w + 1];
        nb[W - 1] = vg == 3 ? vt[W - 1] : dn_b;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          vt[w] = nt[w];
          vb[w] = nb[w];
        }
      }
    }
    // every rotation of this sweep has been decided (the last round decided
    // round 0 of the next sweep into the other flag)
    const int any = S.flags[sweep & 1];
    __syncthreads();
    if (tid == 0) S.flags[sweep & 1] = 0;
    if (!any) {
      ++sweep;
      break;
    }
  }
  // final diagonal: the pending (identity after convergence) records hold it
  if (tid < S_) {
    const SlotRec& p = S.rec[cur * S_ + tid];
    const double2 nd = S.dgr[cur * S_ + tid];
    S.dg[p.a] = nd.x;
    S.dg[p.b] = nd.y;
  }
  if (tid < 2) S.flags[tid] = 0;
  __syncthreads();
  return sweep;
}

// V (registers, round-0 arrangement) <-> row-major DP x DP storage.
template <int DP, int W>
__device__ __forceinline__ void store_v(float2* dst, int stride, const float2 (&vt)[W],
                                        const float2 (&vb)[W]) {
  const int vrow = threadIdx.x >> 2, vg = threadIdx.x & 3;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int s = vg * W + w;
    dst[vrow * stride + top0(s, DP)] = vt[w];
    dst[vrow * stride + bot0(s, DP)] = vb[w];
  }
}
template <int DP, int W>
__device__ __forceinline__ void load_v(const float2* src, int stride, float2 (&vt)[W], float2 (&vb)[W]) {
  const int vrow = threadIdx.x >> 2, vg = threadIdx.x & 3;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int s = vg * W + w;
    vt[w] = src[vrow * stride + top0(s, DP)];
    vb[w] = src[vrow * stride + bot0(s, DP)];
  }
}

}  // namespace

// Registers per thread when one CTA of 4*DP threads (DP/8 warps) owns the
// SM: each of the 4 sub-partitions holds ceil(warps/4) warps in its 16K-entry
// register file.
constexpr int svt_max_regs(int DP) {
  return (512 / ((DP / 8 + 3) / 4)) / 8 * 8 > 255 ? 255 : (512 / ((DP / 8 + 3) / 4)) / 8 * 8;
}

template <int DP, int R>
__global__ void __maxnreg__(svt_max_regs(DP)) hankel_svt_kernel(const SvtParams prm) {
  // (one CTA per SM: the whole register file is available to its 4*DP threads)
  constexpr int NT = 4 * DP;
  constexpr int S_ = DP / 2;
  constexpr int W = DP / 8;
  constexpr int HALF = DP / 2;
  constexpr int GS = DP + 1;
  constexpr int RM = R / 8;
  static_assert(DP % 8 == 0 && DP >= 8 && DP <= 128, "DP must be a multiple of 8 in [8,128]");
  static_assert(R % 8 == 0, "R must be a multiple of 8");

  if (prm.skip && *prm.skip) return;
  int mat;
  const SvtFamily& F = family_of(prm, blockIdx.x, mat);
  if (F.halt && F.halt[mat / F.halt_div]) return;
  if (prm.only_flagged && (prm.only_flag_value ? F.fallback[mat] != prm.only_flag_value : !F.fallback[mat]))
    return;
  const int tid = threadIdx.x;
  const int d = F.d, e = F.e, len = F.len, B = F.B, J = F.J;
  const bool admm = prm.mode != SVT_PLAIN;
  const bool weighted = prm.mode == SVT_ADMM_WEIGHTED;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<DP> S;
  S.G = reinterpret_cast<float2*>(smem_raw);
  if (prm.wl_global) {  // plain lift of contiguous coil vectors: read the source in place
    S.wl = const_cast<float2*>(F.spec) + (long long)mat * F.s_mat;
    S.acc = S.G + DP * GS;
  } else {
    S.wl = S.G + DP * GS;
    S.acc = S.wl + B * len;
  }
  S.A = S.acc + B * len;
  S.X = S.A + R * DP;
  S.rec = reinterpret_cast<SlotRec*>(S.X + R * DP);
  S.dgr = reinterpret_cast<double2*>(S.rec + 2 * S_);
  S.dg = reinterpret_cast<double*>(S.dgr + 2 * S_);
  S.f = reinterpret_cast<float*>(S.dg + DP);
  S.flags = reinterpret_cast<int*>(S.f + DP);
  S.scal = reinterpret_cast<float*>(S.flags + 4);

  float2* Dg = admm ? F.D + (long long)mat * e * d : nullptr;
  float2* Vg = F.V + (long long)mat * DP * DP;
  const bool warm = prm.warm && *prm.warm;
  const bool exact_sv = F.sv != nullptr;

  // ---------------------------------------------------------- phase 0
  {
    const float2* sp = F.spec + (long long)mat * F.s_mat;
    for (int t = tid; t < (prm.wl_global ? 0 : J * len); t += NT) {
      const int j = t / len, n = t - j * len;
      const float2 s = sp[n * F.s_n + j * F.s_j];
      if (weighted) {
        S.wl[j * len + n] = cmul(F.wc[n], s);
        if (F.vc) {
          const int fl = dagger_src(n, len);
          const float2 sf = sp[fl * F.s_n + j * F.s_j];
          S.wl[(J + j) * len + n] = cmul(F.wc[n], cconj(sf));
        }
      } else {
        S.wl[j * len + n] = s;
      }
    }
    for (int t = tid; t < B * len; t += NT) S.acc[t] = make_float2(0.f, 0.f);
    if (tid < 4) S.flags[tid] = 0;
  }
  __syncthreads();

  const int lp = tid % HALF;   // GEMM column pair -> columns 2lp, 2lp+1
  const int kq = tid / HALF;   // 0..7
  const int l0 = 2 * lp;
  float2 vt[W], vb[W];
  int sweeps1 = 0;

  // ---------------------------------------------------------- stage 1 (cold)
  if (!warm) {
    {
      float2 g0[W], g1[W];
#pragma unroll
      for (int m = 0; m < W; ++m) g0[m] = g1[m] = make_float2(0.f, 0.f);
      for (int i0 = 0; i0 < e; i0 += R) {
        const int rows = min(R, e - i0);
        load_chunk<DP, R>(S, F, Dg, i0, rows, prm.inv_beta, false);
        __syncthreads();
        gram_accumulate<DP, W>(S.A, rows, kq, l0, g0, g1);
        __syncthreads();
      }
#pragma unroll
      for (int m = 0; m < W; ++m) store_gram_pair<DP>(S, kq + 8 * m, l0, g0[m], g1[m]);
    }
    __syncthreads();
    if (tid < 32) {
      double mx = 0.0;
      for (int u = tid; u < DP; u += 32) mx = fmax(mx, S.dg[u]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (tid == 0) S.scal[0] = (float)(kTolAbs1 * mx);
    }
    {
      const int vrow = tid >> 2, vg = tid & 3;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int s = vg * W + w;
        vt[w] = make_float2(vrow == top0(s, DP) ? 1.f : 0.f, 0.f);
        vb[w] = make_float2(vrow == bot0(s, DP) ? 1.f : 0.f, 0.f);
      }
    }
    __syncthreads();
    sweeps1 = jacobi<DP, W>(S, vt, vb, kTolRel1, S.scal[0], prm.max_sweeps);
    // V1 -> smem (refinement GEMM operand) and HBM (reloaded for stage 2)
    store_v<DP, W>(S.G, GS, vt, vb);
    store_v<DP, W>(Vg, DP, vt, vb);
  } else {
    for (int t = tid; t < DP * DP; t += NT) {
      const int k = t / DP, l = t - k * DP;
      S.G[k * GS + l] = Vg[t];
    }
  }
  __syncthreads();

  // ---------------------------------------------------------- refinement: G2 = (Ahat V1)^H (Ahat V1)
  {
    float2 g0[W], g1[W];
#pragma unroll
    for (int m = 0; m < W; ++m) g0[m] = g1[m] = make_float2(0.f, 0.f);
    for (int i0 = 0; i0 < e; i0 += R) {
      const int rows = min(R, e - i0);
      load_chunk<DP, R>(S, F, Dg, i0, rows, prm.inv_beta, false);
      __syncthreads();
      float2 z0[RM], z1[RM];
      chunk_gemm<DP, RM>(S.A, S.G, d, kq, l0, z0, z1);
#pragma unroll
      for (int m = 0; m < RM; ++m) {
        S.X[(kq + 8 * m) * DP + l0] = z0[m];
        S.X[(kq + 8 * m) * DP + l0 + 1] = z1[m];
      }
      __syncthreads();
      gram_accumulate<DP, W>(S.X, rows, kq, l0, g0, g1);
      __syncthreads();
    }
    // V1 is no longer needed in smem: G2 takes its place
#pragma unroll
    for (int m = 0; m < W; ++m) store_gram_pair<DP>(S, kq + 8 * m, l0, g0[m], g1[m]);
  }
  load_v<DP, W>(Vg, DP, vt, vb);  // this thread's own stage-1 / previous-iteration values
  __syncthreads();
  // stage 2: relative criterion (G2 is accurate relative to its entries),
  // optionally with an absolute floor and the below-threshold tail rule
  // (the exact singular-value hook keeps the plain relative criterion)
  float s2_abs = 0.f;
  if (prm.s2_tol_abs > 0.f && !exact_sv) {
    if (tid < 32) {
      double mx = 0.0;
      for (int u = tid; u < DP; u += 32) mx = fmax(mx, S.dg[u]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (tid == 0) S.scal[1] = (float)(prm.s2_tol_abs * mx);
    }
    __syncthreads();
    s2_abs = S.scal[1];
  }
  const int sweeps2 = jacobi<DP, W>(S, vt, vb, kTolRel2, s2_abs, prm.max_sweeps,
                                    exact_sv ? 0.f : prm.s2_tail * prm.thresh * prm.thresh);
  if (prm.sweeps_out && tid == 0) prm.sweeps_out[blockIdx.x] = sweeps1 * 100 + sweeps2;
  store_v<DP, W>(Vg, DP, vt, vb);

  // ---------------------------------------------------------- phase 3: f, W = V f V^H
  {
    for (int u = tid; u < DP; u += NT) {
      const double lam = S.dg[u];
      float f = 0.f;
      if (lam > (double)prm.thresh * prm.thresh && lam > 0.0) f = (float)(1.0 - prm.thresh / sqrt(lam));
      S.f[u] = f;
    }
    __syncthreads();
    if (exact_sv) {
      float* sv = F.sv + (long long)mat * d;
      for (int u = tid; u < d; u += NT) {
        const double su = sqrt(fmax(S.dg[u], 0.0));
        int rank = 0;
        for (int v = 0; v < d; ++v) {
          const double s2 = sqrt(fmax(S.dg[v], 0.0));
          rank += (s2 > su) || (s2 == su && v < u);
        }
        sv[rank] = (float)su;
      }
    }
    for (int t = tid; t < DP * GS; t += NT) S.G[t] = make_float2(0.f, 0.f);
    float2* panel = S.A;  // DP x 2W staging in the chunk buffers
    constexpr int PW = 2 * W;
    const int vrow = tid >> 2, vg = tid & 3;
    for (int g = 0; g < 4; ++g) {
      __syncthreads();
      if (vg == g) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int s = g * W + w;
          panel[vrow * PW + 2 * w] = cscale(vt[w], sqrtf(S.f[top0(s, DP)]));
          panel[vrow * PW + 2 * w + 1] = cscale(vb[w], sqrtf(S.f[bot0(s, DP)]));
        }
      }
      __syncthreads();
#pragma unroll 1
      for (int m = 0; m < W; ++m) {
        const int k = kq + 8 * m;
        const float2* pk = panel + k * PW;
        const float2* pl0 = panel + l0 * PW;
        const float2* pl1 = panel + (l0 + 1) * PW;
        float2 s0 = S.G[k * GS + l0], s1 = S.G[k * GS + l0 + 1];
#pragma unroll
        for (int mm = 0; mm < PW; ++mm) {
          const float2 a = pk[mm];
          cfmac(s0, pl0[mm], a);  // W[k][l] += U[k][m] conj(U[l][m])
          cfmac(s1, pl1[mm], a);
        }
        S.G[k * GS + l0] = s0;
        S.G[k * GS + l0 + 1] = s1;
      }
    }
    __syncthreads();
  }

  // ---------------------------------------------------------- phase 4: Z, D, T, adjoint
  for (int i0 = 0; i0 < e; i0 += R) {
    const int rows = min(R, e - i0);
    load_chunk<DP, R>(S, F, Dg, i0, rows, prm.inv_beta, true);
    __syncthreads();
    float2 z0[RM], z1[RM];
    chunk_gemm<DP, RM>(S.A, S.G, d, kq, l0, z0, z1);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < RM; ++m) {
      S.A[(kq + 8 * m) * DP + l0] = z0[m];
      S.A[(kq + 8 * m) * DP + l0 + 1] = z1[m];
    }
    __syncthreads();
    for (int t = tid; t < R * DP; t += NT) {
      const int r = t / DP, u = t - r * DP;
      if (r < rows && u < d) {
        const float2 z = S.A[t];
        float2 tv = z;
        if (admm) {
          const float2 L = lift_elem(S.wl, F, i0 + r, u);
          float2 dn = S.X[t];
          dn.x = fmaf(prm.tau_dual, L.x - z.x, dn.x);
          dn.y = fmaf(prm.tau_dual, L.y - z.y, dn.y);
          Dg[(long long)(i0 + r) * d + u] = dn;
          tv.x = fmaf(-dn.x, prm.inv_beta, z.x);
          tv.y = fmaf(-dn.y, prm.inv_beta, z.y);
        }
        S.X[t] = tv;
      }
    }
    __syncthreads();
    // anti-diagonal sums (Hankel adjoint), fixed summation order
    for (int o = tid; o < B * len; o += NT) {
      const int b = o / len, n = o - b * len;
      float2 s = S.acc[o];
      if (!F.wide) {
        const int ilo = max(i0, n - F.q + 1), ihi = min(i0 + rows - 1, n);
        for (int i = ilo; i <= ihi; ++i) s = cadd(s, S.X[(i - i0) * DP + b * F.q + (n - i)]);
      } else {
        const int tlo = max(max(0, i0 - b * F.q), n - F.P + 1);
        const int thi = min(min(F.q - 1, i0 + rows - 1 - b * F.q), n);
        for (int t = tlo; t <= thi; ++t) s = cadd(s, cconj(S.X[(b * F.q + t - i0) * DP + (n - t)]));
      }
      S.acc[o] = s;
    }
    __syncthreads();
  }

  // ---------------------------------------------------------- phase 5: weighting + store
  {
    float2* op = F.out + (long long)mat * F.o_mat;
    for (int t = tid; t < J * len; t += NT) {
      const int j = t / len, n = t - j * len;
      float2 v = S.acc[j * len + n];
      if (weighted) {
        v = cmulc(F.wc[n], v);  // conj(wc) * v
        if (F.vc) {
          const int fl = dagger_src(n, len);
          v = cadd(v, cmul(F.wc[fl], cconj(S.acc[(J + j) * len + fl])));
        }
      }
      op[n * F.o_n + j * F.o_j] = v;
    }
  }
}

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
template <int KB, int KS, int DP>
__device__ void householder_qr(float2* M, float2* Q, int d, float* tau) {
  constexpr int T = DP / 8;  // rows per thread
  const int g = threadIdx.x >> 3, s = threadIdx.x & 7;
  static_assert(kSubNT / 8 >= KB, "one 8-thread group per column");
  static_assert(DP % 8 == 0, "DP multiple of 8");
  const int w = g >> 2;
  const int k = g;                 // this group's column
  const bool act = k < KB;
  const bool warp_act = 4 * w < KB;
  float2 col[T];
#pragma unroll
  for (int t = 0; t < T; ++t) col[t] = act ? M[(s + 8 * t) * KS + k] : make_float2(0.f, 0.f);
  // executed by a whole warp (full-mask shuffles); the group owning column j
  // stores reflector j
  auto reflect = [&](int j) {
    float ss = 0.f;
    float2 x0 = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + 8 * t;
      if (row >= j) ss = fmaf(col[t].x, col[t].x, fmaf(col[t].y, col[t].y, ss));
      if (row == j) x0 = col[t];
    }
    ss = group8_sum(ss);
    x0.x = group8_sum(x0.x);  // one lane of the group holds row j
    x0.y = group8_sum(x0.y);
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
        const int row = s + 8 * t;
        M[row * KS + j] = row > j ? cmul(col[t], inv_v0) : make_float2(row == j ? 1.f : 0.f, 0.f);
      }
      if (s == 0) tau[j] = tj;
    }
  };
  if (w == 0) reflect(0);
  __syncthreads();
  for (int j = 0; j < KB; ++j) {
    if (warp_act && 4 * w + 3 > j) {  // warp-uniform: some column k > j in this warp
      float2 part = make_float2(0.f, 0.f);
      float2 v[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        v[t] = M[(s + 8 * t) * KS + j];
        cfmac(part, v[t], col[t]);  // sum conj(v) col
      }
      part.x = group8_sum(part.x);
      part.y = group8_sum(part.y);
      const float2 tw = (act && k > j) ? cscale(part, tau[j]) : make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        col[t].x -= v[t].x * tw.x - v[t].y * tw.y;
        col[t].y -= v[t].x * tw.y + v[t].y * tw.x;
      }
      if (j + 1 < KB && w == ((j + 1) >> 2)) reflect(j + 1);
    }
    __syncthreads();
  }
  // explicit Q = H_0 ... H_{KB-1} [I; 0]: column k of the identity, reflectors
  // backwards (H_j leaves e_k alone for j > k)
#pragma unroll
  for (int t = 0; t < T; ++t) col[t] = make_float2(s + 8 * t == k ? 1.f : 0.f, 0.f);
  if (warp_act) {
    for (int j = min(4 * w + 3, KB - 1); j >= 0; --j) {
      float2 part = make_float2(0.f, 0.f);
      float2 v[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        v[t] = M[(s + 8 * t) * KS + j];
        cfmac(part, v[t], col[t]);
      }
      part.x = group8_sum(part.x);
      part.y = group8_sum(part.y);
      const float2 tw = (act && k >= j) ? cscale(part, tau[j]) : make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        col[t].x -= v[t].x * tw.x - v[t].y * tw.y;
        col[t].y -= v[t].x * tw.y + v[t].y * tw.x;
      }
    }
  }
  if (M == Q) __syncthreads();  // in place: every warp is done reading the reflectors
  if (act) {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int row = s + 8 * t;
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
                                      float care = 0.f, long long* clk = nullptr) {
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

template <int DP, int KB, int R, bool BIG, bool L2>
__global__ void __launch_bounds__(kSubNT, 1) svt_subspace_kernel(const SvtParams prm) {
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
  constexpr int KB1 = BIG ? kSubspaceKB : (L2 ? kSubspaceKB1 : KB);
  constexpr int KB2 = BIG ? kSubspaceKBBig : kSubspaceKB;
  static_assert(L2 ? KB == KB2 : (BIG ? KB == kSubspaceKB : (KB == kSubspaceKB1 || KB == kSubspaceKB)),
                "block size of the level");
  constexpr bool NOSPLIT = BIG && L2;
  static_assert(KB % 16 == 0 && KB % 8 == 0, "KB must be a multiple of 16");
  static_assert(R == 32, "the thread mappings assume 32-row chunks");

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
  if (!L2 && F.fallback &&
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
  float2* Yc = C + R * CS;                           // R x KS
  float2* Yc2;                                       // R x KS (second k-half of the chunk GEMM)
  float2* wl;                                        // B x len  (BIG: len)
  float2* acc;                                       // B x len  (BIG: 2 x len)
  float2* tail;
  // NOSPLIT: the Rayleigh-Ritz matrix sits behind the eigen-solver's work
  // area (3 KB^2 floats at C), spilling from C into the Y region
  constexpr int YREG = NOSPLIT ? (KB * KS + 3 * KB * KB / 2 - R * CS > R * KS ? KB * KS + 3 * KB * KB / 2 - R * CS
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
  float2* Hm = BIG ? (NOSPLIT ? C + 3 * KB * KB / 2 : Yc) : X;  // KB x KS Rayleigh-Ritz matrix
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
  const bool chain = BIG && L2 && F.Z1 && F.Vd && F.ndefl;
  float2* Vdg = chain ? F.Vd + (long long)mat * DP * DP : nullptr;
  const int nd_in = defl3 ? F.ndefl[mat] : 0;
  // M <- (I - Vd Vd^H) M over the deflated columns, in blocks of kDeflateK
  // (block classical Gram-Schmidt, repeated: CGS2)
  auto project_defl = [&](float2* M) {
    for (int rep = 0; rep < 2; ++rep)
      for (int b0 = 0; b0 < nd_in; b0 += kDeflateK)
        project_out<KB, KS>(M, Vdg + b0, DP, min(kDeflateK, nd_in - b0), d, C);
  };
  const bool stg = Dg != nullptr && !BIG;  // duals staged by cp.async (non-BIG)

  // ---------------------------------------------------------- spectra
  const float2* spg = F.spec + (long long)mat * F.s_mat;
  if (BIG) {
    for (int t = tid; t < len; t += NT) wl[t] = weighted ? F.wc[t] : make_float2(1.f, 0.f);
    for (int t = tid; t < 2 * len; t += NT) acc[t] = make_float2(0.f, 0.f);
    // block/shift of the lifted index: rows of Ahat (wide) or its columns (tall)
    for (int t = tid; t < (F.wide ? e : d); t += NT) {
      const int b = t / F.q;
      lofs[t] = (b << 16) | (t - b * F.q);
    }
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
    const float2* sp = spg;
    for (int t = tid; t < J * len; t += NT) {
      const int j = t / len, n = t - j * len;
      const float2 s = sp[n * F.s_n + j * F.s_j];
      if (weighted) {
        wl[j * len + n] = cmul(F.wc[n], s);
        if (F.vc) {
          const int fl = dagger_src(n, len);
          const float2 sf = sp[fl * F.s_n + j * F.s_j];
          wl[(J + j) * len + n] = cmul(F.wc[n], cconj(sf));
        }
      } else {
        wl[j * len + n] = s;
      }
    }
    for (int t = tid; t < B * len; t += NT) acc[t] = make_float2(0.f, 0.f);
    for (int t = tid; t < (F.wide ? e : d); t += NT) {
      const int b = t / F.q;
      lofs[t] = b * len + (t - b * F.q);
    }
    if (tid < 4) S.flags[tid] = 0;
    if (tid == 0) *cnt = 0;
  }
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
    householder_qr<KB, KS, DP>(X, V, d, tau);
    // a remainder narrower than the block: the QR's extra columns leave the
    // remainder, projecting them out makes them ~0 (Ritz values ~0, f = 0)
    if (defl3 && d - nd_in < KB) project_defl(V);
  }

  // mappings: Yc rows yi / X rows k0 + 32m, columns c + 16n
  const int yi = tid >> 4, c16 = tid & 15;
  const int iters = warm ? prm.q_warm : prm.q_cold;

  // ---------------------------------------------------------- subspace iteration
  // Duals are staged chunk by chunk with cp.async into a buffer that is free
  // during the pass (X here, V in the epilogue pass): the copy of chunk c+1
  // overlaps the GEMMs of chunk c.
  for (int it = 0; it < iters; ++it) {
    float2 xa[MR][NC];
#pragma unroll
    for (int m = 0; m < MR; ++m)
#pragma unroll
      for (int n = 0; n < NC; ++n) xa[m][n] = make_float2(0.f, 0.f);
    __syncthreads();  // X (reflectors of the last QR) is free from here
    if (stg) stage_d_async(X, Dg, 0, min(R, e), d);
    if (prm.phase_clk) clk_u = clock64();
    for (int i0 = 0; i0 < e; i0 += R) {
      const int rows = min(R, e - i0);
      if (stg) stage_d_wait();
      SUB_ACC(clk_wait);
      if (BIG) build_chunk_big<DP, CS, R>(C, F, spg, wl, weighted, lofs, Dg, i0, rows, prm.inv_beta);
      else build_chunk<DP, CS, R>(C, wl, lofs, F, Dg ? X : nullptr, i0, rows, prm.inv_beta);
      __syncthreads();
      SUB_ACC(clk_build);
      if (stg && i0 + R < e) stage_d_async(X, Dg, i0 + R, min(R, e - i0 - R), d);
      chunk_block<CS, KS, NC, R, NOSPLIT>(C, V, Yc, Yc2, d, nullptr);  // Yc = C V
      SUB_ACC(clk_g1);
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
      if (!stg) __syncthreads();  // with staged duals the next stage_d_wait() is the barrier
      SUB_ACC(clk_g2);
    }
    if (stg) __syncthreads();
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int k = yi + 32 * m;
      if (k < DP)
#pragma unroll
        for (int n = 0; n < NC; ++n) X[k * KS + c16 + 16 * n] = xa[m][n];
    }
    __syncthreads();
    clk_pass += clock64() - clk_t;
    clk_t = clock64();
    if (defl3) project_defl(X);
    if (warm && prm.inner_norm && it + 1 < iters) {
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
      householder_qr<KB, KS, DP>(X, V, d, tau);
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
    float2 h[HM][NC];
#pragma unroll
    for (int m = 0; m < HM; ++m)
#pragma unroll
      for (int n = 0; n < NC; ++n) h[m][n] = make_float2(0.f, 0.f);
    __syncthreads();  // X is free from here
    if (stg) stage_d_async(X, Dg, 0, min(R, e), d);
    for (int i0 = 0; i0 < e; i0 += R) {
      const int rows = min(R, e - i0);
      if (stg) stage_d_wait();
      if (BIG) build_chunk_big<DP, CS, R>(C, F, spg, wl, weighted, lofs, Dg, i0, rows, prm.inv_beta);
      else build_chunk<DP, CS, R>(C, wl, lofs, F, Dg ? X : nullptr, i0, rows, prm.inv_beta);
      __syncthreads();
      if (stg && i0 + R < e) stage_d_async(X, Dg, i0 + R, min(R, e - i0 - R), d);
      chunk_block<CS, KS, NC, R, NOSPLIT>(C, V, Yc, Yc2, d, nullptr);
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
      if (!stg) __syncthreads();
    }
    if (stg) __syncthreads();
    // H (full Hermitian, stride KB+1 = KS) into Hm, diagonal to S.dg
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
  __syncthreads();
  if (!prm.rr_jacobi) {
    SUB_STAMP(4);
    hermitian_eig_tridiag<KB, KS>(Hm, reinterpret_cast<float*>(S.rec), reinterpret_cast<float*>(C), C, S.dg,
                                  0.25f * prm.thresh * prm.thresh,
                                  prm.phase_clk ? prm.phase_clk + (long long)blockIdx.x * kPhaseSlots + 16 : nullptr);
    SUB_STAMP(5);
    if (prm.sweeps_out && tid == 0) prm.sweeps_out[blockIdx.x] = 0;
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
  {
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
  // the last level accepts Ritz pairs up to KB - kSubspaceMarginLast: pairs
  // that close to the block edge converge slowest but sit near the threshold,
  // where the shrink factor 1 - tau / sigma is ~0.  It keeps a matrix until
  // its rank falls well inside level 1's range (hysteresis).
  constexpr int kMarginHere = (BIG && L2) ? kSubspaceMarginLast : kSubspaceMargin;
  // level 2 (large d) with too many values above the threshold and a Z1
  // buffer: keep the leading kDeflateK Ritz pairs (Z1 = Ahat V1 f1 V1^H to
  // HBM) and hand the rest to the deflated level 3
  // (level 3 again while the remainder is wider than its block; a remainder
  // the block spans is solved exactly, so the chain always finishes)
  const bool to_defl = chain && r > KB - kMarginHere && d - nd_in > KB;
  if (F.fallback && tid == 0) {
    if (defl3)
      F.fallback[mat] = to_defl ? kLevelDeflate : kLevelDeflDone;
    else if (L2)
      F.fallback[mat] = to_defl ? kLevelDeflate
                        : r > KB - kMarginHere ? kLevelOverflow
                        : r <= KB1 - 2 * kSubspaceMargin ? 0 : kLevelStay2;
    else
      F.fallback[mat] = (r > KB - kSubspaceMargin) ? kLevelHanded : 0;
  }
  if (to_defl) {  // append the leading kDeflateK Ritz vectors to the deflated basis
    for (int t = tid; t < DP * kDeflateK; t += NT) {
      const int k = t / kDeflateK, j = t - k * kDeflateK;
      Vdg[(long long)k * DP + nd_in + j] = Vf[k * KS + j];
    }
    if (tid == 0) F.ndefl[mat] = nd_in + kDeflateK;
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
  if (!(BIG && L2) && r > KB - kMarginHere) return;

  // ---------------------------------------------------------- Z = (Ahat V) f V^H, duals, adjoint
  SUB_STAMP(6);
  float2* Ds = V;  // the old basis is dead: stage the duals there (non-BIG)
  __syncthreads();
  if (stg) stage_d_async(Ds, Dg, 0, min(R, e), d);
  for (int i0 = 0; i0 < e; i0 += R) {
    const int rows = min(R, e - i0);
    if (stg) stage_d_wait();
    if (BIG) build_chunk_big<DP, CS, R>(C, F, spg, wl, weighted, lofs, Dg, i0, rows, prm.inv_beta);
    else build_chunk<DP, CS, R>(C, wl, lofs, F, Dg ? Ds : nullptr, i0, rows, prm.inv_beta);
    __syncthreads();
    {
      // only the first r (sorted) Ritz columns have f > 0 (Z1 mode: the
      // leading kDeflateK)
      static_assert(NC <= 4, "NC > 4 needs more cases");
      const int nb = ((to_defl ? kDeflateK : r) + 15) >> 4;
      if (nb <= 1) chunk_block<CS, KS, 1, R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
      else if (nb == 2 || NC == 2) chunk_block<CS, KS, (NC >= 2 ? 2 : 1), R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
      else if (nb == 3 || NC == 3) chunk_block<CS, KS, (NC >= 3 ? 3 : 1), R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
      else chunk_block<CS, KS, NC, R, NOSPLIT>(C, Vf, Yc, Yc2, d, S.f);
    }
    {
      // Z[yi][k] = sum_{j < r} Yc[yi][j] conj(Vf[k][j]), k = c16 + 16 m
      constexpr int MZ = (DP + 15) / 16;
      float2 z[MZ];
#pragma unroll
      for (int m = 0; m < MZ; ++m) z[m] = make_float2(0.f, 0.f);
      const int rz = to_defl ? kDeflateK : r;
      for (int j = 0; j < rz; ++j) {
        const float2 yv = Yc[yi * KS + j];
#pragma unroll
        for (int m = 0; m < MZ; ++m) {
          const int k = c16 + 16 * m;
          if (k < DP) cfmac(z[m], Vf[k * KS + j], yv);  // yv * conj(V[k][j])
        }
      }
#pragma unroll
      for (int m = 0; m < MZ; ++m) {
        const int k = c16 + 16 * m;
        if (yi < rows && k < d) {
          if (to_defl) {  // Z1 only (accumulated along the chain): level 3 finishes this matrix
            float2* z1p = F.Z1 + (long long)mat * e * d + (long long)(i0 + yi) * d + k;
            *z1p = defl3 ? cadd(__ldcg(z1p), z[m]) : z[m];
            continue;
          }
          if (defl3) {
            const float2 z1 = __ldcg(F.Z1 + (long long)mat * e * d + (long long)(i0 + yi) * d + k);
            z[m].x += z1.x;
            z[m].y += z1.y;
          }
          float2 tv = z[m];
          if (admm) {
            const float2 L = BIG ? (F.wide ? lift_global(F, spg, wl, weighted, lofs[i0 + yi], k)
                                           : cconj(lift_global(F, spg, wl, weighted, lofs[k], i0 + yi)))
                                 : lift_tab(wl, lofs, F.wide, i0 + yi, k);
            const long long gi = (long long)(i0 + yi) * d + k;
            float2 dn = BIG ? __ldcg(Dg + gi) : Ds[yi * d + k];
            dn.x = fmaf(prm.tau_dual, L.x - z[m].x, dn.x);
            dn.y = fmaf(prm.tau_dual, L.y - z[m].y, dn.y);
            Dg[gi] = dn;
            tv.x = fmaf(-dn.x, prm.inv_beta, z[m].x);
            tv.y = fmaf(-dn.y, prm.inv_beta, z[m].y);
          }
          C[yi * CS + k] = tv;
        }
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

size_t svt_subspace_smem_bytes(int DP, int KB, int R, int maxB, int maxLen, int maxE, bool big) {
  const int KS = KB + 1, CS = DP + 1;
  const size_t spectra = big ? 3ull * maxLen : 2ull * maxB * maxLen;
  const bool nosplit = big && KB > kSubspaceKB;  // BIG level 2
  const size_t yreg = nosplit ? (size_t)std::max(R * KS, KB * KS + 3 * KB * KB / 2 - R * CS) : 2ull * R * KS;
  return sizeof(float2) * ((big ? 1ull : 2ull) * DP * KS + (size_t)R * CS + yreg + spectra) +
         sizeof(SlotRec) * KB + sizeof(double2) * KB + sizeof(double) * KB + 2 * sizeof(float) * KB +
         16 * sizeof(int) + sizeof(int) * KB + sizeof(int) * std::max(DP, maxE) + 64;
}

namespace {
template <int DP, int KB, bool BIG, bool L2>
void launch_sub(const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    SHLR_CUDA(cudaFuncSetAttribute(svt_subspace_kernel<DP, KB, 32, BIG, L2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = true;
  }
  svt_subspace_kernel<DP, KB, 32, BIG, L2><<<total, kSubNT, smem, stream>>>(prm);
  SHLR_LAUNCH_CHECK();
}

struct SubGeom {
  int dmin = 1 << 30, dmax = 0, maxB = 0, maxLen = 0, maxE = 0;
  bool all_wide = true, stores = true;
};
SubGeom sub_geom(const SvtParams& prm) {
  SubGeom g;
  for (int f = 0; f < prm.nfam; ++f) {
    g.dmin = std::min(g.dmin, prm.fam[f].d);
    g.dmax = std::max(g.dmax, prm.fam[f].d);
    g.maxB = std::max(g.maxB, prm.fam[f].B);
    g.maxLen = std::max(g.maxLen, prm.fam[f].len);
    g.maxE = std::max(g.maxE, prm.fam[f].e);
    g.all_wide = g.all_wide && prm.fam[f].wide;
    g.stores = g.stores && prm.fam[f].Vs && prm.fam[f].fallback;
  }
  return g;
}

// Launches level L2 of the subspace solver (d <= 128 level 1 with KB1
// columns); false if the geometry is out of its range (nothing launched).
template <bool L2, int KB1 = kSubspaceKB1>
bool launch_level(const SvtParams& prm, int total, cudaStream_t stream) {
  const SubGeom g = sub_geom(prm);
  if (!g.stores) return false;
  // worthwhile only when the level-1 block is well below d
  if (g.dmin < kSubspaceKB + 24) return false;
  if (g.dmax > 128) {
    // large-d variant (spectra and adjoint not resident)
    // (tall lifts accumulate the adjoint in the zeroed output, weighted and
    // virtual-coil blocks included; plain lifts have no virtual coils)
    if (g.maxLen > 0xffff) return false;
    for (int f = 0; f < prm.nfam; ++f)
      if (prm.fam[f].vc && prm.mode != SVT_ADMM_WEIGHTED) return false;
    const int dpb = svt_big_padded_dim(g.dmax);
    if (!dpb) return false;
    constexpr int KB = L2 ? kSubspaceKBBig : kSubspaceKB;
    const size_t smem = svt_subspace_smem_bytes(dpb, KB, 32, g.maxB, g.maxLen, g.maxE, true);
    if (smem > 227 * 1024) return false;
    switch (dpb) {
      case 160: launch_sub<160, KB, true, L2>(prm, total, smem, stream); return true;
      case 192: launch_sub<192, KB, true, L2>(prm, total, smem, stream); return true;
      case 248: launch_sub<248, KB, true, L2>(prm, total, smem, stream); return true;
    }
    return false;
  }
  constexpr int KB = L2 ? kSubspaceKB : KB1;
  const int dp = svt_padded_dim(g.dmax);
  const size_t smem = svt_subspace_smem_bytes(dp, KB, 32, g.maxB, g.maxLen, g.maxE, false);
  if (smem > 227 * 1024) return false;
  switch (dp) {
    case 72: launch_sub<72, KB, false, L2>(prm, total, smem, stream); return true;
    case 80: launch_sub<80, KB, false, L2>(prm, total, smem, stream); return true;
    case 88: launch_sub<88, KB, false, L2>(prm, total, smem, stream); return true;
    case 96: launch_sub<96, KB, false, L2>(prm, total, smem, stream); return true;
    case 104: launch_sub<104, KB, false, L2>(prm, total, smem, stream); return true;
    case 112: launch_sub<112, KB, false, L2>(prm, total, smem, stream); return true;
    case 120: launch_sub<120, KB, false, L2>(prm, total, smem, stream); return true;
    case 128: launch_sub<128, KB, false, L2>(prm, total, smem, stream); return true;
    default: return false;
  }
}
}  // namespace

bool launch_hankel_svt_subspace(const SvtParams& prm, int total, cudaStream_t stream, int kb1) {
  if (total <= 0) return true;
  return kb1 == kSubspaceKB1 ? launch_level<false, kSubspaceKB1>(prm, total, stream)
                             : launch_level<false, kSubspaceKB>(prm, total, stream);
}

int launch_hankel_svt_levels(const SvtParams& sp, int total, cudaStream_t stream, int kb1) {
  int dmax = 0;
  for (int f = 0; f < sp.nfam; ++f) dmax = std::max(dmax, sp.fam[f].d);
  const bool big = dmax > 128;
  if (big) kb1 = kSubspaceKB;
  if (!launch_hankel_svt_subspace(sp, total, stream, kb1)) return 0;
  int n = 1;
  if (big || kb1 == kSubspaceKB1) {
    SvtParams l2 = sp;
    l2.only_flagged = sp.fam[0].fallback;
    l2.q_cold = std::getenv("SHLR_L2_Q") ? std::atoi(std::getenv("SHLR_L2_Q")) : 8;
    launch_hankel_svt_level2(l2, total, stream);
    ++n;
  }
  if (big) {
    if (sp.fam[0].Z1 && sp.fam[0].Vd && sp.fam[0].ndefl) {
      // level 3: the deflated remainder of level 2's overflow, one launch per
      // chain step (matrices that finished skip the later launches)
      SvtParams l3 = sp;
      l3.only_flagged = sp.fam[0].fallback;
      l3.only_flag_value = kLevelDeflate;
      l3.deflate = 1;
      l3.warm = nullptr;
      l3.q_cold = std::getenv("SHLR_L3_Q") ? std::atoi(std::getenv("SHLR_L3_Q")) : 8;
      for (int k = 0; k < svt_deflation_steps(dmax); ++k) {
        launch_hankel_svt_level2(l3, total, stream);
        ++n;
      }
    }
    return n;
  }
  // the full solver redoes what the last subspace level handed on (cold)
  SvtParams fs = sp;
  fs.only_flagged = sp.fam[0].fallback;
  fs.only_flag_value = kb1 == kSubspaceKB1 ? kLevelOverflow : kLevelHanded;
  fs.warm = nullptr;
  launch_hankel_svt(fs, total, stream);
  return n + 1;
}

void launch_hankel_svt_level2(const SvtParams& prm, int total, cudaStream_t stream) {
  if (total <= 0) return;
  if (!prm.only_flagged) throw InvalidArg("hankel_svt level 2: only_flagged required");
  if (!launch_level<true>(prm, total, stream))
    throw Unsupported("hankel_svt: subspace level-2 geometry out of range");
}

size_t svt_smem_bytes(int DP, int R, int maxB, int maxLen, bool wl_smem) {
  const int S_ = DP / 2;
  return sizeof(float2) * ((size_t)DP * (DP + 1) + (wl_smem ? 2ull : 1ull) * maxB * maxLen + 2ull * R * DP) +
         (sizeof(SlotRec) + sizeof(double2)) * 2 * S_ + sizeof(double) * DP + sizeof(float) * DP + 8 * sizeof(int) + 64;
}

int svt_padded_dim(int d) { return std::max(8, ((d + 7) / 8) * 8); }

namespace {

template <int DP, int R>
void launch_one(const SvtParams& prm, int total, size_t smem, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    SHLR_CUDA(cudaFuncSetAttribute(hankel_svt_kernel<DP, R>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = true;
  }
  hankel_svt_kernel<DP, R><<<total, 4 * DP, smem, stream>>>(prm);
  SHLR_LAUNCH_CHECK();
}

template <int DP>
void dispatch_r(const SvtParams& prm, int total, int maxB, int maxLen, cudaStream_t stream) {
  const size_t lim = 227 * 1024;
  const size_t s32 = svt_smem_bytes(DP, 32, maxB, maxLen);
  // the W-panel staging needs 2 R DP >= DP * DP / 4 complex: true for R >= 16, DP <= 128
  if (s32 <= lim) return launch_one<DP, 32>(prm, total, s32, stream);
  const size_t s16 = svt_smem_bytes(DP, 16, maxB, maxLen);
  if (s16 <= lim) return launch_one<DP, 16>(prm, total, s16, stream);
  // plain lifts of contiguous coil vectors can read their source from global
  // memory (L2-resident) instead of an smem copy
  bool direct = prm.mode == SVT_PLAIN;
  for (int f = 0; f < prm.nfam; ++f)
    direct = direct && prm.fam[f].s_n == 1 && prm.fam[f].s_j == prm.fam[f].len && !prm.fam[f].vc;
  if (direct) {
    SvtParams pg = prm;
    pg.wl_global = 1;
    const size_t g32 = svt_smem_bytes(DP, 32, maxB, maxLen, false);
    if (g32 <= lim) return launch_one<DP, 32>(pg, total, g32, stream);
    const size_t g16 = svt_smem_bytes(DP, 16, maxB, maxLen, false);
    if (g16 <= lim) return launch_one<DP, 16>(pg, total, g16, stream);
  }
  throw Unsupported("hankel_svt: shared-memory footprint exceeds 227 KB for this geometry");
}

}  // namespace

void launch_hankel_svt(const SvtParams& prm, int total, cudaStream_t stream) {
  if (total <= 0) return;
  int dmax = 0, maxB = 0, maxLen = 0;
  for (int f = 0; f < prm.nfam; ++f) {
    dmax = std::max(dmax, prm.fam[f].d);
    maxB = std::max(maxB, prm.fam[f].B);
    maxLen = std::max(maxLen, prm.fam[f].len);
    if (prm.fam[f].J * prm.fam[f].len < 1) throw InvalidArg("hankel_svt: empty family");
  }
  const int dp = svt_padded_dim(dmax);
  for (int f = 0; f < prm.nfam; ++f)
    if (!prm.fam[f].V) throw InvalidArg("hankel_svt: missing eigenvector store");
  switch (dp) {
    case 8: return dispatch_r<8>(prm, total, maxB, maxLen, stream);
    case 16: return dispatch_r<16>(prm, total, maxB, maxLen, stream);
    case 24: return dispatch_r<24>(prm, total, maxB, maxLen, stream);
    case 32: return dispatch_r<32>(prm, total, maxB, maxLen, stream);
    case 40: return dispatch_r<40>(prm, total, maxB, maxLen, stream);
    case 48: return dispatch_r<48>(prm, total, maxB, maxLen, stream);
    case 56: return dispatch_r<56>(prm, total, maxB, maxLen, stream);
    case 64: return dispatch_r<64>(prm, total, maxB, maxLen, stream);
    case 72: return dispatch_r<72>(prm, total, maxB, maxLen, stream);
    case 80: return dispatch_r<80>(prm, total, maxB, maxLen, stream);
    case 88: return dispatch_r<88>(prm, total, maxB, maxLen, stream);
    case 96: return dispatch_r<96>(prm, total, maxB, maxLen, stream);
    case 104: return dispatch_r<104>(prm, total, maxB, maxLen, stream);
    case 112: return dispatch_r<112>(prm, total, maxB, maxLen, stream);
    case 120: return dispatch_r<120>(prm, total, maxB, maxLen, stream);
    case 128: return dispatch_r<128>(prm, total, maxB, maxLen, stream);
    default:
      throw Unsupported("hankel_svt: min(m, n) = " + std::to_string(dmax) +
                        " exceeds the single-CTA eigen-solver limit of 128 in this build");
  }
}

}  // namespace shlr_b200
