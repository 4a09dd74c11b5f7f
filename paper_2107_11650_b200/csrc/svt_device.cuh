// Device building blocks shared by the Hankel-SVT kernels (full two-sided
// Jacobi solver in hankel_svt.cu, subspace solver in svt_subspace.cuh):
// lifted-element addressing, chunk builders, chunk GEMMs, the parallel
// Jacobi rotations.  Included by every translation unit that instantiates
// a Hankel-SVT kernel (internal linkage).
#pragma once
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

// Stage the J coil spectra of one lifted matrix in shared memory
// (lift_weighted, operators.cpp:25-58): weighted modes hold wc[n] s_j[n] in
// block j and, with virtual coils, wc[n] conj(s_j[dagger(n)]) in block J + j
// (hankel.cpp:99-113); plain modes hold s_j[n].  Threads tid, tid + nt, ...
__device__ __forceinline__ void stage_spectra(float2* wl, const SvtFamily& F, const float2* sp, bool weighted,
                                              int tid, int nt) {
  const int len = F.len, J = F.J;
  for (int t = tid; t < J * len; t += nt) {
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
}

// Per-index lift offsets over the lifted matrix's block index (columns of A
// when tall, rows of A^H when wide): b * len + t for the smem-staged spectra
// (lift_tab), (b << 16) | t for the L2-resident spectra (lift_global).
__device__ __forceinline__ void build_lofs(int* lofs, const SvtFamily& F, bool packed, int tid, int nt) {
  for (int t = tid; t < (F.wide ? F.e : F.d); t += nt) {
    const int b = t / F.q;
    lofs[t] = packed ? ((b << 16) | (t - b * F.q)) : (b * F.len + (t - b * F.q));
  }
}

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

// L2 prefetch of `count` contiguous complex64 (the dual rows of a coming
// chunk): the large-d layout reads its duals straight from HBM, one
// dependent load per element; with the lines already in L2 the chunk build
// and the dual update pay L2 latency instead of HBM latency.
__device__ __forceinline__ void prefetch_l2(const float2* p, int count) {
  for (int t = threadIdx.x * 16; t < count; t += blockDim.x * 16)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + t));
}

template <int DP, int CS, int R>
__device__ __forceinline__ void build_chunk_big(float2* dst, const SvtFamily& F, const float2* __restrict__ sp,
                                                const float2* wcs, bool weighted, const int* lofs,
                                                const float2* __restrict__ Dg, int i0, int rows, float inv_beta) {
  const int d = F.d;
  // batches of four elements per thread: the four dual loads (HBM / L2) and
  // the four lift sources (L2) are issued before the first is consumed
  constexpr int NB4 = 4;
  for (int t0 = threadIdx.x; t0 < R * DP; t0 += NB4 * blockDim.x) {
    float2 dd[NB4], v[NB4];
    int ru[NB4];
#pragma unroll
    for (int q = 0; q < NB4; ++q) {
      const int t = t0 + q * blockDim.x;
      const int r = t / DP, u = t - r * DP;
      const bool ok = t < R * DP && r < rows && u < d;
      ru[q] = t < R * DP ? r * CS + u : -1;
      dd[q] = make_float2(0.f, 0.f);
      v[q] = make_float2(0.f, 0.f);
      if (ok) {
        if (Dg) dd[q] = __ldcg(Dg + (long long)(i0 + r) * d + u);  // duals straight from HBM/L2 (coalesced rows)
        v[q] = F.wide ? lift_global(F, sp, wcs, weighted, lofs[i0 + r], u)
                      : cconj(lift_global(F, sp, wcs, weighted, lofs[u], i0 + r));  // tall: Ahat = A
      }
    }
#pragma unroll
    for (int q = 0; q < NB4; ++q)
      if (ru[q] >= 0) dst[ru[q]] = make_float2(fmaf(dd[q].x, inv_beta, v[q].x), fmaf(dd[q].y, inv_beta, v[q].y));
  }
}

// Large-d layout, staged lift sources.  A chunk of R rows of Ahat only touches
// a few hundred distinct source elements (a wide chunk: the whole vector of
// the 3-4 blocks its rows belong to; a tall chunk: rows + q - 1 positions of
// every block), each of them ~R times (Hankel structure).  With two CTAs per
// SM there is almost no L1 left, so lift_global's per-element loads all go to
// L2, one 32-byte sector per lane (coil-fastest spectra).  Here the sources
// are loaded once per chunk into a small shared buffer, weighting and
// virtual-coil dagger applied (lift_weighted, operators.cpp:36-56), and the
// chunk is built from shared memory.
constexpr int kBuildThreads = 512;  // threads of the subspace kernel (kSubNT)
struct ChunkSources {
  int b_lo, span, ok;
};
__device__ __forceinline__ ChunkSources stage_chunk_sources(float2* st, int cap, const SvtFamily& F,
                                                            const float2* __restrict__ sp, const float2* wcs,
                                                            bool weighted, int i0, int rows) {
  ChunkSources cs;
  int nblk, n0;
  if (F.wide) {
    cs.b_lo = i0 / F.q;
    nblk = (i0 + rows - 1) / F.q - cs.b_lo + 1;
    cs.span = F.len;
    n0 = 0;
  } else {
    cs.b_lo = 0;
    nblk = F.B;
    cs.span = min(rows + F.q - 1, F.len - i0);
    n0 = i0;
  }
  cs.ok = nblk * cs.span <= cap;
  if (!cs.ok) return cs;
  for (int t = threadIdx.x; t < nblk * cs.span; t += blockDim.x) {
    const int bb = t / cs.span, n = n0 + (t - bb * cs.span);
    const int b = cs.b_lo + bb;
    float2 v;
    if (b < F.J) {
      v = __ldg(sp + (long long)n * F.s_n + (long long)b * F.s_j);
      if (weighted) v = cmul(wcs[n], v);
    } else {
      const int fl = dagger_src(n, F.len);
      v = cmul(wcs[n], cconj(__ldg(sp + (long long)fl * F.s_n + (long long)(b - F.J) * F.s_j)));
    }
    st[t] = v;
  }
  return cs;
}

// Chunk build from the staged sources (after a barrier): same values as build_chunk_big.
template <int DP, int CS, int R>
__device__ __forceinline__ void build_chunk_staged(float2* dst, const SvtFamily& F, const float2* st,
                                                   const ChunkSources cs, const int* lofs,
                                                   const float2* __restrict__ Dg, int i0, int rows, float inv_beta) {
  const int d = F.d;
  auto lift = [&](int r, int u) -> float2 {
    if (F.wide) {
      const int bt = lofs[i0 + r];
      return cconj(st[((bt >> 16) - cs.b_lo) * cs.span + (bt & 0xffff) + u]);
    }
    const int bt = lofs[u];
    return st[(bt >> 16) * cs.span + (bt & 0xffff) + r];
  };
  if (Dg && (d & 1) == 0 && (DP & 1) == 0 && (reinterpret_cast<uintptr_t>(Dg) & 15) == 0) {
    // the chunk's duals are rows * d contiguous complex64: 16-byte loads, two
    // elements each, all of a thread's loads (<= 4) in flight before the first use
    constexpr int HP = DP / 2;                                  // element pairs per chunk row
    constexpr int NP = (R * HP + kBuildThreads - 1) / kBuildThreads;  // pairs per thread
    static_assert(NP <= 8, "pairs per thread");
    const float4* d4 = reinterpret_cast<const float4*>(Dg + (long long)i0 * d);
    float4 dd[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int t = threadIdx.x + q * kBuildThreads;
      const int r = t / HP, u = 2 * (t - r * HP);
      dd[q] = (t < R * HP && r < rows && u < d) ? __ldcg(d4 + ((long long)r * d + u) / 2) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int t = threadIdx.x + q * kBuildThreads;
      if (t < R * HP) {
        const int r = t / HP, u = 2 * (t - r * HP);
        float2 v0 = make_float2(0.f, 0.f), v1 = v0;
        if (r < rows && u < d) {
          v0 = lift(r, u);
          v1 = lift(r, u + 1);
          v0.x = fmaf(dd[q].x, inv_beta, v0.x);
          v0.y = fmaf(dd[q].y, inv_beta, v0.y);
          v1.x = fmaf(dd[q].z, inv_beta, v1.x);
          v1.y = fmaf(dd[q].w, inv_beta, v1.y);
        }
        dst[r * CS + u] = v0;
        dst[r * CS + u + 1] = v1;
      }
    }
    return;
  }
  constexpr int NB4 = 4;
  for (int t0 = threadIdx.x; t0 < R * DP; t0 += NB4 * blockDim.x) {
    float2 dd[NB4];
#pragma unroll
    for (int q = 0; q < NB4; ++q) {
      const int t = t0 + q * blockDim.x;
      const int r = t / DP, u = t - r * DP;
      dd[q] = (Dg && t < R * DP && r < rows && u < d) ? __ldcg(Dg + (long long)(i0 + r) * d + u)
                                                      : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < NB4; ++q) {
      const int t = t0 + q * blockDim.x;
      if (t < R * DP) {
        const int r = t / DP, u = t - r * DP;
        float2 v = make_float2(0.f, 0.f);
        if (r < rows && u < d) {
          v = lift(r, u);
          v.x = fmaf(dd[q].x, inv_beta, v.x);
          v.y = fmaf(dd[q].y, inv_beta, v.y);
        }
        dst[r * CS + u] = v;
      }
    }
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

}  // namespace shlr_b200
