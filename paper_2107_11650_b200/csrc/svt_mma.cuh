// 3xTF32 chunk contractions of the subspace SVT on the tensor cores
// (warp-level mma.sync m16n8k8, FP32 accumulate).
//
// north_star allows tensor cores for the streaming contractions only if a
// 3xTF32 split meets the 1e-4 tolerance.  Each FP32 operand is split into
// hi = its leading 11 significand bits (what the TF32 datapath reads) and
// lo = x - hi (exact in FP32); a real product is hi*hi + hi*lo + lo*hi, the
// dropped lo*lo term is ~2^-22 relative.  A complex product is four real
// ones, so one 16 x 8 x 8 complex tile step costs 12 mma.sync.  Operands stay
// in the kernel's existing shared-memory layouts: fragments are gathered with
// 8-byte loads and split in registers, so the tensor path needs no extra
// shared memory (a tcgen05 path would need hi and lo operand copies in the
// canonical UMMA layouts: 2 x (R x 2d + 2d x 2KB) x 4 B > 227 KB at d = 120).
// Measured issue rate on the B200 (scripts/probes/mma_rate.cu): 0.47
// mma.sync/clk/SM = 279 TFLOP/s dense TF32, 93 TFLOP/s after the 3x split,
// against 72 TFLOP/s for FFMA.
#pragma once

#include "common.cuh"
#include "svt_device.cuh"

namespace shlr_b200 {

__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A fragment of a complex 16 x 8 tile: real / imaginary parts, hi / lo splits.
struct CFragA {
  uint32_t rh[4], rl[4], ih[4], il[4];
  __device__ __forceinline__ void set(int i, float2 v) {
    tf32_split(v.x, rh[i], rl[i]);
    tf32_split(v.y, ih[i], il[i]);
  }
};
// B fragment of a complex 8 x 8 tile.
struct CFragB {
  uint32_t rh[2], rl[2], ih[2], il[2];
  __device__ __forceinline__ void set(int i, float2 v) {
    tf32_split(v.x, rh[i], rl[i]);
    tf32_split(v.y, ih[i], il[i]);
  }
};

// 3xTF32 real product accumulate: c += a b (small terms first)
__device__ __forceinline__ void mma3(float (&c)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     uint32_t bh0, uint32_t bh1, uint32_t bl0, uint32_t bl1) {
  mma_tf32(c, al, bh0, bh1);
  mma_tf32(c, ah, bl0, bl1);
  mma_tf32(c, ah, bh0, bh1);
}

// (yr + i yi) += op(a) b on one 16 x 8 x 8 complex tile step; op = conj when
// CONJ_A, and b is conjugated when CONJ_B.
template <bool CONJ_A, bool CONJ_B>
__device__ __forceinline__ void cmma(float (&yr)[4], float (&yi)[4], const CFragA& a, const CFragB& b) {
  constexpr uint32_t SGN = 0x80000000u;
  // re: ar br - sa sb ai bi;  im: sb ar bi + sa ai br  (sa / sb = -1 for a conjugated operand)
  constexpr uint32_t s_re = (CONJ_A != CONJ_B) ? 0u : SGN;  // sign flip of the ai bi term
  constexpr uint32_t s_bi = CONJ_B ? SGN : 0u;              // ar bi term
  constexpr uint32_t s_ai = CONJ_A ? SGN : 0u;              // ai br term
  mma3(yr, a.rh, a.rl, b.rh[0], b.rh[1], b.rl[0], b.rl[1]);
  mma3(yr, a.ih, a.il, b.ih[0] ^ s_re, b.ih[1] ^ s_re, b.il[0] ^ s_re, b.il[1] ^ s_re);
  mma3(yi, a.rh, a.rl, b.ih[0] ^ s_bi, b.ih[1] ^ s_bi, b.il[0] ^ s_bi, b.il[1] ^ s_bi);
  mma3(yi, a.ih, a.il, b.rh[0] ^ s_ai, b.rh[1] ^ s_ai, b.rl[0] ^ s_ai, b.rl[1] ^ s_ai);
}

// One complex 16 x 8 output tile in eight accumulator chains: a dependent
// mma.sync waits ~60+ cycles for its predecessor, so the twelve products of a
// tile step go to separate chains (depth <= 2 per step) -- leading and
// correction products of ar x b and of ai x b apart -- and are summed once.
struct CAcc8 {
  float r1[4], r2[4], i1[4], i2[4], sr1[4], sr2[4], si1[4], si2[4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i) r1[i] = r2[i] = i1[i] = i2[i] = sr1[i] = sr2[i] = si1[i] = si2[i] = 0.f;
  }
  template <bool CONJ_A, bool CONJ_B>
  __device__ __forceinline__ void mma(const CFragA& a, const CFragB& b) {
    constexpr uint32_t SGN = 0x80000000u;
    constexpr uint32_t s_re = (CONJ_A != CONJ_B) ? 0u : SGN;  // sign of the ai bi term
    constexpr uint32_t s_bi = CONJ_B ? SGN : 0u;              // ar bi term
    constexpr uint32_t s_ai = CONJ_A ? SGN : 0u;              // ai br term
    mma_tf32(sr1, a.rl, b.rh[0], b.rh[1]);
    mma_tf32(si1, a.rl, b.ih[0] ^ s_bi, b.ih[1] ^ s_bi);
    mma_tf32(sr2, a.il, b.ih[0] ^ s_re, b.ih[1] ^ s_re);
    mma_tf32(si2, a.il, b.rh[0] ^ s_ai, b.rh[1] ^ s_ai);
    mma_tf32(r1, a.rh, b.rh[0], b.rh[1]);
    mma_tf32(i1, a.rh, b.ih[0] ^ s_bi, b.ih[1] ^ s_bi);
    mma_tf32(r2, a.ih, b.ih[0] ^ s_re, b.ih[1] ^ s_re);
    mma_tf32(i2, a.ih, b.rh[0] ^ s_ai, b.rh[1] ^ s_ai);
    mma_tf32(sr1, a.rh, b.rl[0], b.rl[1]);
    mma_tf32(si1, a.rh, b.il[0] ^ s_bi, b.il[1] ^ s_bi);
    mma_tf32(sr2, a.ih, b.il[0] ^ s_re, b.il[1] ^ s_re);
    mma_tf32(si2, a.ih, b.rl[0] ^ s_ai, b.rl[1] ^ s_ai);
  }
  __device__ __forceinline__ float2 get(int i) const {
    return make_float2((r1[i] + r2[i]) + (sr1[i] + sr2[i]), (i1[i] + i2[i]) + (si1[i] + si2[i]));
  }
};

// Fragment gathers without shared-memory bank conflicts.  The kernel's
// buffers have odd row strides (CS = DP + 1, KS = KB + 1: 9 or 1 modulo 16 in
// 8-byte units), so the natural fragment (row g, column t) puts lanes of one
// 16-lane phase in the same bank.  An MMA is indifferent to which physical
// row / column / k index sits in which logical slot as long as A, B and the
// output agree, so each operand is gathered through a permutation that
// spreads one phase's 16 lanes over 16 distinct banks:
//   stride = 1 (mod 16): slot g -> 4 (g & 3) + (g >> 2), second row set +2,
//                        k slots t, t + 4;
//   stride = 9 (mod 16), rows as MMA rows: slot g -> {0,1,8,9,2,3,10,11}[g],
//                        second row set +4, k slots 2 t, 2 t + 1.
__device__ __forceinline__ int perm_s1(int g) { return ((g & 3) << 2) | (g >> 2); }
__device__ __forceinline__ int perm_s9(int g) { return (g & 1) | ((g & 2) << 2) | ((g & 4) >> 1); }

// Yc (32 x 8 ntiles) = C B: warp w < 2 ntiles owns one 16 x 8 tile (row tile
// w & 1, column tile w >> 1: eight columns of a 16-column group) over the whole k
// range, the leading and the correction products in separate accumulator
// chains.  C is the R x CS chunk (zero padded to a multiple of 8 columns), B
// the d x KS block.
template <int CS, int KS>
__device__ __forceinline__ void chunk_times_block_mma(const float2* C, const float2* Bm, float2* Yc, int d,
                                                      const float* scale, int ntiles) {
  static_assert(KS % 16 == 1 && (CS % 16 == 9 || CS % 16 == 1), "fragment permutations assume these strides");
  constexpr bool S9 = CS % 16 == 9;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= 2 * ntiles) return;
  const int g = lane >> 2, t = lane & 3;
  const int mt = w & 1, tl = w >> 1;
  const int ks = (d + 7) >> 3;
  CAcc8 acc;
  acc.zero();
  const int pg = S9 ? perm_s9(g) : perm_s1(g);
  const int ka = S9 ? 2 * t : t, kb = S9 ? 2 * t + 1 : t + 4;  // physical k of the two k slots
  const int row2 = S9 ? 4 : 2, sub = S9 ? 4 : 2;
  const float2* crow = C + (16 * mt + pg) * CS;
  const int col = 16 * (tl >> 1) + sub * (tl & 1) + pg;
#pragma unroll 2
  for (int s = 0; s < ks; ++s) {
    const int k0 = 8 * s;
    CFragA a;
    a.set(0, crow[k0 + ka]);
    a.set(1, crow[row2 * CS + k0 + ka]);
    a.set(2, crow[k0 + kb]);
    a.set(3, crow[row2 * CS + k0 + kb]);
    CFragB b;
    b.set(0, Bm[(k0 + ka) * KS + col]);
    b.set(1, Bm[(k0 + kb) * KS + col]);
    acc.mma<false, false>(a, b);
  }
  const int cb = 16 * (tl >> 1) + sub * (tl & 1);
  const int c0 = cb + (S9 ? perm_s9(2 * t) : perm_s1(2 * t)), c1 = cb + (S9 ? perm_s9(2 * t + 1) : perm_s1(2 * t + 1));
  const float f0 = scale ? scale[c0] : 1.f, f1 = scale ? scale[c1] : 1.f;
  float2* out = Yc + (16 * mt + pg) * KS;
  out[c0] = cscale(acc.get(0), f0);
  out[c1] = cscale(acc.get(1), f1);
  out[row2 * KS + c0] = cscale(acc.get(2), f0);
  out[row2 * KS + c1] = cscale(acc.get(3), f1);
}

// Chunk GEMM Yc = C B (columns 16 NB), optionally column-scaled: the tensor
// form of chunk_block (svt_device.cuh).  Ends with a barrier.
template <int CS, int KS, int NB, int R>
__device__ __forceinline__ void chunk_block_mma(const float2* C, const float2* Bm, float2* Yc, float2* Yc2, int d,
                                                const float* scale) {
  static_assert(R == 32, "two 16-row tiles");
  (void)Yc2;
  chunk_times_block_mma<CS, KS>(C, Bm, Yc, d, scale, 2 * NB);
  __syncthreads();
}

// Accumulators of a DP x KB block product (KB = 48 or 32), 16 warps: warp w
// takes the 16-row tile w >> 1 and NTW = KB / 16 8-column tiles (tile index
// NTW (w & 1) + j: the two tiles of a 16-column group hold its columns
// 4 a + b + 2 sub).  Rows at or beyond DP are computed from whatever follows
// in shared memory and never stored (an MMA output row depends on its own A
// row only).
template <int NTW>
struct XAccMma {
  float xr[NTW][4], xi[NTW][4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < NTW; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) xr[j][i] = xi[j][i] = 0.f;
  }
};
// first physical column of tile tl in the stride-1 scheme
__device__ __forceinline__ int tile_col_s1(int tl) { return 16 * (tl >> 1) + 2 * (tl & 1); }

// X (DP x KB) += C^H Yc over one chunk of R = 32 rows.
template <int CS, int KS>
__device__ __forceinline__ void xacc_mma(XAccMma<(KS - 1) / 16>& x, const float2* C, const float2* Yc) {
  static_assert(KS % 16 == 1 && (CS % 16 == 9 || CS % 16 == 1), "fragment permutations assume these strides");
  constexpr int NTW = (KS - 1) / 16;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int pg = perm_s1(g);
  const float2* ccol = C + t * CS + 16 * (w >> 1) + pg;
  const float2* ycol = Yc + t * KS + pg;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int i0 = 8 * s;
    CFragA a;  // A[m][kk] = conj(C[i0 + kk][m0 + m])
    a.set(0, ccol[i0 * CS]);
    a.set(1, ccol[i0 * CS + 2]);
    a.set(2, ccol[(i0 + 4) * CS]);
    a.set(3, ccol[(i0 + 4) * CS + 2]);
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      const int cb = tile_col_s1(NTW * (w & 1) + j);
      CFragB b;
      b.set(0, ycol[i0 * KS + cb]);
      b.set(1, ycol[(i0 + 4) * KS + cb]);
      cmma<true, false>(x.xr[j], x.xi[j], a, b);
    }
  }
}

// Stores the accumulators; perm (optional) maps a column to its destination.
template <int DP, int KS>
__device__ __forceinline__ void xacc_store_perm(const XAccMma<(KS - 1) / 16>& x, float2* X, const int* perm) {
  constexpr int NTW = (KS - 1) / 16;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = 16 * (w >> 1) + perm_s1(g);
#pragma unroll
  for (int j = 0; j < NTW; ++j) {
    const int cb = tile_col_s1(NTW * (w & 1) + j);
    int c0 = cb + perm_s1(2 * t), c1 = cb + perm_s1(2 * t + 1);
    if (perm) {
      c0 = perm[c0];
      c1 = perm[c1];
    }
    if (m0 < DP) {
      X[m0 * KS + c0] = make_float2(x.xr[j][0], x.xi[j][0]);
      X[m0 * KS + c1] = make_float2(x.xr[j][1], x.xi[j][1]);
    }
    if (m0 + 2 < DP) {
      X[(m0 + 2) * KS + c0] = make_float2(x.xr[j][2], x.xi[j][2]);
      X[(m0 + 2) * KS + c1] = make_float2(x.xr[j][3], x.xi[j][3]);
    }
  }
}
template <int DP, int KS>
__device__ __forceinline__ void xacc_store(const XAccMma<(KS - 1) / 16>& x, float2* X) {
  xacc_store_perm<DP, KS>(x, X, nullptr);
}

// acc (DP x KB) = V M: V a DP x KS block, M a KB x KS matrix.
template <int KS, int KB>
__device__ __forceinline__ void vu_mma(XAccMma<KB / 16>& x, const float2* V, const float2* U) {
  static_assert((KB == 48 || KB == 32) && KS == KB + 1, "32- or 48-column block");
  constexpr int NTW = KB / 16;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int pg = perm_s1(g);
  const float2* arow = V + (16 * (w >> 1) + pg) * KS + t;
  const float2* bcol = U + t * KS + pg;
#pragma unroll 2
  for (int s = 0; s < KB / 8; ++s) {
    const int k0 = 8 * s;
    CFragA a;
    a.set(0, arow[k0]);
    a.set(1, arow[2 * KS + k0]);
    a.set(2, arow[k0 + 4]);
    a.set(3, arow[2 * KS + k0 + 4]);
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      const int cb = tile_col_s1(NTW * (w & 1) + j);
      CFragB b;
      b.set(0, bcol[k0 * KS + cb]);
      b.set(1, bcol[(k0 + 4) * KS + cb]);
      cmma<false, false>(x.xr[j], x.xi[j], a, b);
    }
  }
}

// H (48 x 48) += Y^H Y over 8 ksteps rows of Y (row stride KS): the upper
// block triangle only (six 16 x 16 blocks mt <= grp, two 8-column tiles
// each) on warps 0-11, one tile per warp in eight chains; the strictly lower
// blocks are the conjugate transposes (gram_at).
struct HAccMma {
  CAcc8 acc;
  __device__ __forceinline__ void zero() { acc.zero(); }
};
// tile w of the upper block triangle of an NBK x NBK grid of 16 x 16 blocks
// (NBK = 3: 12 tiles, NBK = 2: 6 tiles); false beyond the last tile
template <int NBK>
__device__ __forceinline__ bool sym_tile(int w, int& mt, int& grp, int& sub) {
  static_assert(NBK == 2 || NBK == 3, "32- or 48-column block");
  const int bi = w >> 1;
  sub = w & 1;
  if (NBK == 3) {
    mt = bi < 3 ? 0 : bi < 5 ? 1 : 2;
    grp = bi < 3 ? bi : bi < 5 ? bi - 2 : 2;
    return w < 12;
  }
  mt = bi < 2 ? 0 : 1;
  grp = bi < 2 ? bi : 1;
  return w < 6;
}

template <int KS>
__device__ __forceinline__ void hacc_mma(HAccMma& h, const float2* Y, int ksteps = 4) {
  static_assert(KS % 16 == 1, "fragment permutations assume this stride");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  int mt, grp, sub;
  if (!sym_tile<(KS - 1) / 16>(w, mt, grp, sub)) return;
  const int pg = perm_s1(g);
  const float2* acol = Y + t * KS + 16 * mt + pg;
  const float2* bcol = Y + t * KS + 16 * grp + 2 * sub + pg;
#pragma unroll 2
  for (int s = 0; s < ksteps; ++s) {
    const int i0 = 8 * s;
    CFragA a;  // A[m][kk] = conj(Y[i0 + kk][16 mt + m])
    a.set(0, acol[i0 * KS]);
    a.set(1, acol[i0 * KS + 2]);
    a.set(2, acol[(i0 + 4) * KS]);
    a.set(3, acol[(i0 + 4) * KS + 2]);
    CFragB b;
    b.set(0, bcol[i0 * KS]);
    b.set(1, bcol[(i0 + 4) * KS]);
    h.acc.mma<true, false>(a, b);
  }
}

template <int KS>
__device__ __forceinline__ void hacc_store(const HAccMma& h, float2* Hm) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  int mt, grp, sub;
  if (!sym_tile<(KS - 1) / 16>(w, mt, grp, sub)) return;
  float2* out = Hm + (16 * mt + perm_s1(g)) * KS + 16 * grp + 2 * sub;
  const int c0 = perm_s1(2 * t), c1 = perm_s1(2 * t + 1);
  out[c0] = h.acc.get(0);
  out[c1] = h.acc.get(1);
  out[2 * KS + c0] = h.acc.get(2);
  out[2 * KS + c1] = h.acc.get(3);
}
template <int KS>
__device__ __forceinline__ float2 gram_at(const float2* Sm, int a, int b) {
  return (b >> 4) >= (a >> 4) ? Sm[a * KS + b] : cconj(Sm[b * KS + a]);
}

// Z (32 x DP) = Yc (32 x 8 ks) Vf^H: warp w takes the 16-row tile w & 1 and
// the 16-column group w >> 1 of Z (two tiles).
struct ZAccMma {
  float zr[2][4], zi[2][4];
  // f(row, column, value) for every element this thread holds
  template <int DP, class Fn>
  __device__ __forceinline__ void for_each(Fn&& f) const {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int r0 = 16 * (w & 1) + perm_s1(g);
    if (16 * (w >> 1) >= DP) return;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c0 = 16 * (w >> 1) + 2 * j + perm_s1(2 * t), c1 = 16 * (w >> 1) + 2 * j + perm_s1(2 * t + 1);
      f(r0, c0, make_float2(zr[j][0], zi[j][0]));
      f(r0, c1, make_float2(zr[j][1], zi[j][1]));
      f(r0 + 2, c0, make_float2(zr[j][2], zi[j][2]));
      f(r0 + 2, c1, make_float2(zr[j][3], zi[j][3]));
    }
  }
};

template <int DP, int KS>
__device__ __forceinline__ void zgemm_mma(ZAccMma& z, const float2* Yc, const float2* Vf, int ks) {
  static_assert(DP % 8 == 0 && DP <= 128 && KS % 16 == 1, "at most 8 column groups");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) z.zr[j][i] = z.zi[j][i] = 0.f;
  if (16 * (w >> 1) >= DP) return;  // warp-uniform
  const int pg = perm_s1(g);
  const float2* arow = Yc + (16 * (w & 1) + pg) * KS + t;
  const float2* vrow = Vf + (16 * (w >> 1) + pg) * KS + t;  // B[kk][n] = conj(Vf[n0 + n][k0 + kk])
  for (int s = 0; s < ks; ++s) {
    const int k0 = 8 * s;
    CFragA a;
    a.set(0, arow[k0]);
    a.set(1, arow[2 * KS + k0]);
    a.set(2, arow[k0 + 4]);
    a.set(3, arow[2 * KS + k0 + 4]);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      CFragB b;
      b.set(0, vrow[2 * j * KS + k0]);
      b.set(1, vrow[2 * j * KS + k0 + 4]);
      cmma<false, true>(z.zr[j], z.zi[j], a, b);
    }
  }
}

// In place Yc[:, 0 : 16 nb) <- Yc (32 x 48) Us (48 x 16 nb, row stride US):
// the cached Ahat V rotated (and scaled) into the leading sorted Ritz
// columns.  Warp w < 4 nb owns the tile (row tile w & 1, column tile w >> 1).
// Called by the whole CTA; two barriers.
template <int KS, int US>
__device__ __forceinline__ void ycache_rotate_mma(float2* Yc, const float2* Us, int nb) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int mt = w & 1, tl = w >> 1;
  const bool act = w < 4 * nb;
  const int pg = perm_s1(g);
  float yr[4] = {0.f, 0.f, 0.f, 0.f}, yi[4] = {0.f, 0.f, 0.f, 0.f};
  if (act) {
    const float2* arow = Yc + (16 * mt + pg) * KS + t;
    const float2* bcol = Us + t * US + tile_col_s1(tl) + pg;
#pragma unroll 2
    for (int s = 0; s < (KS - 1) / 8; ++s) {
      const int k0 = 8 * s;
      CFragA a;
      a.set(0, arow[k0]);
      a.set(1, arow[2 * KS + k0]);
      a.set(2, arow[k0 + 4]);
      a.set(3, arow[2 * KS + k0 + 4]);
      CFragB b;
      b.set(0, bcol[k0 * US]);
      b.set(1, bcol[(k0 + 4) * US]);
      cmma<false, false>(yr, yi, a, b);
    }
  }
  __syncthreads();
  if (act) {
    float2* out = Yc + (16 * mt + pg) * KS + tile_col_s1(tl);
    const int c0 = perm_s1(2 * t), c1 = perm_s1(2 * t + 1);
    out[c0] = make_float2(yr[0], yi[0]);
    out[c1] = make_float2(yr[1], yi[1]);
    out[2 * KS + c0] = make_float2(yr[2], yi[2]);
    out[2 * KS + c1] = make_float2(yr[3], yi[3]);
  }
  __syncthreads();
}

// Upper block triangle of S = B^H B (48 x 48, row stride KS) for a DP x KS
// block B (rows beyond d zero); the strictly lower blocks are the conjugate
// transposes (gram_at).
template <int KS>
__device__ __forceinline__ void gram_sym_mma(const float2* B, float2* Sm, int ksteps) {
  HAccMma h;
  h.zero();
  hacc_mma<KS>(h, B, ksteps);
  hacc_store<KS>(h, Sm);
}

// Orthonormal basis of span(X) by Newton-Schulz iteration on the polar
// factor, all contractions on the tensor cores:
//   X_0 = X D (unit columns),  X_{k+1} = X_k (3 I - X_k^H X_k) / 2.
// With E = X_k^H X_k - I the next ||E||_F is <= 0.75 ||E||_F^2, so a warm
// block (X = G V0 with V0 the previous Ritz vectors: nearly orthogonal
// columns of different lengths) needs one or two steps where the Householder
// QR is 48 barrier-separated column steps.  Subspace iteration only needs an
// orthonormal basis of the same span, not the triangular factor.  Returns the
// number of steps, or 0 without touching V when the columns are too far from
// orthogonal (||E_0||_F > 0.5) or degenerate: the caller runs the QR then.
// X: DP x KS block, rows beyond d zero; V: result (may alias X); Sm: KB x KS
// scratch; red: 32 floats of scratch.  Called by the whole CTA.
template <int KB, int KS, int DP>
__device__ int newton_schulz_orth(const float2* X, float2* V, float2* Sm, float* red) {
  static_assert(KB == 48 || KB == 32, "32- or 48-column block");
  constexpr int NT = 512, PER = (KB * KB + NT - 1) / NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float2* B = X;
  int it = 0;
  for (; it < 6; ++it) {
    gram_sym_mma<KS>(B, Sm, DP / 8);
    __syncthreads();
    float2 m[PER];
    float e2 = 0.f;
    bool bad = false;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = tid + NT * q;
      m[q] = make_float2(0.f, 0.f);
      if (idx < KB * KB) {
        const int a = idx / KB, b = idx - a * KB;
        float2 sv = gram_at<KS>(Sm, a, b);
        float da = 1.f;
        if (it == 0) {
          const float saa = Sm[a * KS + a].x, sbb = Sm[b * KS + b].x;
          bad = bad || !(saa > 1e-30f) || !(sbb > 1e-30f);
          da = rsqrtf(saa);
          const float db = rsqrtf(sbb);
          sv = cscale(sv, da * db);
        }
        const float dl = a == b ? 1.f : 0.f;
        const float ex = sv.x - dl, ey = a == b ? 0.f : sv.y;
        e2 = fmaf(ex, ex, fmaf(ey, ey, e2));
        m[q] = make_float2(da * (1.5f * dl - 0.5f * sv.x), a == b ? 0.f : da * (-0.5f * sv.y));
      }
    }
    if (bad) e2 = 1e30f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    if (lane == 0) red[16 * (it & 1) + warp] = e2;
    __syncthreads();  // Sm fully read, partial sums visible
    float err2 = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) err2 += red[16 * (it & 1) + k];
    if (it == 0 && !(err2 <= 0.25f)) return 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = tid + NT * q;
      if (idx < KB * KB) {
        const int a = idx / KB, b = idx - a * KB;
        Sm[a * KS + b] = m[q];
      }
    }
    __syncthreads();
    XAccMma<KB / 16> acc;
    acc.zero();
    vu_mma<KS, KB>(acc, B, Sm);
    __syncthreads();  // in place: all reads of B are done
    xacc_store<DP, KS>(acc, V);
    __syncthreads();
    B = V;
    if (0.75f * err2 < 2e-6f) {  // predicted ||E||_F after this step
      ++it;
      break;
    }
  }
  return it;
}

// Orthonormal basis of span(X) by a Cholesky QR of the column-normalised
// block, contractions on the tensor cores:
//   S' = D X^H X D = L L^H  (D = column norms^-1),  Q = X D L^-H.
// The Householder QR of the warm pass is 48 barrier-separated column steps
// (~93 k cycles); here the Gram matrix and the final product are two short
// mma.sync phases and only the 48 x 48 factorisation is serial.  Column
// normalisation removes the scale spread of X = G V0 (columns ~ lambda_j v_j),
// after which cond(S') is modest; the loss of orthogonality is eps cond(S').
// Returns 1, or 0 without touching V when a pivot falls below `pivtol` (the
// caller runs the Householder QR then).
// X: DP x KS block, rows beyond d zero; V: result (may alias X); Sm, Mb:
// KB x KS scratch each (Mb may alias V when V does not alias X); dinv: KB
// floats; flag: one int.  Called by the whole CTA (512 threads).
template <int KB, int KS, int DP>
__device__ int cholesky_qr_mma(const float2* X, float2* V, float2* Sm, float2* Mb, float* dinv, int* flag,
                               float pivtol, long long* clk = nullptr) {
  static_assert(KB == 48 || KB == 32, "32- or 48-column block");
  constexpr int NT = 512, PER = (KB * KB + NT - 1) / NT;
  const int tid = threadIdx.x;
  // diagnostics: durations of Gram + scaling / Cholesky / inverse / product
  // into clk[0], clk[1], clk[2], clk[7] (phase slots 13, 14, 15, 20 are taken: see the caller)
  long long t_ = clk ? clock64() : 0;
#define CQR_ACC(k)                         \
  if (clk && tid == 0) {                   \
    const long long n_ = clock64();        \
    clk[k] = n_ - t_;                      \
    t_ = n_;                               \
  }
  gram_sym_mma<KS>(X, Sm, DP / 8);
  if (tid == 0) *flag = 0;
  __syncthreads();
  // ---- S' = D S D, full Hermitian, through registers (in place)
  {
    float2 m[PER];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = tid + NT * q;
      m[q] = make_float2(0.f, 0.f);
      if (idx < KB * KB) {
        const int a = idx / KB, b = idx - a * KB;
        const float saa = Sm[a * KS + a].x, sbb = Sm[b * KS + b].x;
        bad = bad || !(saa > 1e-30f) || !(sbb > 1e-30f);
        const float da = rsqrtf(saa), db = rsqrtf(sbb);
        m[q] = a == b ? make_float2(1.f, 0.f) : cscale(gram_at<KS>(Sm, a, b), da * db);
        if (b == 0) dinv[a] = da;
      }
    }
    if (__syncthreads_or(bad)) return 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = tid + NT * q;
      if (idx < KB * KB) Sm[(idx / KB) * KS + (idx % KB)] = m[q];
    }
  }
  __syncthreads();
  CQR_ACC(0);
  // ---- Cholesky and the inverse factor in one right-looking sweep, all 16
  // warps, one barrier per column.  Every thread keeps up to PERL elements
  // (i, k), i >= k, in registers: the trailing-matrix value S(i, k) until
  // column k is final (after step k - 1), then B(i, k), the forward
  // substitution of the identity (L^-1 = diag(d)^-1/2 B).  With the unscaled
  // column C_j = L[:, j] sqrt(d_j), d_j = C_j[j], step j is one rank-1 update
  // for both roles,
  //     v(i, k) -= (C_j[i] / d_j) g_j[k],   g_j = [B(j, 0..j-1), 1, conj(C_j[j+1..])],
  // so row j of the work matrix Gm (= Mb) holds g_j (and C_j[i] = conj(g_j[i])),
  // published by the owners of column j / of row j of B at step j - 1; d_j
  // goes to the diagonal of Sm.  (The left-looking factorisation on two warps
  // plus the 8-lane substitution this replaces took 174 k of the co-located
  // CTA's 1175 k cycles; a first fused version with separate branches for the
  // two roles was issue-bound at ~300 instructions per warp and step.)
  {
    constexpr int NL = KB * (KB + 1) / 2, PERL = (NL + NT - 1) / NT;
    int eik[PERL];
    float2 ev[PERL];
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int e = tid + NT * q;
      int i = (int)((sqrtf(8.f * (float)e + 1.f) - 1.f) * 0.5f);
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      while (i * (i + 1) / 2 > e) --i;
      const int k = e - i * (i + 1) / 2;
      eik[q] = e < NL ? (i | (k << 8)) : 0;  // (i = 0: never active)
      ev[q] = make_float2(0.f, 0.f);         // column 0 is final: B role
      if (e < NL) {
        const float2 sv = Sm[i * KS + k];
        if (k > 0) ev[q] = sv;
        else Mb[i] = i == 0 ? make_float2(1.f, 0.f) : cconj(sv);  // g_0
      }
    }
    for (int j = 0; j < KB; ++j) {
      __syncthreads();  // g_j and d_j are published
      const float dj = Sm[j * KS + j].x;
      if (!(dj > pivtol)) *flag = 1;  // (every thread writes the same value)
      const float inv = 1.f / fmaxf(dj, 1e-30f);
      const float2* gj = Mb + j * KS;
      float2* gn = Mb + (j + 1) * KS;
      // (all loads before the first publishing store: the compiler cannot
      // reorder them across a store that may alias)
      float2 ga[PERL], gg[PERL];
#pragma unroll
      for (int q = 0; q < PERL; ++q) {
        const int i = eik[q] & 0xff, k = eik[q] >> 8;
        ga[q] = gj[i];
        gg[q] = gj[k];
      }
#pragma unroll
      for (int q = 0; q < PERL; ++q) {
        const int i = eik[q] & 0xff, k = eik[q] >> 8;
        if (i > j) {
          const float2 a = ga[q], g = gg[q];
          const float cx = a.x * inv, cy = -a.y * inv;  // C_j[i] / d_j
          float2 v = ev[q];
          v.x -= cx * g.x - cy * g.y;
          v.y -= cx * g.y + cy * g.x;
          if (k == j + 1) {  // column j + 1 is final: publish, switch to the B role
            if (i == k) {
              Sm[k * KS + k] = make_float2(v.x, 0.f);
              gn[k] = make_float2(1.f, 0.f);
            } else {
              gn[i] = cconj(v);
            }
            v = make_float2(0.f, 0.f);
          } else if (i == j + 1) {  // row j + 1 of B is final
            gn[k] = v;
          }
          ev[q] = v;
        }
      }
    }
  }
  __syncthreads();
  CQR_ACC(1);
  if (*flag) return 0;
  // ---- M = D W^H, W = L^-1: M[c][i] = dinv[c] conj(W[i][c]) = dinv[c] conj(B(i, c)) / sqrt(d_i), i >= c,
  // B(i, c) = Gm[i][c]: transposed in place through registers
  {
    float2 m[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int t = tid + NT * q;
      m[q] = make_float2(0.f, 0.f);
      if (t < KB * KB) {
        const int c = t / KB, i = t - c * KB;
        if (i >= c) {
          const float w = dinv[c] * rsqrtf(Sm[i * KS + i].x);
          m[q] = i == c ? make_float2(w, 0.f) : cscale(cconj(Mb[i * KS + c]), w);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int t = tid + NT * q;
      if (t < KB * KB) Mb[(t / KB) * KS + (t % KB)] = m[q];
    }
  }
  __syncthreads();
  CQR_ACC(2);
  XAccMma<KB / 16> acc;
  acc.zero();
  vu_mma<KS, KB>(acc, X, Mb);
  __syncthreads();  // all reads of X and of Mb (which may alias V) are done
  xacc_store<DP, KS>(acc, V);
  __syncthreads();
  CQR_ACC(10);
#undef CQR_ACC
  return 1;
}

}  // namespace shlr_b200
