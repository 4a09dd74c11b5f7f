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

#include <vector>

#include "solver_util.cuh"
#include "svt_device.cuh"
#include "svt_subspace_launch.cuh"

namespace shlr_b200 {

size_t svt_subspace_smem_bytes(int DP, int KB, int R, int maxB, int maxLen, int maxE, bool big, bool coloc) {
  const int KS = KB + 1, CS = DP + 1;
  // co-located layout: chunk buffer padded to hold the eigen-solver's work area (CROWS in the kernel)
  const int crows = (coloc && 2 * R * CS < 3 * KB * KB) ? (3 * KB * KB / 2 + CS - 1) / CS : R;
  const size_t spectra = big ? 3ull * maxLen : 2ull * maxB * maxLen;
  const bool huge = big && R == 16;
  const bool nosplit = big && KB > kSubspaceKB;  // BIG level 2
  const size_t yreg = huge      ? (size_t)R * KS
                      : nosplit ? (size_t)std::max(R * KS, KB * KS + 3 * KB * KB / 2 - R * CS)
                                : 2ull * R * KS;
  return sizeof(float2) * ((big ? 1ull : 2ull) * DP * KS + (size_t)crows * CS + yreg + spectra) +
         sizeof(SlotRec) * KB + sizeof(double2) * KB + sizeof(double) * KB + 2 * sizeof(float) * KB +
         16 * sizeof(int) + sizeof(int) * KB + sizeof(int) * std::max(DP, maxE) + 64;
}

namespace {

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
    if (!prm.wl_global) stage_spectra(S.wl, F, sp, weighted, tid, NT);
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
  if (g.dmax < 72) {  // small d: 16-column level 1, 32-column level 2
    if (g.dmin < kSubspaceSmallMinD) return false;
    constexpr int KBs = L2 ? kSubspaceKB1 : kSubspaceKBSmall;
    const int dp = svt_padded_dim(g.dmax);
    const size_t smem = svt_subspace_smem_bytes(dp, KBs, 32, g.maxB, g.maxLen, g.maxE, false);
    if (smem > 227 * 1024) return false;
    return launch_sub_small(dp, KBs, L2, prm, total, smem, stream);
  }
  if (g.dmin < kSubspaceKB + 24) return false;
  if (g.dmax > 248) {
    // HUGE variant: 32-column block, 16-row chunks (every level is KB 32)
    if (g.maxLen > 0xffff) return false;
    for (int f = 0; f < prm.nfam; ++f)
      if (prm.fam[f].vc && prm.mode != SVT_ADMM_WEIGHTED) return false;
    const int dph = svt_huge_padded_dim(g.dmax);
    if (!dph) return false;
    const size_t smem = svt_subspace_smem_bytes(dph, kSubspaceKBHuge, 16, g.maxB, g.maxLen, g.maxE, true);
    if (smem > 227 * 1024) return false;
    return launch_sub_huge(dph, L2, prm, total, smem, stream);
  }
  // 112 < d <= 120 with a 48-column level 1 (the headline, config 2: 242 x
  // 120): the large-d layout (spectra and duals read from L2, the adjoint
  // read-modify-written in place, no split staging: 111 KB of shared memory)
  // lets two CTAs share an SM, so one matrix's latency-bound QR and
  // Rayleigh-Ritz phases overlap the other's chunk GEMMs (1.74 -> 1.66 ms
  // per config-2 launch, same arithmetic).  Level 2 and the full solver
  // behind it are unchanged.
  static const bool coloc = std::getenv("SHLR_NO_COLOC") == nullptr;
  // The chunk contractions run as 3xTF32 on the tensor cores (svt_mma.cuh)
  // and warm passes orthonormalise by a tensor-core Cholesky QR; SHLR_MMA=0 /
  // SHLR_NS=0 keep the FP32 CUDA-core contractions / the Householder QR
  // (config 2, per launch: 1.66 ms FP32 -> 1.40 ms)
  static const bool mma = !std::getenv("SHLR_MMA") || std::atoi(std::getenv("SHLR_MMA")) != 0;
  static const int ns = std::getenv("SHLR_NS") ? std::atoi(std::getenv("SHLR_NS")) : 1;
  SvtParams pm = prm;
  pm.ns_orth = ns;
  if (coloc && !L2 && KB1 == kSubspaceKB && svt_padded_dim(g.dmax) == 120 && g.dmin >= 72 && g.maxLen <= 0xffff) {
    const size_t smem = svt_subspace_smem_bytes(120, kSubspaceKB, 32, g.maxB, g.maxLen, g.maxE, true);
    if (2 * (smem + 1024) <= 228 * 1024)
      return mma ? launch_sub_mma(120, kSubspaceKB, false, true, pm, total, smem, stream)
                 : launch_sub_big(120, false, prm, total, smem, stream);
  }
  // config 1 (256 lifts of 120 x 72): same layout with the chunk buffer padded to
  // the eigen-solver's work area; 256 CTAs on 2 x 148 slots are one wave
  // instead of 1.73 with one CTA per SM (tensor variant only)
  static const bool coloc_c1 = std::getenv("SHLR_NO_COLOC_C1") == nullptr;
  if (coloc && coloc_c1 && mma && !L2 && KB1 == kSubspaceKB && svt_padded_dim(g.dmax) == 72 && g.dmin >= 72 &&
      g.maxLen <= 0xffff) {
    bool vc_ok = true;
    for (int f = 0; f < prm.nfam; ++f) vc_ok = vc_ok && !(prm.fam[f].vc && prm.mode != SVT_ADMM_WEIGHTED);
    const size_t smem = svt_subspace_smem_bytes(72, kSubspaceKB, 32, g.maxB, g.maxLen, g.maxE, true, true);
    if (vc_ok && 2 * (smem + 1024) <= 228 * 1024 && launch_sub_mma(72, kSubspaceKB, false, true, pm, total, smem, stream))
      return true;
  }
  // the parameter path's PE lifts (config 4: 244 x 104, 32-column level 1): same layout, tensor variant only
  static const bool coloc_pe = std::getenv("SHLR_NO_COLOC_PE") == nullptr;
  if (coloc && coloc_pe && mma && !L2 && KB1 == kSubspaceKB1 && svt_padded_dim(g.dmax) == 104 && g.dmin >= 72 &&
      g.maxLen <= 0xffff) {
    bool vc_ok = true;  // (plain lifts have no virtual coils in the large-d layout)
    for (int f = 0; f < prm.nfam; ++f) vc_ok = vc_ok && !(prm.fam[f].vc && prm.mode != SVT_ADMM_WEIGHTED);
    const size_t smem = svt_subspace_smem_bytes(104, kSubspaceKB1, 32, g.maxB, g.maxLen, g.maxE, true);
    if (vc_ok && 2 * (smem + 1024) <= 228 * 1024 &&
        launch_sub_mma(104, kSubspaceKB1, false, true, pm, total, smem, stream))
      return true;
  }
  if (mma && g.dmax <= 128) {
    // resident layout (one CTA per SM): Householder QR (the Cholesky QR only
    // pays at 64 registers)
    constexpr int KBm = L2 ? kSubspaceKB : KB1;
    const int dp = svt_padded_dim(g.dmax);
    const size_t smem = svt_subspace_smem_bytes(dp, KBm, 32, g.maxB, g.maxLen, g.maxE, false);
    if (smem <= 227 * 1024 && launch_sub_mma(dp, KBm, L2, false, prm, total, smem, stream)) return true;
  }
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
    return launch_sub_big(dpb, L2, prm, total, smem, stream);
  }
  constexpr int KB = L2 ? kSubspaceKB : KB1;
  const int dp = svt_padded_dim(g.dmax);
  const size_t smem = svt_subspace_smem_bytes(dp, KB, 32, g.maxB, g.maxLen, g.maxE, false);
  if (smem > 227 * 1024) return false;
  return launch_sub_small(dp, KB, L2, prm, total, smem, stream);
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
  const bool big = dmax > 128, huge = dmax > 248, small = dmax < 72;
  if (big) kb1 = kSubspaceKB;
  if (small) kb1 = kSubspaceKBSmall;
  // HUGE level 1 hands its leading 24 of 32 Ritz pairs to the chain when the
  // rank exceeds the block: cold starts need 8 passes for that head to be
  // invariant enough (4 left 1.5e-4 at rank ~40, 8 left < 1e-4)
  SvtParams s1 = sp;
  if (huge) s1.q_cold = std::max(s1.q_cold, 8);
  if (!launch_hankel_svt_subspace(s1, total, stream, kb1)) return 0;
  int n = 1;
  if ((big && !huge) || kb1 == kSubspaceKB1 || small) {  // (HUGE: level 1 hands straight to the chain)
    SvtParams l2 = sp;
    l2.only_flagged = sp.fam[0].fallback;
    l2.q_cold = std::getenv("SHLR_L2_Q") ? std::atoi(std::getenv("SHLR_L2_Q")) : 8;
    l2.l2_warm_passes = std::getenv("SHLR_L2_WARM_Q") ? std::atoi(std::getenv("SHLR_L2_WARM_Q")) : 2;
    l2.l2_pass_margin = std::getenv("SHLR_L2_MARGIN") ? std::atoi(std::getenv("SHLR_L2_MARGIN")) : 16;
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
  fs.only_flag_value = (kb1 == kSubspaceKB1 || small) ? kLevelOverflow : kLevelHanded;
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

namespace {
// Lift stage of the Hankel-SVT kernels on one matrix, dumped: the same
// staging (stage_spectra, build_lofs) and chunk builders the kernels run --
// path 0: load_chunk / lift_elem (full solver), path 1: build_chunk /
// lift_tab (subspace solver, d <= 128), path 2: build_chunk_big / lift_global
// (large-d subspace variants) -- writing Ahat (e x d, row-major).  Used on
// index-encoded spectra by lift_index_map_device.
constexpr int kDumpDP = 256, kDumpR = 32;
__global__ void k_lift_dump(const SvtFamily F, int path, float2* ahat) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int CS = kDumpDP + 1;
  float2* chunk = reinterpret_cast<float2*>(smem_raw);      // R x CS (path 0: R x DP)
  float2* wl = chunk + kDumpR * CS;                         // B x len
  float2* wcs = wl + F.B * F.len;                           // len
  int* lofs = reinterpret_cast<int*>(wcs + F.len);          // max(d, e)
  const float2* sp = F.spec;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (path == 2) {
    for (int t = tid; t < F.len; t += nt) wcs[t] = F.wc[t];
    build_lofs(lofs, F, true, tid, nt);
  } else {
    stage_spectra(wl, F, sp, true, tid, nt);
    build_lofs(lofs, F, false, tid, nt);
  }
  __syncthreads();
  Smem<kDumpDP> S{};
  S.wl = wl;
  S.A = chunk;
  for (int i0 = 0; i0 < F.e; i0 += kDumpR) {
    const int rows = min(kDumpR, F.e - i0);
    if (path == 0) load_chunk<kDumpDP, kDumpR>(S, F, nullptr, i0, rows, 0.f, false);
    else if (path == 1) build_chunk<kDumpDP, CS, kDumpR>(chunk, wl, lofs, F, nullptr, i0, rows, 0.f);
    else build_chunk_big<kDumpDP, CS, kDumpR>(chunk, F, sp, wcs, true, lofs, nullptr, i0, rows, 0.f);
    __syncthreads();
    const int stride = path == 0 ? kDumpDP : CS;
    for (int t = tid; t < rows * F.d; t += nt) {
      const int r = t / F.d, u = t - r * F.d;
      ahat[(long long)(i0 + r) * F.d + u] = chunk[r * stride + u];
    }
    __syncthreads();
  }
}
}  // namespace

void lift_index_map_device(int n, int p, int coils, int vc, int path, int32_t* map_host) {
  const int q = n - p + 1, J = coils, B = coils * (vc ? 2 : 1);
  const int P = p, Bq = B * q, e = std::max(P, Bq), d = std::min(P, Bq);
  if (d > kDumpDP || path < 0 || path > 2) throw InvalidArg("lift_index_map: geometry outside the dump kernel");
  // index-encoded spectra: s_j[n] = (j + 1) + i (n + 1), unit weights (taps = [1])
  std::vector<float2> spec((size_t)n * J), wc(n, make_float2(1.f, 0.f));
  for (int t = 0; t < n; ++t)
    for (int j = 0; j < J; ++j) spec[(size_t)t * J + j] = make_float2((float)(j + 1), (float)(t + 1));
  float2 *dspec = util::dalloc<float2>(spec.size()), *dwc = util::dalloc<float2>(n),
         *dah = util::dalloc<float2>((size_t)e * d);
  SHLR_CUDA(cudaMemcpy(dspec, spec.data(), spec.size() * sizeof(float2), cudaMemcpyHostToDevice));
  SHLR_CUDA(cudaMemcpy(dwc, wc.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
  SvtFamily F{};
  F.count = 1;
  F.len = n;
  F.P = P;
  F.q = q;
  F.J = J;
  F.B = B;
  F.vc = vc;
  F.wide = Bq > P ? 1 : 0;
  F.e = e;
  F.d = d;
  F.spec = dspec;
  F.s_mat = 0;
  F.s_n = J;
  F.s_j = 1;
  F.wc = dwc;
  const size_t smem = sizeof(float2) * ((size_t)kDumpR * (kDumpDP + 1) + (size_t)B * n + n) + sizeof(int) * e + 64;
  SHLR_CUDA(cudaFuncSetAttribute(k_lift_dump, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  k_lift_dump<<<1, 512, smem>>>(F, path, dah);
  SHLR_LAUNCH_CHECK();
  std::vector<float2> ah((size_t)e * d);
  SHLR_CUDA(cudaMemcpy(ah.data(), dah, ah.size() * sizeof(float2), cudaMemcpyDeviceToHost));
  cudaFree(dspec);
  cudaFree(dwc);
  cudaFree(dah);
  // decode A[i][c] (Ahat = A tall, A^H wide): coil = re - 1, index = |im| - 1, conj = im < 0
  for (int i = 0; i < P; ++i)
    for (int c = 0; c < Bq; ++c) {
      float2 v = F.wide ? ah[(size_t)c * d + i] : ah[(size_t)i * d + c];
      if (F.wide) v.y = -v.y;
      int32_t* m = map_host + 3 * ((size_t)i * Bq + c);
      m[0] = (int32_t)lrintf(v.x) - 1;
      m[1] = (int32_t)lrintf(fabsf(v.y)) - 1;
      m[2] = v.y < 0.f ? 1 : 0;
    }
}

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
