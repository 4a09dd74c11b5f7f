// Fused batched Hankel-SVT kernel: one CTA per lifted matrix.
//
// Per matrix (proj/src/solvers.cpp:172-181 for the ADMM mode, and the
// lift_plain -> svt -> adjoint_lift_plain composition of solvers.cpp:264-282
// for the plain mode):
//   0. stage the J coil spectra of one k-space row/column in smem, weighted by
//      the centred filter spectrum wc and, with virtual coils, conjugate-
//      flipped (lift_weighted, operators.cpp:25-58);
//   1. Gram  G = Ahat^H Ahat  (FP32 FMA), Ahat = L + D/beta streamed in row
//      chunks of R (Ahat = A for tall A, A^H for wide A; d = min(m, n));
//   2. cyclic parallel two-sided Jacobi on G (Brent-Luk ring ordering): G in
//      smem (upper representation, stride d+1 so row and column walks are
//      bank-conflict free), V in registers, 4 threads per row of V, one ring
//      shift per round done with register moves and width-4 shuffles;
//   3. f = (1 - tau/sigma)_+ and W = V diag(f) V^H (W replaces G in smem);
//   4. Zhat = Ahat W per chunk, fused dual update D += tau_d (L - Z), and
//      T = Z - D/beta (ADMM) or T = Z (plain);
//   5. Hankel adjoint of T (deterministic anti-diagonal sums, no atomics) and
//      the adjoint weighting conj(wc) (+ virtual-coil dagger)
//      (adjoint_lift_weighted, operators.cpp:60-91).
// Output is the k-space contribution of this row/column to the next RHS.
#pragma once

#include "common.cuh"

namespace shlr_b200 {

enum SvtMode : int { SVT_ADMM_WEIGHTED = 0, SVT_PLAIN = 1, SVT_ADMM_PLAIN = 2 };

struct SvtFamily {
  int count;           // matrices in this family
  int len;             // vector length (N for rows, M for columns)
  int P;               // pencil = rows of A
  int q;               // len - P + 1
  int J;               // coils
  int B;               // blocks = J * (vc ? 2 : 1)
  int vc;
  int wide;            // 1: B*q > P, Ahat = A^H
  int e, d;            // e = max(P, B*q), d = min(P, B*q)
  // spectra in: element (mat, n, j) at spec[mat*s_mat + n*s_n + j*s_j]
  const float2* spec;
  long long s_mat, s_n, s_j;
  // adjoint out, same addressing convention
  float2* out;
  long long o_mat, o_n, o_j;
  const float2* wc;    // centred weights (len) for weighted modes
  float2* D;           // duals, per matrix e*d row-major (Ahat orientation)
  float* sv;           // optional: count x d singular values (descending)
  float2* V;           // full solver: count x DP x DP eigenvector store (V1 spill and
                       // the ADMM warm start; DP = svt_padded_dim of the launch)
  float2* Vs;          // subspace solver: count x DP x KB dominant-subspace store
  int* rank_prev;      // optional: Ritz values above the threshold in the previous solve of each matrix
  int* fallback;       // subspace solver: per-matrix flag, 1 = rank above threshold too
                       // close to KB, the full solver must redo this matrix
  float2* Z1;          // large d: count x e x d buffer for the deflation chain's Z1
                       // (nullptr: no deflation; also requires Vd and ndefl)
  float2* Vd;          // large d: count x DP x DP deflation basis (row-major, the leading
                       // ndefl[mat] columns hold the Ritz vectors already solved)
  int* ndefl;          // large d: per-matrix column count of Vd
  float2* Vs2;         // large-d level 2: count x DP x kSubspaceKBBig store (warm start of the
                       // matrices that stay at level 2); nullptr: level 2 always starts seeded
  const int* halt;     // optional per-group stop flags: matrix `mat` is skipped when
  int halt_div;        // halt[mat / halt_div] != 0 (independent ADMM problems batched in
                       // one launch, each with its own early stop: parammap.cpp:37-51)
};

struct SvtParams {
  SvtFamily fam[2];
  int nfam;
  int mode;
  float inv_beta;      // 1/beta
  float tau_dual;      // ADMM multiplier step tau
  float thresh;        // SVT threshold (1/beta or lambda2/beta or user tau)
  int max_sweeps;
  const int* skip;     // optional device flag: nonzero -> kernel is a no-op
  const int* warm;     // optional device flag: nonzero -> V holds a warm start
  int* sweeps_out;     // optional diagnostics: Jacobi sweeps used per matrix
  int q_cold, q_warm;  // subspace solver: iterations from a random / stored start
  int rr_orth_mode;      // Rayleigh-Ritz eigenvectors: 0 first-order symmetric correction (Gram-Schmidt fallback), 2 Gram-Schmidt, 1 none
  int l2_warm_passes;    // large-d level 2: warm passes per ADMM iteration (0 / 1: as q_warm)
  int l2_pass_margin;    // ... only for matrices whose previous rank is within this margin of the block (0: all)
  long long* phase_clk;  // optional diagnostics: kPhaseSlots clock64 stamps per matrix
  const int* only_flagged;  // nonzero pointer -> process only matrices whose fallback flag is
                            // set (fam[f].fallback); with only_flag_value != 0 (full solver):
                            // only matrices whose flag equals it
  int only_flag_value;
  int deflate;         // large-d level 3 launch (SvtFamily::Z1, flags kLevelDeflate)
  float rr_tol_rel, rr_tol_abs;  // subspace Rayleigh-Ritz rotation tolerances (0 = defaults)
  float rr_tail;                 // pairs with both Ritz values < rr_tail * thresh^2 not rotated
  float s2_tail;                 // full solver, stage 2: same rule (0 = rotate every pair)
  float s2_tol_abs;              // full solver, stage 2: absolute floor x max diagonal (0 = none)
  int rr_jacobi;                 // 1: Rayleigh-Ritz by parallel Jacobi instead of tridiagonal + bisection
  int inner_norm;                // warm: normalise (instead of QR) after all but the last pass
  const double* relc;            // optional: the ADMM relative change of the previous outer
                                 // iteration (device); while it is large the warm start is
                                 // far from the new subspace and warm solves take more passes
  float relc_q2, relc_q3;        // relc above these: at least 2 / 3 warm passes (with QR)
  int ns_orth;         // tensor-core variants: warm passes orthonormalise by Newton-Schulz
                       // (svt_mma.cuh) instead of the Householder QR
  float2* ycache;      // optional scratch, total_matrices x max e x kSubspaceKB: the tensor-core
                       // variants keep Ahat V of the Rayleigh-Ritz pass for the Z pass
  int wl_global;       // set by launch_hankel_svt: the lift source is read straight from
                       // fam[f].spec (plain mode, contiguous coils) instead of an smem copy
};

// Stage-2 Jacobi rules of the full solver in the ADMM modes (SvtParams::s2_tail,
// s2_tol_abs).
constexpr float kS2Tail = 0.25f;
constexpr float kS2TolAbs = 1e-8f;
// Block sizes of the subspace SVT solver's levels.  d <= 128: level 1 with
// kSubspaceKB columns, then the full solver; or level 1 kSubspaceKB1, level 2
// kSubspaceKB, then the full solver (low-rank families: the parameter path's
// PE lifts).  d > 128 (large-d variant): level 1 kSubspaceKB, level 2
// kSubspaceKBBig, then nothing.
constexpr int kSubspaceKB1 = 32;
constexpr int kSubspaceKB = 48;
// Small d (40 <= d < 72, config-5 points 250 x 56, 122 x 56, 506 x 56): level 1
// with kSubspaceKBSmall columns, level 2 with kSubspaceKB1, then the full solver.
constexpr int kSubspaceKBSmall = 16;
constexpr int kSubspaceSmallMinD = 40;
// Large-d variant (128 < d <= 248, wide matrices): the same block size, with
// spectra and adjoint accumulators not resident in shared memory.  Its
// fallback for matrices whose rank above the threshold exceeds
// kSubspaceKB - kSubspaceMargin is the same kernel with a kSubspaceKBBig
// block (no split-k buffer); a matrix beyond kSubspaceKBBig - kSubspaceMargin
// there keeps its flag, which the host reports as unsupported.
constexpr int kSubspaceKBBig = 64;
// HUGE variant (248 < d <= 496): the block of level 1 and of every deflation step.
constexpr int kSubspaceKBHuge = 32;
// Per-matrix fallback flag values of the large-d levels.
constexpr int kLevelHanded = 1;    // level 1 handed the matrix to level 2 in this launch
constexpr int kLevelOverflow = 2;  // level 2 ran out of block: reported as unsupported
constexpr int kLevelStay2 = 3;     // stays at level 2 (warm from its own store) next iteration
constexpr int kLevelDeflate = 4;   // large d: level 2 keeps its leading kDeflateK Ritz pairs (Z1),
                                   // level 3 solves the orthogonal remainder (again deflating its
                                   // own leading pairs while the remainder exceeds its block)
constexpr int kLevelDeflDone = 5;  // large d: the deflation chain finished this matrix
// Ritz pairs each deflation step keeps (the converged head of a 64 block).
constexpr int kDeflateK = kSubspaceKBBig - 8;
// Level-3 launches the chain needs for dimension d: level 2 deflates
// kDeflateK, every level-3 step kDeflateK more until the remainder fits one
// kSubspaceKBBig block (then the block spans it: exact).
// (HUGE: level 1 deflates kSubspaceKBHuge - 8, each step as many again,
// until the remainder fits one kSubspaceKBHuge block.)
inline int svt_deflation_steps(int d) {
  const bool huge = d > 248;
  const int step = huge ? kSubspaceKBHuge - 8 : kDeflateK, kb = huge ? kSubspaceKBHuge : kSubspaceKBBig;
  int rem = d - step, n = 1;
  while (rem > kb) {
    rem -= step;
    ++n;
  }
  return n;
}
// Padded dimension of the large-d variant for d (0 if out of range).
inline int svt_big_padded_dim(int d) { return d <= 128 ? 0 : d <= 160 ? 160 : d <= 192 ? 192 : d <= 248 ? 248 : 0; }
// HUGE variant (248 < d <= 496: config-5 points 498 x 480 and 482 x 992):
// 16-row chunks and a 32-column block for level 1 and every deflation step.
inline int svt_huge_padded_dim(int d) { return d <= 248 ? 0 : d <= 320 ? 320 : d <= 384 ? 384 : d <= 496 ? 496 : 0; }
int svt_padded_dim(int d);
// Row count of the per-matrix subspace store (F.Vs: store_dim x kSubspaceKB)
// the subspace kernels use for dimension d.
inline int svt_subspace_store_dim(int d) {
  return d > 248 && svt_huge_padded_dim(d) ? svt_huge_padded_dim(d)
         : d > 128 && svt_big_padded_dim(d) ? svt_big_padded_dim(d)
                                            : svt_padded_dim(d);
}
// clock64 diagnostics slots per matrix (SvtParams::phase_clk)
constexpr int kPhaseSlots = 24;
// Matrices with more than KB - margin singular values above the threshold
// are redone by the full eigen-solver.
constexpr int kSubspaceMargin = 8;
// Margin of the last level (large-d fallback block): it has nothing behind it.
constexpr int kSubspaceMarginLast = 2;

// Subspace SVT: the thresholded spectral function needs only the eigenpairs
// of G = Ahat^H Ahat with sigma > tau.  Subspace iteration on a KB-column
// block (one fused streaming pass over Ahat per iteration: X = Ahat^H (Ahat V),
// then Householder QR), a final Rayleigh-Ritz projection H = (Ahat V)^H
// (Ahat V) solved by the Jacobi kernel, and the same fused Z / dual / adjoint
// epilogue.  Returns false (no launch) when the geometry is outside its range.
bool launch_hankel_svt_subspace(const SvtParams& prm, int total, cudaStream_t stream,
                                int kb1 = kSubspaceKB);
// Level 2 of the subspace solver for the matrices level 1 handed over or
// kept at level 2 (prm.only_flagged = the flags; fam[f].Vs2 its store).
void launch_hankel_svt_level2(const SvtParams& prm, int total, cudaStream_t stream);
// The whole subspace pipeline: level 1, level 2 (warm from fam[f].Vs2 when
// set), and for d <= 128 the full solver for level-2 overflow (cold).
// Returns the number of launches; 0 = the subspace solver does not apply to
// this geometry (nothing launched).  Matrices with d > 128 that overflow
// level 2 keep kLevelOverflow in their flag for the host to report.
int launch_hankel_svt_levels(const SvtParams& sp, int total, cudaStream_t stream, int kb1);

// One-thread-per-matrix Hankel-SVT for tiny plain lifts (small_svt.cu): the
// parameter-imaging echo term (5 x 32 at config 4).  Plain / plain-ADMM
// modes, one family, P <= kSmallSvtMaxP rows, P <= J q, len * J <=
// kSmallSvtMaxLJ, no singular-value output.  Its duals are stored
// structure-of-arrays: element (i, c) of matrix m at D[(i * J q + c) * count + m].
constexpr int kSmallSvtMaxP = 8;
constexpr int kSmallSvtMaxLJ = 64;
bool small_svt_applicable(const SvtParams& prm);
bool launch_small_svt(const SvtParams& prm, cudaStream_t stream);
// One-warp-per-matrix Hankel-SVT for plain lifts with d <= 32 (tiny_svt.cu):
// the config-5 single-coil points.  Plain mode, one family, J * len <= 1024,
// no singular-value output.
bool tiny_svt_applicable(const SvtParams& prm);
bool launch_tiny_svt(const SvtParams& prm, cudaStream_t stream);

// Hankel lift index map of a p x (blocks q) weighted lift as the kernels
// build it (operators.cpp:36-56, hankel.cpp:31-41,99-113): the lift stage of
// path 0 (full solver), 1 (subspace solver) or 2 (large-d variants) run on
// index-encoded spectra, decoded to (coil, source index, conj) per element,
// row-major (map_host: 3 p blocks q int32).
void lift_index_map_device(int n, int p, int coils, int vc, int path, int32_t* map_host);

size_t svt_smem_bytes(int DP, int R, int maxB, int maxLen, bool wl_smem = true);
int svt_padded_dim(int d);
void launch_hankel_svt(const SvtParams& prm, int total_matrices, cudaStream_t stream);

}  // namespace shlr_b200
