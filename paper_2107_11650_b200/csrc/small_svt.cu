// Hankel-SVT for tiny plain lifts: one THREAD per lifted matrix.
//
// The echo-direction term of the parameter-imaging ADMM lifts, for every
// (FE slice, PE row), the J coil vectors of L echoes with pencil P
// (lift_plain, proj/src/operators.cpp:93-103) -- at BASELINE config 4 a
// 5 x 32 matrix, 65 536 of them per outer iteration -- and applies
// svt (solvers.cpp:11-21), the dual update and adjoint_lift_plain
// (solvers.cpp:264-268,279-283).  A CTA per matrix (the general kernels)
// leaves those SMs idle; here every thread owns one matrix:
//   * the J*L source samples and the J*L adjoint accumulators live in shared
//     memory, interleaved across the CTA's threads (conflict-free);
//   * G = A A^H (P x P, A = L + D/beta) and its cyclic complex Jacobi
//     eigen-decomposition stay in registers (P is a template parameter, all
//     loops unrolled);
//   * W = V diag((1 - tau/sigma)_+) V^H, then a second sweep over the columns
//     forms Z = W A, the dual update D += tau_d (L - Z), T = Z - D/beta and
//     the anti-diagonal adjoint sums;
//   * the duals are stored structure-of-arrays (element-major, matrix
//     fastest), so each of a warp's D accesses is one coalesced 256-byte
//     transaction.
// No barriers, no atomics: bitwise deterministic.
#include "hankel_svt.cuh"

namespace shlr_b200 {

namespace {

constexpr int kSmallNT = 128;

template <int P>
__global__ void __launch_bounds__(kSmallNT) small_svt_kernel(const SvtParams prm) {
  const SvtFamily& F = prm.fam[0];
  const int tid = threadIdx.x;
  const int mat = blockIdx.x * kSmallNT + tid;
  if (prm.skip && *prm.skip) return;
  if (mat >= F.count) return;
  if (F.halt && F.halt[mat / F.halt_div]) return;
  const bool admm = prm.mode != SVT_PLAIN;
  const int J = F.J, Lq = F.q, len = F.len, n = J * Lq;
  const long long cnt = F.count;
  extern __shared__ float2 sm_small[];
  float2* xs = sm_small;                       // [len * J][NT]
  float2* os = sm_small + (size_t)len * J * kSmallNT;  // [len * J][NT]
  const float2* sp = F.spec + (long long)mat * F.s_mat;
  for (int l = 0; l < len; ++l)
    for (int j = 0; j < J; ++j) {
      xs[(l * J + j) * kSmallNT + tid] = __ldg(sp + (long long)l * F.s_n + (long long)j * F.s_j);
      os[(l * J + j) * kSmallNT + tid] = make_float2(0.f, 0.f);
    }
  const float ib = prm.inv_beta;
  float2* Dm = admm ? F.D + mat : nullptr;  // element e of this matrix at Dm[e * cnt]

  // ---- G = A A^H with A[i][c] = x_j[i + t] + D[i][c] / beta, c = j * Lq + t
  float2 G[P][P];
#pragma unroll
  for (int a = 0; a < P; ++a)
#pragma unroll
    for (int b = 0; b < P; ++b) G[a][b] = make_float2(0.f, 0.f);
  for (int c = 0; c < n; ++c) {
    const int j = c / Lq, t = c - j * Lq;
    float2 col[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      float2 v = xs[((i + t) * J + j) * kSmallNT + tid];
      if (admm) {
        const float2 dd = __ldcg(Dm + (long long)(i * n + c) * cnt);
        v.x = fmaf(dd.x, ib, v.x);
        v.y = fmaf(dd.y, ib, v.y);
      }
      col[i] = v;
    }
#pragma unroll
    for (int a = 0; a < P; ++a)
#pragma unroll
      for (int b = a; b < P; ++b) cfmac(G[a][b], col[b], col[a]);  // col[a] conj(col[b])
  }
#pragma unroll
  for (int a = 0; a < P; ++a) {
    G[a][a].y = 0.f;
#pragma unroll
    for (int b = a + 1; b < P; ++b) G[b][a] = cconj(G[a][b]);
  }

  // ---- cyclic complex Jacobi: G <- J^H G J, V <- V J
  float2 V[P][P];
#pragma unroll
  for (int a = 0; a < P; ++a)
#pragma unroll
    for (int b = 0; b < P; ++b) V[a][b] = make_float2(a == b ? 1.f : 0.f, 0.f);
  // pairs inside the below-threshold tail (shrink factor 0 either way) and
  // off-diagonals at the FP32 noise floor of the trace are not rotated
  float tr = 0.f;
#pragma unroll
  for (int a = 0; a < P; ++a) tr += fabsf(G[a][a].x);
  const float tail = 0.25f * prm.thresh * prm.thresh, floor_abs = 1e-9f * tr;
  for (int sweep = 0; sweep < 12; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < P - 1; ++p)
#pragma unroll
      for (int q = p + 1; q < P; ++q) {
        const float2 g = G[p][q];
        const float ag = hypotf(g.x, g.y);
        const float al = G[p][p].x, be = G[q][q].x;
        if (!(ag > 1e-7f * sqrtf(fabsf(al * be)) && ag > floor_abs && ag > 1e-30f)) continue;
        // both eigenvalues of the 2 x 2 block below the tail: no rotation
        if (0.5f * (al + be) + sqrtf(0.25f * (al - be) * (al - be) + ag * ag) < tail) continue;
        rotated = true;
        const float2 u = make_float2(g.x / ag, g.y / ag);
        const float z = (be - al) / (2.f * ag);
        const float tt = (z >= 0.f ? 1.f : -1.f) / (fabsf(z) + sqrtf(1.f + z * z));
        const float c = rsqrtf(1.f + tt * tt), s = tt * c;
        const float2 su = cscale(u, s), suc = cscale(cconj(u), s);  // s u, s conj(u)
#pragma unroll
        for (int k = 0; k < P; ++k) {
          if (k == p || k == q) continue;
          const float2 gp = G[k][p], gq = G[k][q];
          const float2 np_ = csub(cscale(gp, c), cmul(suc, gq));
          const float2 nq = cadd(cmul(su, gp), cscale(gq, c));
          G[k][p] = np_;
          G[k][q] = nq;
          G[p][k] = cconj(np_);
          G[q][k] = cconj(nq);
        }
        G[p][p] = make_float2(al - tt * ag, 0.f);
        G[q][q] = make_float2(be + tt * ag, 0.f);
        G[p][q] = G[q][p] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const float2 vp = V[k][p], vq = V[k][q];
          V[k][p] = csub(cscale(vp, c), cmul(suc, vq));
          V[k][q] = cadd(cmul(su, vp), cscale(vq, c));
        }
      }
    if (!rotated) break;
  }

  // ---- W = V diag(f) V^H, f = (1 - tau / sigma)_+
  float f[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const float lam = G[k][k].x;
    f[k] = (lam > prm.thresh * prm.thresh && lam > 0.f) ? 1.f - prm.thresh * rsqrtf(lam) : 0.f;
  }
  float2 W[P][P];
#pragma unroll
  for (int a = 0; a < P; ++a)
#pragma unroll
    for (int b = 0; b < P; ++b) {
      float2 w = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < P; ++k) cfmac(w, V[b][k], cscale(V[a][k], f[k]));  // V[a][k] f_k conj(V[b][k])
      W[a][b] = w;
    }

  // ---- Z = W A per column, duals, T = Z - D/beta (or Z), adjoint sums
  for (int c = 0; c < n; ++c) {
    const int j = c / Lq, t = c - j * Lq;
    float2 lv[P], av[P], dv[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      lv[i] = xs[((i + t) * J + j) * kSmallNT + tid];
      av[i] = lv[i];
      if (admm) {
        dv[i] = __ldcg(Dm + (long long)(i * n + c) * cnt);
        av[i].x = fmaf(dv[i].x, ib, av[i].x);
        av[i].y = fmaf(dv[i].y, ib, av[i].y);
      }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
      float2 z = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < P; ++k) cfma(z, W[i][k], av[k]);
      float2 tv = z;
      if (admm) {
        float2 dn = dv[i];
        dn.x = fmaf(prm.tau_dual, lv[i].x - z.x, dn.x);
        dn.y = fmaf(prm.tau_dual, lv[i].y - z.y, dn.y);
        Dm[(long long)(i * n + c) * cnt] = dn;
        tv.x = fmaf(-dn.x, ib, z.x);
        tv.y = fmaf(-dn.y, ib, z.y);
      }
      float2* o = os + ((i + t) * J + j) * kSmallNT + tid;
      *o = cadd(*o, tv);
    }
  }
  float2* op = F.out + (long long)mat * F.o_mat;
  for (int l = 0; l < len; ++l)
    for (int j = 0; j < J; ++j) op[(long long)l * F.o_n + (long long)j * F.o_j] = os[(l * J + j) * kSmallNT + tid];
}

template <int P>
void launch_small(const SvtParams& prm, cudaStream_t stream) {
  const SvtFamily& F = prm.fam[0];
  const size_t smem = 2ull * F.len * F.J * kSmallNT * sizeof(float2);
  static bool configured = false;
  if (!configured) {
    SHLR_CUDA(cudaFuncSetAttribute(small_svt_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   227 * 1024));
    configured = true;
  }
  small_svt_kernel<P><<<(F.count + kSmallNT - 1) / kSmallNT, kSmallNT, smem, stream>>>(prm);
  SHLR_LAUNCH_CHECK();
}

}  // namespace

bool small_svt_applicable(const SvtParams& prm) {
  if (prm.nfam != 1 || prm.mode == SVT_ADMM_WEIGHTED) return false;
  const SvtFamily& F = prm.fam[0];
  return F.vc == 0 && F.sv == nullptr && F.P >= 1 && F.P <= kSmallSvtMaxP && F.P <= F.J * F.q &&
         F.len * F.J <= kSmallSvtMaxLJ && F.B == F.J;
}

bool launch_small_svt(const SvtParams& prm, cudaStream_t stream) {
  if (!small_svt_applicable(prm)) return false;
  if (prm.fam[0].count <= 0) return true;
  switch (prm.fam[0].P) {
    case 1: launch_small<1>(prm, stream); return true;
    case 2: launch_small<2>(prm, stream); return true;
    case 3: launch_small<3>(prm, stream); return true;
    case 4: launch_small<4>(prm, stream); return true;
    case 5: launch_small<5>(prm, stream); return true;
    case 6: launch_small<6>(prm, stream); return true;
    case 7: launch_small<7>(prm, stream); return true;
    case 8: launch_small<8>(prm, stream); return true;
  }
  return false;
}

}  // namespace shlr_b200
