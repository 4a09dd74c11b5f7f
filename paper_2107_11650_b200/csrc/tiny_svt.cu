// Hankel-SVT for plain lifts with d = min(m, n) <= 32: one WARP per lifted
// matrix (config-5 points with one coil: 122x7 ... 482x31).
//
// The CTA-per-matrix full solver (hankel_svt.cu) runs these at 4 d threads
// per CTA with a CTA barrier per Jacobi round -- a 242x15 matrix took ~540 k
// cycles of latency.  Here each warp owns one matrix and synchronises with
// __syncwarp only:
//   * the coil vectors (Nc x N complex64) are staged in the warp's slice of
//     shared memory; the lift is addressed on the fly, Ahat[i][u] =
//     v_b[i + t] with (b, t) = divmod(u, q) for tall A (Ahat = A) and the
//     conjugate of the transposed element for wide A (lift_plain,
//     operators.cpp:93-103);
//   * G = Ahat^H Ahat (d x d) in FP32, each lane a fixed set of entries;
//   * cyclic parallel Jacobi on G in shared memory (round-robin pairing, d/2
//     rotations per round, the p/q rows then the p/q columns updated by the
//     whole warp), V accumulated alongside, until a sweep rotates nothing
//     (|g_pq| <= 1e-7 sqrt(g_pp g_qq)) or 20 sweeps;
//   * W = V diag((1 - tau/sigma)_+) V^H, Z = Ahat W row by row, and the
//     anti-diagonal adjoint sums accumulated per coil in shared memory
//     (adjoint_lift_plain, operators.cpp:105-119) -- deterministic (fixed
//     order, no atomics).
#include "hankel_svt.cuh"

namespace shlr_b200 {

namespace {

constexpr int kTinyWarps = 4;   // matrices per CTA
constexpr int kTinyMaxD = 32;
constexpr int kTinyMaxLJ = 1024;  // staged vector elements per matrix
constexpr int kTinyStride = kTinyMaxD + 1;

// shared-memory float2 per warp: vectors and accumulators (2 J len), G and V
__host__ __device__ __forceinline__ int tiny_warp_floats(int LJ, int d) { return 2 * LJ + 2 * d * kTinyStride; }

// element (i, u) of Ahat from the staged vectors vs[b * len + n]
__device__ __forceinline__ float2 tiny_elem(const float2* vs, int len, int q, bool wide, int i, int u) {
  if (!wide) {
    const int b = u / q, t = u - b * q;
    return vs[b * len + i + t];
  }
  const int b = i / q, t = i - b * q;
  return cconj(vs[b * len + u + t]);
}

__global__ void __launch_bounds__(32 * kTinyWarps) tiny_svt_kernel(const SvtParams prm) {
  const SvtFamily& F = prm.fam[0];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mat = blockIdx.x * kTinyWarps + warp;
  if (prm.skip && *prm.skip) return;
  if (mat >= F.count) return;
  const int d = F.d, e = F.e, len = F.len, J = F.J, q = F.q;
  const bool wide = F.wide;
  extern __shared__ __align__(16) float2 sm_tiny[];
  const int LJ = J * len;
  float2* base = sm_tiny + (size_t)warp * tiny_warp_floats(LJ, d);
  float2* vs = base;                     // J x len staged vectors
  float2* acc = vs + LJ;                 // J x len adjoint accumulators
  float2* G = acc + LJ;                  // d x d (stride kTinyStride): Gram, then W
  float2* V = G + d * kTinyStride;       // d x d eigenvectors (column k = vector k)

  const float2* sp = F.spec + (long long)mat * F.s_mat;
  for (int t = lane; t < LJ; t += 32) {
    const int j = t / len, n = t - j * len;
    vs[t] = __ldg(sp + (long long)n * F.s_n + (long long)j * F.s_j);
    acc[t] = make_float2(0.f, 0.f);
  }
  __syncwarp();

  // ---- G = Ahat^H Ahat: lane owns entries (a, b) = (lane / d + s, lane % d) strided
  for (int ab = lane; ab < d * d; ab += 32) {
    const int a = ab / d, b = ab - a * d;
    if (b < a) continue;
    float2 g = make_float2(0.f, 0.f);
    for (int i = 0; i < e; ++i) cfmac(g, tiny_elem(vs, len, q, wide, i, a), tiny_elem(vs, len, q, wide, i, b));
    G[a * kTinyStride + b] = g;                       // sum conj(A[i][a]) A[i][b]
    G[b * kTinyStride + a] = cconj(g);
  }
  for (int ab = lane; ab < d * d; ab += 32) {
    const int a = ab / d, b = ab - a * d;
    V[a * kTinyStride + b] = make_float2(a == b ? 1.f : 0.f, 0.f);
  }
  __syncwarp();
  for (int a = lane; a < d; a += 32) G[a * kTinyStride + a].y = 0.f;
  __syncwarp();

  // ---- cyclic parallel Jacobi (round robin over an even count m >= d)
  const int m = d + (d & 1);
  const int half = m / 2;
  int sweeps = 0;
  for (; sweeps < 20; ++sweeps) {
    unsigned any = 0;
    for (int r = 0; r < m - 1; ++r) {
      // pair k of round r: (x, y) from the circle method with player m-1 fixed
      // lane k < half computes the rotation of its pair
      int p = -1, qq = -1;
      float c = 1.f;
      float2 sw = make_float2(0.f, 0.f);  // s * phase
      if (lane < half) {
        const int x = lane == 0 ? m - 1 : (r + lane) % (m - 1);
        const int y = (r + m - 1 - lane) % (m - 1);
        p = min(x, y);
        qq = max(x, y);
        if (qq < d) {
          const float app = G[p * kTinyStride + p].x, aqq = G[qq * kTinyStride + qq].x;
          const float2 apq = G[p * kTinyStride + qq];
          const float mag = sqrtf(apq.x * apq.x + apq.y * apq.y);
          if (mag > 1e-7f * sqrtf(fabsf(app * aqq)) && mag > 1e-30f) {
            // rotation annihilating the Hermitian 2x2 [[app, apq], [conj(apq), aqq]]
            const float theta = 0.5f * atan2f(2.f * mag, aqq - app);
            float sn;
            __sincosf(theta, &sn, &c);
            const float2 ph = make_float2(apq.x / mag, apq.y / mag);
            sw = make_float2(sn * ph.x, sn * ph.y);
            any = 1;
          } else {
            qq = -1;
          }
        } else {
          qq = -1;
        }
      }
      __syncwarp();
      // rows p, q of G: G' = R^H G R with R = [[c, s ph], [-s conj(ph), c]] on (p, q)
      // apply to columns (right multiply) then rows (left multiply), and V <- V R
      for (int k = 0; k < half; ++k) {
        const int pk = __shfl_sync(0xffffffffu, p, k), qk = __shfl_sync(0xffffffffu, qq, k);
        const float ck = __shfl_sync(0xffffffffu, c, k);
        const float2 sk = make_float2(__shfl_sync(0xffffffffu, sw.x, k), __shfl_sync(0xffffffffu, sw.y, k));
        if (qk < 0) continue;
        // columns p, q of G and V: row index i = lane
        for (int i = lane; i < d; i += 32) {
          const float2 gp = G[i * kTinyStride + pk], gq = G[i * kTinyStride + qk];
          // [gp', gq'] = [gp, gq] R : gp' = c gp - conj(s) gq ; gq' = s gp + c gq
          G[i * kTinyStride + pk] = csub(cscale(gp, ck), cmulc(sk, gq));
          G[i * kTinyStride + qk] = cadd(cmul(sk, gp), cscale(gq, ck));
          const float2 vp = V[i * kTinyStride + pk], vq = V[i * kTinyStride + qk];
          V[i * kTinyStride + pk] = csub(cscale(vp, ck), cmulc(sk, vq));
          V[i * kTinyStride + qk] = cadd(cmul(sk, vp), cscale(vq, ck));
        }
      }
      __syncwarp();
      for (int k = 0; k < half; ++k) {
        const int pk = __shfl_sync(0xffffffffu, p, k), qk = __shfl_sync(0xffffffffu, qq, k);
        const float ck = __shfl_sync(0xffffffffu, c, k);
        const float2 sk = make_float2(__shfl_sync(0xffffffffu, sw.x, k), __shfl_sync(0xffffffffu, sw.y, k));
        if (qk < 0) continue;
        // rows p, q: [rp'; rq'] = R^H [rp; rq] : rp' = c rp - s rq ; rq' = conj(s) rp + c rq
        for (int j = lane; j < d; j += 32) {
          const float2 rp = G[pk * kTinyStride + j], rq = G[qk * kTinyStride + j];
          G[pk * kTinyStride + j] = csub(cscale(rp, ck), cmul(sk, rq));
          G[qk * kTinyStride + j] = cadd(cmulc(sk, rp), cscale(rq, ck));
        }
      }
      __syncwarp();
      // clean the annihilated pairs and keep the diagonal real
      if (lane < half && qq >= 0) {
        G[p * kTinyStride + qq] = make_float2(0.f, 0.f);
        G[qq * kTinyStride + p] = make_float2(0.f, 0.f);
        G[p * kTinyStride + p].y = 0.f;
        G[qq * kTinyStride + qq].y = 0.f;
      }
      __syncwarp();
    }
    if (!__any_sync(0xffffffffu, any)) break;
  }
  if (prm.sweeps_out && lane == 0) prm.sweeps_out[mat] = sweeps;

  // ---- shrink factors, W = V f V^H into G
  float fk = 0.f;
  if (lane < d) {
    const float lam = G[lane * kTinyStride + lane].x;
    const float sig = sqrtf(fmaxf(lam, 0.f));
    fk = sig > prm.thresh ? 1.f - prm.thresh / sig : 0.f;
  }
  __syncwarp();
  for (int ab = lane; ab < d * d; ab += 32) {
    const int a = ab / d, b = ab - a * d;
    float2 w = make_float2(0.f, 0.f);
    for (int k = 0; k < d; ++k) {
      const float f = __shfl_sync(0xffffffffu, fk, k);  // (uniform loop: every lane reaches it)
      if (f != 0.f) cfmac(w, V[b * kTinyStride + k], cscale(V[a * kTinyStride + k], f));  // V[a][k] f conj(V[b][k])
    }
    G[a * kTinyStride + b] = w;
  }
  __syncwarp();

  // ---- Z = Ahat W row by row; adjoint: lane u adds Z[i][u] into its (block, index) slot
  for (int i = 0; i < e; ++i) {
    if (lane < d) {
      float2 z = make_float2(0.f, 0.f);
      for (int w = 0; w < d; ++w) cfma(z, tiny_elem(vs, len, q, wide, i, w), G[w * kTinyStride + lane]);
      // element (i, u = lane) of Ahat -> A index: tall (row i, col u), wide (row u, col i) conj
      int b, t, row;
      if (!wide) {
        b = lane / q;
        t = lane - b * q;
        row = i;
      } else {
        b = i / q;
        t = i - b * q;
        row = lane;
        z = cconj(z);
      }
      float2* a = acc + b * len + row + t;
      *a = cadd(*a, z);
    }
    __syncwarp();
  }
  float2* op = F.out + (long long)mat * F.o_mat;
  for (int t = lane; t < LJ; t += 32) {
    const int j = t / len, n = t - j * len;
    op[(long long)n * F.o_n + (long long)j * F.o_j] = acc[t];
  }
}

}  // namespace

bool tiny_svt_applicable(const SvtParams& prm) {
  if (prm.nfam != 1 || prm.mode != SVT_PLAIN) return false;
  const SvtFamily& F = prm.fam[0];
  return F.d >= 1 && F.d <= kTinyMaxD && F.J * F.len <= kTinyMaxLJ && !F.vc && !F.sv && !F.halt;
}

bool launch_tiny_svt(const SvtParams& prm, cudaStream_t stream) {
  if (!tiny_svt_applicable(prm)) return false;
  const SvtFamily& F = prm.fam[0];
  if (F.count <= 0) return true;
  const size_t smem = sizeof(float2) * (size_t)kTinyWarps * tiny_warp_floats(F.J * F.len, F.d);
  static bool configured = false;
  if (!configured) {
    SHLR_CUDA(cudaFuncSetAttribute(tiny_svt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(float2) * kTinyWarps * tiny_warp_floats(kTinyMaxLJ, kTinyMaxD))));
    configured = true;
  }
  tiny_svt_kernel<<<(F.count + kTinyWarps - 1) / kTinyWarps, 32 * kTinyWarps, smem, stream>>>(prm);
  SHLR_LAUNCH_CHECK();
  return true;
}

}  // namespace shlr_b200
