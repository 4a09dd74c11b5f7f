// Fused batched Hankel-SVT kernel (see hankel_svt.cuh for the algorithm).
#include "hankel_svt.cuh"

namespace shlr_b200 {

namespace {

constexpr float kTolRel = 3.0e-7f;   // rotate iff |g_ab| > kTolRel sqrt(g_aa g_bb)
constexpr float kTolAbs = 1.0e-7f;   //        and |g_ab| > kTolAbs max_u g_uu

struct __align__(16) RotParam {
  float c, sn;       // cos, sin
  float2 cw, sw;     // c * conj(phase), s * conj(phase)
  float na, nb;      // new diagonal entries
  int flag;          // 1 = non-identity rotation
  int pad;
};

// Ring (round-robin / circle method) pairing at round r for DP indices.
// Position k < DP-1 on the ring holds storage index (k - r) mod (DP-1);
// top[0] is fixed at DP-1.  top[s] = ring position s-1 (s >= 1),
// bot[s] = ring position DP-2-s.
__device__ __forceinline__ int ring_idx(int k, int r, int DP) {
  int v = k - r;
  v %= (DP - 1);
  return v < 0 ? v + DP - 1 : v;
}
__device__ __forceinline__ int top_of(int s, int r, int DP) {
  return s == 0 ? DP - 1 : ring_idx(s - 1, r, DP);
}
__device__ __forceinline__ int bot_of(int s, int r, int DP) { return ring_idx(DP - 2 - s, r, DP); }

template <int DP>
__device__ __forceinline__ float2 gget(const float2* G, int x, int y) {
  return x <= y ? G[x * (DP + 1) + y] : cconj(G[y * (DP + 1) + x]);
}
template <int DP>
__device__ __forceinline__ void gput(float2* G, int x, int y, float2 v) {
  if (x <= y)
    G[x * (DP + 1) + y] = v;
  else
    G[y * (DP + 1) + x] = cconj(v);
}

__device__ __forceinline__ const SvtFamily& family_of(const SvtParams& p, int blk, int& local) {
  if (p.nfam > 1 && blk >= p.fam[0].count) {
    local = blk - p.fam[0].count;
    return p.fam[1];
  }
  local = blk;
  return p.fam[0];
}

// Lifted element L at (row i of Ahat, storage column u) from staged weighted
// spectra wl[b * len + n].
__device__ __forceinline__ float2 lift_elem(const float2* wl, const SvtFamily& F, int i, int u) {
  if (!F.wide) {
    const int b = u / F.q, t = u - b * F.q;
    return wl[b * F.len + i + t];
  } else {
    const int b = i / F.q, t = i - b * F.q;
    return cconj(wl[b * F.len + u + t]);
  }
}

}  // namespace

template <int DP, int R>
__global__ void __launch_bounds__(4 * DP, 1) hankel_svt_kernel(const SvtParams prm) {
  constexpr int NT = 4 * DP;
  constexpr int S = DP / 2;         // slots
  constexpr int W = DP / 8;         // slots per V thread (4 groups)
  constexpr int HALF = DP / 2;      // GEMM column pairs
  constexpr int GS = DP + 1;        // G / W row stride
  static_assert(DP % 8 == 0 && DP >= 8 && DP <= 128, "DP must be a multiple of 8 in [8,128]");
  static_assert(R % 8 == 0, "R must be a multiple of 8");

  if (prm.skip && *prm.skip) return;
  int mat;
  const SvtFamily& F = family_of(prm, blockIdx.x, mat);
  const int tid = threadIdx.x;
  const int d = F.d, e = F.e, len = F.len, B = F.B, J = F.J;
  const bool admm = prm.mode != SVT_PLAIN;
  const bool weighted = prm.mode == SVT_ADMM_WEIGHTED;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* Gs = reinterpret_cast<float2*>(smem_raw);            // DP x GS
  float2* wl = Gs + DP * GS;                                   // B x len
  float2* acc = wl + B * len;                                  // B x len
  float2* Abuf = acc + B * len;                                // R x DP
  float2* Dbuf = Abuf + R * DP;                                // R x DP
  RotParam* prmS = reinterpret_cast<RotParam*>(Dbuf + R * DP); // S
  float* fbuf = reinterpret_cast<float*>(prmS + S);            // DP
  int* flags = reinterpret_cast<int*>(fbuf + DP);              // 4
  float* scal = reinterpret_cast<float*>(flags + 4);           // 4

  float2* Dg = admm ? F.D + (long long)mat * e * d : nullptr;

  // ---------------------------------------------------------- phase 0
  {
    const float2* sp = F.spec + (long long)mat * F.s_mat;
    for (int t = tid; t < J * len; t += NT) {
      const int j = t / len, n = t - j * len;
      float2 s = sp[n * F.s_n + j * F.s_j];
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
    if (tid < 4) flags[tid] = 0;
  }
  __syncthreads();

  // GEMM tile coordinates
  const int lp = tid % HALF;          // column pair -> columns 2lp, 2lp+1
  const int kq = tid / HALF;          // 0..7
  const int l0 = 2 * lp;

  // ---------------------------------------------------------- phase 1: Gram
  {
    float2 g0[W], g1[W];
#pragma unroll
    for (int m = 0; m < W; ++m) g0[m] = g1[m] = make_float2(0.f, 0.f);
    for (int i0 = 0; i0 < e; i0 += R) {
      const int rows = min(R, e - i0);
      for (int t = tid; t < R * DP; t += NT) {
        const int r = t / DP, u = t - r * DP;
        float2 v = make_float2(0.f, 0.f);
        if (r < rows && u < d) {
          v = lift_elem(wl, F, i0 + r, u);
          if (admm) {
            const float2 dd = Dg[(long long)(i0 + r) * d + u];
            v.x = fmaf(dd.x, prm.inv_beta, v.x);
            v.y = fmaf(dd.y, prm.inv_beta, v.y);
          }
        }
        Abuf[t] = v;
      }
      __syncthreads();
      for (int r = 0; r < rows; ++r) {
        const float2* row = Abuf + r * DP;
        const float2 b0 = row[l0], b1 = row[l0 + 1];
#pragma unroll
        for (int m = 0; m < W; ++m) {
          const float2 a = row[kq + 8 * m];
          cfmac(g0[m], a, b0);
          cfmac(g1[m], a, b1);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int m = 0; m < W; ++m) {
      const int k = kq + 8 * m;
      Gs[k * GS + l0] = g0[m];
      Gs[k * GS + l0 + 1] = g1[m];
    }
  }
  __syncthreads();

  // ---------------------------------------------------------- phase 2: Jacobi
  const int vrow = tid >> 2, vg = tid & 3;
  float2 vt[W], vb[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int s = vg * W + w;
    const int t0 = s == 0 ? DP - 1 : s - 1;
    const int b0 = DP - 2 - s;
    vt[w] = make_float2(vrow == t0 ? 1.f : 0.f, 0.f);
    vb[w] = make_float2(vrow == b0 ? 1.f : 0.f, 0.f);
  }
  if (tid < 32) {
    float mx = 0.f;
    for (int u = tid; u < DP; u += 32) mx = fmaxf(mx, Gs[u * GS + u].x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (tid == 0) scal[0] = kTolAbs * mx;
  }
  __syncthreads();
  const float tol_abs = scal[0];
  constexpr int NBLK = S * (S + 1) / 2;

  for (int sweep = 0; sweep < prm.max_sweeps; ++sweep) {
    int* rot_flag = &flags[sweep & 1];
    for (int r = 0; r < DP - 1; ++r) {
      if (tid < S) {
        const int s = tid;
        const int a = top_of(s, r, DP), b = bot_of(s, r, DP);
        const float al = Gs[a * GS + a].x, be = Gs[b * GS + b].x;
        const float2 gm = gget<DP>(Gs, a, b);
        const float g = hypotf(gm.x, gm.y);
        RotParam rp;
        rp.flag = 0;
        if (g > 0.f && g > tol_abs && g > kTolRel * sqrtf(fmaxf(al * be, 0.f))) {
          const float zeta = (be - al) / (2.f * g);
          const float az = fabsf(zeta);
          float t = (az > 1e18f) ? 0.5f / az : 1.f / (az + sqrtf(1.f + az * az));
          t = zeta < 0.f ? -t : t;
          const float c = rsqrtf(1.f + t * t);
          const float sn = c * t;
          const float2 ph = make_float2(gm.x / g, -gm.y / g);  // conj(g)/|g|
          rp.c = c;
          rp.sn = sn;
          rp.cw = cscale(ph, c);
          rp.sw = cscale(ph, sn);
          rp.na = al - t * g;
          rp.nb = be + t * g;
          rp.flag = 1;
          *rot_flag = 1;
        }
        prmS[s] = rp;
      }
      __syncthreads();
      // G <- J^H G J on slot-pair blocks (s1 <= s2)
      for (int blk = tid; blk < NBLK; blk += NT) {
        // triangular decode: row s1 holds S - s1 entries
        int s1 = (int)((2.f * S + 1.f - sqrtf((2.f * S + 1.f) * (2.f * S + 1.f) - 8.f * blk)) * 0.5f);
        int base = s1 * S - (s1 * (s1 - 1)) / 2;
        while (s1 > 0 && base > blk) { --s1; base = s1 * S - (s1 * (s1 - 1)) / 2; }
        while (blk >= base + (S - s1)) { base += S - s1; ++s1; }
        const int s2 = s1 + (blk - base);
        const RotParam& p1 = prmS[s1];
        const RotParam& p2 = prmS[s2];
        if (!p1.flag && !p2.flag) continue;
        const int x0 = top_of(s1, r, DP), x1 = bot_of(s1, r, DP);
        if (s1 == s2) {
          Gs[x0 * GS + x0] = make_float2(p1.na, 0.f);
          Gs[x1 * GS + x1] = make_float2(p1.nb, 0.f);
          gput<DP>(Gs, x0, x1, make_float2(0.f, 0.f));
          continue;
        }
        const int y0 = top_of(s2, r, DP), y1 = bot_of(s2, r, DP);
        float2 a00 = gget<DP>(Gs, x0, y0), a01 = gget<DP>(Gs, x0, y1);
        float2 a10 = gget<DP>(Gs, x1, y0), a11 = gget<DP>(Gs, x1, y1);
        if (p2.flag) {  // X J2 on columns
          const float2 n00 = csub(cscale(a00, p2.c), cmul(p2.sw, a01));
          const float2 n01 = cadd(cscale(a00, p2.sn), cmul(p2.cw, a01));
          const float2 n10 = csub(cscale(a10, p2.c), cmul(p2.sw, a11));
          const float2 n11 = cadd(cscale(a10, p2.sn), cmul(p2.cw, a11));
          a00 = n00; a01 = n01; a10 = n10; a11 = n11;
        }
        if (p1.flag) {  // J1^H X on rows
          const float2 n00 = csub(cscale(a00, p1.c), cmulc(p1.sw, a10));
          const float2 n10 = cadd(cscale(a00, p1.sn), cmulc(p1.cw, a10));
          const float2 n01 = csub(cscale(a01, p1.c), cmulc(p1.sw, a11));
          const float2 n11 = cadd(cscale(a01, p1.sn), cmulc(p1.cw, a11));
          a00 = n00; a01 = n01; a10 = n10; a11 = n11;
        }
        gput<DP>(Gs, x0, y0, a00);
        gput<DP>(Gs, x0, y1, a01);
        gput<DP>(Gs, x1, y0, a10);
        gput<DP>(Gs, x1, y1, a11);
      }
      // V <- V J on this thread's slots
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const RotParam& p = prmS[vg * W + w];
        if (p.flag) {
          const float2 a = vt[w], b = vb[w];
          vt[w] = csub(cscale(a, p.c), cmul(p.sw, b));
          vb[w] = cadd(cscale(a, p.sn), cmul(p.cw, b));
        }
      }
      __syncthreads();
      // ring shift of V columns: top moves right, bottom moves left
      {
        const float2 up_t = make_float2(__shfl_up_sync(0xffffffffu, vt[W - 1].x, 1, 4),
                                        __shfl_up_sync(0xffffffffu, vt[W - 1].y, 1, 4));
        const float2 up_b = make_float2(__shfl_up_sync(0xffffffffu, vb[0].x, 1, 4),
                                        __shfl_up_sync(0xffffffffu, vb[0].y, 1, 4));
        const float2 dn_b = make_float2(__shfl_down_sync(0xffffffffu, vb[0].x, 1, 4),
                                        __shfl_down_sync(0xffffffffu, vb[0].y, 1, 4));
        float2 nt[W], nb[W];
        if (W == 1) {
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
    __syncthreads();
    const int any = *rot_flag;
    if (tid == 0) flags[(sweep + 1) & 1] = 0;
    __syncthreads();
    if (prm.sweeps_out && tid == 0) prm.sweeps_out[blockIdx.x] = sweep + 1;
    if (!any) break;
  }

  // ---------------------------------------------------------- phase 3: f, W
  {
    for (int u = tid; u < DP; u += NT) {
      const float lam = Gs[u * GS + u].x;
      float f = 0.f;
      if (lam > prm.thresh * prm.thresh && lam > 0.f) f = 1.f - prm.thresh / sqrtf(lam);
      fbuf[u] = f;
    }
    __syncthreads();
    if (F.sv) {
      float* sv = F.sv + (long long)mat * d;
      for (int u = tid; u < d; u += NT) {
        const float su = sqrtf(fmaxf(Gs[u * GS + u].x, 0.f));
        int rank = 0;
        for (int v = 0; v < d; ++v) {
          const float s2 = sqrtf(fmaxf(Gs[v * GS + v].x, 0.f));
          rank += (s2 > su) || (s2 == su && v < u);
        }
        sv[rank] = su;
      }
    }
    __syncthreads();
    for (int t = tid; t < DP * GS; t += NT) Gs[t] = make_float2(0.f, 0.f);
    // panel staging area: DP x 2W in Abuf/Dbuf (R*DP*2 >= DP*2W)
    float2* panel = Abuf;
    constexpr int PW = 2 * W;
    for (int g = 0; g < 4; ++g) {
      __syncthreads();
      if (vg == g) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int s = g * W + w;
          const int ct = s == 0 ? DP - 1 : s - 1;
          const int cb = DP - 2 - s;
          panel[vrow * PW + 2 * w] = cscale(vt[w], sqrtf(fbuf[ct]));
          panel[vrow * PW + 2 * w + 1] = cscale(vb[w], sqrtf(fbuf[cb]));
        }
      }
      __syncthreads();
#pragma unroll 1
      for (int m = 0; m < W; ++m) {
        const int k = kq + 8 * m;
        const float2* pk = panel + k * PW;
        const float2* pl0 = panel + l0 * PW;
        const float2* pl1 = panel + (l0 + 1) * PW;
        float2 s0 = Gs[k * GS + l0], s1 = Gs[k * GS + l0 + 1];
#pragma unroll
        for (int mm = 0; mm < PW; ++mm) {
          const float2 a = pk[mm];
          // W[k][l] += U[k][m] conj(U[l][m])
          cfmac(s0, pl0[mm], a);
          cfmac(s1, pl1[mm], a);
        }
        Gs[k * GS + l0] = s0;
        Gs[k * GS + l0 + 1] = s1;
      }
    }
    __syncthreads();
  }

  // ---------------------------------------------------------- phase 4: Z, D, T, adjoint
  {
    constexpr int RM = R / 8;
    for (int i0 = 0; i0 < e; i0 += R) {
      const int rows = min(R, e - i0);
      for (int t = tid; t < R * DP; t += NT) {
        const int r = t / DP, u = t - r * DP;
        float2 v = make_float2(0.f, 0.f), dd = make_float2(0.f, 0.f);
        if (r < rows && u < d) {
          v = lift_elem(wl, F, i0 + r, u);
          if (admm) {
            dd = Dg[(long long)(i0 + r) * d + u];
            v.x = fmaf(dd.x, prm.inv_beta, v.x);
            v.y = fmaf(dd.y, prm.inv_beta, v.y);
          }
        }
        Abuf[t] = v;
        Dbuf[t] = dd;
      }
      __syncthreads();
      float2 z0[RM], z1[RM];
#pragma unroll
      for (int m = 0; m < RM; ++m) z0[m] = z1[m] = make_float2(0.f, 0.f);
      for (int k = 0; k < d; ++k) {
        const float2 w0 = Gs[k * GS + l0], w1 = Gs[k * GS + l0 + 1];
#pragma unroll
        for (int m = 0; m < RM; ++m) {
          const float2 a = Abuf[(kq + 8 * m) * DP + k];
          cfma(z0[m], a, w0);
          cfma(z1[m], a, w1);
        }
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < RM; ++m) {
        Abuf[(kq + 8 * m) * DP + l0] = z0[m];
        Abuf[(kq + 8 * m) * DP + l0 + 1] = z1[m];
      }
      __syncthreads();
      for (int t = tid; t < R * DP; t += NT) {
        const int r = t / DP, u = t - r * DP;
        if (r < rows && u < d) {
          const float2 z = Abuf[t];
          float2 tv = z;
          if (admm) {
            const float2 L = lift_elem(wl, F, i0 + r, u);
            float2 dn = Dbuf[t];
            dn.x = fmaf(prm.tau_dual, L.x - z.x, dn.x);
            dn.y = fmaf(prm.tau_dual, L.y - z.y, dn.y);
            Dg[(long long)(i0 + r) * d + u] = dn;
            tv.x = fmaf(-dn.x, prm.inv_beta, z.x);
            tv.y = fmaf(-dn.y, prm.inv_beta, z.y);
          }
          Dbuf[t] = tv;
        }
      }
      __syncthreads();
      // anti-diagonal sums (Hankel adjoint), fixed summation order
      for (int o = tid; o < B * len; o += NT) {
        const int b = o / len, n = o - b * len;
        float2 s = acc[o];
        if (!F.wide) {
          // T[i][b*q + t], i + t = n, i in chunk, 0 <= t < q
          const int ilo = max(i0, n - F.q + 1), ihi = min(i0 + rows - 1, n);
          for (int i = ilo; i <= ihi; ++i) s = cadd(s, Dbuf[(i - i0) * DP + b * F.q + (n - i)]);
        } else {
          // rows i = b*q + t of That, T[k][b*q+t] = conj(That[i][k]), k + t = n
          const int tlo = max(max(0, i0 - b * F.q), n - F.P + 1);
          const int thi = min(min(F.q - 1, i0 + rows - 1 - b * F.q), n);
          for (int t = tlo; t <= thi; ++t) {
            const int i = b * F.q + t;
            s = cadd(s, cconj(Dbuf[(i - i0) * DP + (n - t)]));
          }
        }
        acc[o] = s;
      }
      __syncthreads();
    }
  }

  // ---------------------------------------------------------- phase 5: weighting + store
  {
    float2* op = F.out + (long long)mat * F.o_mat;
    for (int t = tid; t < J * len; t += NT) {
      const int j = t / len, n = t - j * len;
      float2 v = acc[j * len + n];
      if (weighted) {
        v = cmulc(F.wc[n], v);  // conj(wc) * v
        if (F.vc) {
          const int fl = dagger_src(n, len);
          v = cadd(v, cmul(F.wc[fl], cconj(acc[(J + j) * len + fl])));
        }
      }
      op[n * F.o_n + j * F.o_j] = v;
    }
  }
}

size_t svt_smem_bytes(int DP, int R, int maxB, int maxLen) {
  const int S = DP / 2;
  return sizeof(float2) * ((size_t)DP * (DP + 1) + 2ull * maxB * maxLen + 2ull * R * DP) +
         sizeof(RotParam) * S + sizeof(float) * DP + 8 * sizeof(int) + 64;
}

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
  size_t s32 = svt_smem_bytes(DP, 32, maxB, maxLen);
  if (s32 <= lim) return launch_one<DP, 32>(prm, total, s32, stream);
  size_t s16 = svt_smem_bytes(DP, 16, maxB, maxLen);
  if (s16 <= lim) return launch_one<DP, 16>(prm, total, s16, stream);
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
  const int dp = ((dmax + 7) / 8) * 8;
  switch (dp) {
    case 8: return dispatch_r<8>(prm, total, maxB, maxLen, stream);
    case 16: return dispatch_r<16>(prm, total, maxB, maxLen, stream);
    case 24: return dispatch_r<24>(prm, total, maxB, maxLen, stream);
    case 32: return dispatch_r<32>(prm, total, maxB, maxLen, stream);
    case 40: case 48: return dispatch_r<48>(prm, total, maxB, maxLen, stream);
    case 56: case 64: return dispatch_r<64>(prm, total, maxB, maxLen, stream);
    case 72: return dispatch_r<72>(prm, total, maxB, maxLen, stream);
    case 80: case 88: case 96: return dispatch_r<96>(prm, total, maxB, maxLen, stream);
    case 104: return dispatch_r<104>(prm, total, maxB, maxLen, stream);
    case 112: case 120: return dispatch_r<120>(prm, total, maxB, maxLen, stream);
    case 128: return dispatch_r<128>(prm, total, maxB, maxLen, stream);
    default:
      throw Unsupported("hankel_svt: min(m, n) = " + std::to_string(dmax) +
                        " exceeds the single-CTA eigen-solver limit of 128 in this build");
  }
}

}  // namespace shlr_b200
