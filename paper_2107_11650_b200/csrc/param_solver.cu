// Parameter-imaging ADMM on the device (see param_solver.cuh).
//
// Per FE slice the reference solves (proj/src/solvers.cpp:193-298)
//   min_x  lambda/2 ||U F_PE x - y||^2
//          + sum_r ||P_r x||_*  (plain lift along echoes, threshold lambda2/beta)
//          + sum_l ||Q_l x||_*  (weighted lift along PE, threshold 1/beta)
// with ADMM.  Its X-update operator (apply_a, :235-255) is diagonal in
// (k_PE, echo, coil):
//   lambda U(k, l) + beta counts_par(l) + beta a_N(k)
// with a_N the weighted-lift normal diagonal (+ virtual-coil mirror), so the
// state is kept in PE k-space, X^ = F_PE x, and the capped warm-started CG
// of cg_solve (solvers.cpp:23-67) is replayed per slice by one CTA with the
// reference's iteration-count rule, real pairing, break and divergence
// tests.  All slices of recon_param_dataset (parammap.cpp:21-54) run in the
// same launches; each keeps its own CG scalars, stop flag and log.
//
// Layouts: k-space vectors [S][L][N][J] (so the PE lift of (slice, echo) is
// one contiguous N x J block); image-domain vectors [S][N][L][J] (so the echo
// lift of (slice, PE row) is one contiguous L x J block, and it is the
// output layout of recon_param_dataset).
#include "param_solver.cuh"
#include "solver_util.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

namespace shlr_b200 {

namespace {

using util::block_sum;
using util::block_sum_all;
using util::dalloc;
using util::dalloc_s;
using util::grid_for;
using util::kThreads;

constexpr int kCgThreads = 1024;

__global__ void k_p_from_double(const double* __restrict__ src, float2* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_float2((float)src[2 * i], (float)src[2 * i + 1]);
}

__global__ void k_p_to_double(const float2* __restrict__ src, double* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    dst[2 * i] = src[i].x;
    dst[2 * i + 1] = src[i].y;
  }
}

__global__ void k_p_copy(float2* __restrict__ dst, const float2* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_p_fill(float2* __restrict__ p, size_t n, float2 v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Hybrid data h [S][N][L][J] (FE image, PE k-space) -> masked k-space
// x0 [S][L][N][J] (= F_PE fid_rhs, solvers.cpp:225-226,233) and lambda * x0.
__global__ void k_p_prep(const float2* __restrict__ h, const uint8_t* __restrict__ mask, int S, int N,
                         int L, int J, float lambda, float2* __restrict__ x0, float2* __restrict__ yk) {
  const size_t nel = (size_t)S * L * N * J;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < nel;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % J);
    size_t t = idx / J;
    const int k = (int)(t % N);
    t /= N;
    const int l = (int)(t % L);
    const size_t s = t / L;
    const bool m = mask[(size_t)k * L + l] != 0;
    const float2 v = m ? h[((s * N + k) * L + l) * J + j] : make_float2(0.f, 0.f);
    x0[idx] = v;
    yk[idx] = make_float2(lambda * v.x, lambda * v.y);
  }
}

// First-iteration adjoints (Z = 0, D = 1): hpe[s][l][k][j] = hpe0[k],
// hecho[s][r][l][j] = hecho0[l].
__global__ void k_p_init_h(float2* __restrict__ hpe, float2* __restrict__ hecho,
                           const float2* __restrict__ hpe0, const float* __restrict__ hecho0, int S,
                           int N, int L, int J) {
  const size_t nel = (size_t)S * L * N * J;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < nel;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t t = idx / J;
    hpe[idx] = hpe0[t % N];
    hecho[idx] = make_float2(hecho0[t % L], 0.f);
  }
}

__global__ void k_p_reset(ParamSliceCtl* ctl, int* halt, int* have_v, int S) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    memset(&ctl[s], 0, sizeof(ParamSliceCtl));
    halt[s] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *have_v = 0;
}

// RHS (solvers.cpp:260-275) in PE k-space, one FFT along PE per slice:
// b^ = lambda y^ + beta (hpe + F_PE(hecho)).  Transform view: outer = slice,
// n = PE, inner = (echo, coil) of the image-domain hecho.
struct ParamRhsOp {
  const float2* hecho;
  const float2* hpe;
  const float2* yk;
  float2* bk;
  int N, L, J;
  float beta;
  const int* halt;
  __device__ bool skip() const { return false; }
  __device__ float2 load(int o, int k, int i) const {
    return hecho[((long long)o * N + k) * (L * J) + i];
  }
  __device__ void store(int o, int k, int i, float2 v) const {
    if (halt[o]) return;
    const int l = i / J, j = i - l * J;
    const long long idx = (((long long)o * L + l) * N + k) * J + j;
    const float2 h = hpe[idx], y = yk[idx];
    bk[idx] = make_float2(fmaf(beta, h.x + v.x, y.x), fmaf(beta, h.y + v.y, y.y));
  }
};

// x = iF_PE(X^): [S][L][N][J] k-space -> [S][N][L][J] image.
struct ParamToImageOp {
  const float2* x;
  float2* out;
  int N, L, J;
  const int* halt;   // nullable
  __device__ bool skip() const { return false; }
  __device__ float2 load(int o, int k, int i) const {
    const int l = i / J, j = i - l * J;
    return x[(((long long)o * L + l) * N + k) * J + j];
  }
  __device__ void store(int o, int k, int i, float2 v) const {
    if (halt && halt[o]) return;
    out[((long long)o * N + k) * (L * J) + i] = v;
  }
};

// Capped, warm-started CG of one slice (cg_solve, solvers.cpp:23-67) on the
// diagonal operator dg, one CTA per slice.  Vectors stay in HBM/L2 (each
// thread revisits its own elements, so they mostly hit L1); the two scalar
// reductions per iteration are deterministic FP64 block sums.
__global__ void __launch_bounds__(kCgThreads) k_p_cg(const float2* __restrict__ bk, const float* __restrict__ dg,
                                                     float2* __restrict__ x, float2* __restrict__ xold,
                                                     float2* __restrict__ r, float2* __restrict__ p, int nel_s,
                                                     int J, ParamSliceCtl* __restrict__ ctl,
                                                     int* __restrict__ halt, int cg_max, double cg_tol) {
  __shared__ double sh[33];
  const int s = blockIdx.x;
  if (halt[s]) return;
  const size_t base = (size_t)s * nel_s;
  const float2* b = bk + base;
  float2* xs = x + base;
  float2* xo = xold + base;
  float2* rs = r + base;
  float2* ps = p + base;
  double sb = 0.0, sr = 0.0;
  for (int i = threadIdx.x; i < nel_s; i += blockDim.x) {
    const float2 xv = xs[i], bv = b[i];
    const float dv = __ldg(dg + i / J);
    xo[i] = xv;
    const float2 rv = make_float2(fmaf(-dv, xv.x, bv.x), fmaf(-dv, xv.y, bv.y));
    rs[i] = rv;
    sb += (double)bv.x * bv.x + (double)bv.y * bv.y;
    sr += (double)rv.x * rv.x + (double)rv.y * rv.y;
  }
  const double b2 = block_sum_all(sb, sh);
  const double r2 = block_sum_all(sr, sh);
  const double bnorm = sqrt(b2);
  if (bnorm == 0.0) {  // solvers.cpp:30-33: zero right-hand side -> x = 0
    for (int i = threadIdx.x; i < nel_s; i += blockDim.x) xs[i] = make_float2(0.f, 0.f);
    if (threadIdx.x == 0) {
      ctl[s].cg_it = 0;
      ctl[s].cg_rel = 0.0;
    }
    return;
  }
  double rel = sqrt(r2) / bnorm;
  int err = 0;
  if (!isfinite(rel)) err = 1;  // solvers.cpp:35-36
  int it = 0;
  if (!err && rel > cg_tol) {
    double rho = r2;
    float g = 0.f;
    for (; it < cg_max; ++it) {
      double sd = 0.0;
      for (int i = threadIdx.x; i < nel_s; i += blockDim.x) {
        float2 pv = rs[i];
        if (it > 0) {
          const float2 po = ps[i];
          pv = make_float2(fmaf(g, po.x, pv.x), fmaf(g, po.y, pv.y));
        }
        ps[i] = pv;
        const float dv = __ldg(dg + i / J);
        const float2 ap = make_float2(dv * pv.x, dv * pv.y);
        sd += (double)pv.x * ap.x + (double)pv.y * ap.y;
      }
      const double denom = block_sum_all(sd, sh);
      if (!isfinite(denom) || denom <= 0.0) {  // solvers.cpp:44-45
        err = 2;
        break;
      }
      const float a = (float)(rho / denom);
      double sn = 0.0;
      for (int i = threadIdx.x; i < nel_s; i += blockDim.x) {
        const float2 pv = ps[i];
        const float dv = __ldg(dg + i / J);
        const float2 ap = make_float2(dv * pv.x, dv * pv.y);
        float2 xv = xs[i], rv = rs[i];
        xv = make_float2(fmaf(a, pv.x, xv.x), fmaf(a, pv.y, xv.y));
        rv = make_float2(fmaf(-a, ap.x, rv.x), fmaf(-a, ap.y, rv.y));
        xs[i] = xv;
        rs[i] = rv;
        sn += (double)rv.x * rv.x + (double)rv.y * rv.y;
      }
      const double rho_next = block_sum_all(sn, sh);
      if (!isfinite(rho_next)) {  // solvers.cpp:52-53
        err = 1;
        break;
      }
      rel = sqrt(rho_next) / bnorm;
      if (rel <= cg_tol) {
        ++it;
        break;
      }
      g = (float)(rho_next / rho);
      rho = rho_next;
    }
  }
  if (threadIdx.x == 0) {
    ctl[s].cg_it = it;
    ctl[s].cg_rel = rel;
    if (err) {
      ctl[s].error = err;
      halt[s] = 1;
    }
  }
}

// rel_change_sq (solvers.cpp:80-87) per slice by Parseval in PE k-space,
// the log record and the slice's stop rule (solvers.cpp:290-294).
__global__ void k_p_relchange(const float2* __restrict__ x, const float2* __restrict__ xold, int nel_s,
                              ParamSliceCtl* __restrict__ ctl, int* __restrict__ halt,
                              int* __restrict__ have_v, double* __restrict__ log, double tol,
                              int max_outer) {
  __shared__ double sh[33];
  const int s = blockIdx.x;
  if (halt[s]) return;
  const size_t base = (size_t)s * nel_s;
  double sn = 0.0, sd = 0.0;
  for (int i = threadIdx.x; i < nel_s; i += blockDim.x) {
    const float2 a = x[base + i], b = xold[base + i];
    const double dx = (double)a.x - b.x, dy = (double)a.y - b.y;
    sn += dx * dx + dy * dy;
    sd += (double)b.x * b.x + (double)b.y * b.y;
  }
  const double num = block_sum(sn, sh);
  const double den = block_sum(sd, sh);
  if (threadIdx.x == 0) {
    const double rc = den > 0.0 ? num / den : (num > 0.0 ? 1.0 : 0.0);
    ParamSliceCtl& c = ctl[s];
    c.relchange = rc;
    const int k = c.outer;
    if (k < max_outer) {
      double* lg = log + ((size_t)s * max_outer + k) * 3;
      lg[0] = rc;
      lg[1] = (double)c.cg_it;
      lg[2] = c.cg_rel;
    }
    c.outer = k + 1;
    if (rc < tol) {
      c.stopped = 1;
      halt[s] = 1;
    }
    *have_v = 1;  // this iteration's SVTs left their eigenvectors in HBM
  }
}

}  // namespace

ParamPlan::ParamPlan(const ParamConfig& cfg, const double* y, const uint8_t* mask, const double* taps,
                     size_t ntaps)
    : cfg_(cfg) {
  const int S = cfg.S, N = cfg.N, L = cfg.L, J = cfg.J;
  SHLR_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  SHLR_CUDA(cudaEventCreate(&ev0_));
  SHLR_CUDA(cudaEventCreate(&ev1_));
  SHLR_CUDA(cudaEventCreate(&evA_));
  SHLR_CUDA(cudaEventCreate(&evB_));
  nel_ = (size_t)S * L * N * J;
  qpe_ = N - cfg.Ppe + 1;
  qpar_ = L - cfg.Ppar + 1;
  Bpe_ = J * (cfg.vc ? 2 : 1);

  // ---- host-side constants (fp64, rounded once)
  const auto wN = util::weights_centered_h(taps, ntaps, N);
  const auto cN = util::hankel_counts_h(N, cfg.Ppe);
  const auto cpar = util::hankel_counts_h(L, cfg.Ppar);
  const auto aN = util::lift_normal_diag_h(wN, cN, N, cfg.vc);
  std::vector<float> dg((size_t)L * N);
  for (int l = 0; l < L; ++l)
    for (int k = 0; k < N; ++k) {
      const bool s = mask[(size_t)k * L + l] != 0;
      dg[(size_t)l * N + k] = (float)((s ? cfg.lambda : 0.0) + cfg.beta * cpar[l] + cfg.beta * aN[k]);
    }
  const auto hpe0 = util::initial_weighted_adjoint_h(wN, cN, N, cfg.vc, cfg.beta);
  std::vector<float> hecho0(L);
  for (int l = 0; l < L; ++l) hecho0[l] = (float)(-cpar[l] / cfg.beta);
  std::vector<float2> wcNf(N);
  for (int k = 0; k < N; ++k) wcNf[k] = make_float2((float)wN[2 * k], (float)wN[2 * k + 1]);

  // ---- device buffers
  x0_ = dalloc_s<float2>(nel_, stream_);
  yk_ = dalloc_s<float2>(nel_, stream_);
  x_ = dalloc_s<float2>(nel_, stream_);
  xold_ = dalloc_s<float2>(nel_, stream_);
  r_ = dalloc_s<float2>(nel_, stream_);
  p_ = dalloc_s<float2>(nel_, stream_);
  bk_ = dalloc_s<float2>(nel_, stream_);
  hpe_ = dalloc_s<float2>(nel_, stream_);
  ximg_ = dalloc_s<float2>(nel_, stream_);
  hecho_ = dalloc_s<float2>(nel_, stream_);
  dg_ = dalloc_s<float>((size_t)L * N, stream_);
  hpe0_ = dalloc_s<float2>(N, stream_);
  hecho0_ = dalloc_s<float>(L, stream_);
  wcN_ = dalloc_s<float2>(N, stream_);
  halt_ = dalloc_s<int>(S, stream_);
  have_v_ = dalloc_s<int>(1, stream_);
  ctl_ = dalloc_s<ParamSliceCtl>(S, stream_);
  log_ = dalloc_s<double>((size_t)S * std::max(cfg.max_outer, 1) * 3, stream_);
  {
    const int e = std::max(cfg.Ppe, Bpe_ * qpe_), d = std::min(cfg.Ppe, Bpe_ * qpe_);
    dpe_elems_ = (size_t)S * L * e * d;
    dp_pe_ = svt_padded_dim(d);
    dpe_ = dalloc_s<float2>(dpe_elems_, stream_);
    vpe_ = dalloc_s<float2>((size_t)S * L * dp_pe_ * dp_pe_, stream_);
    vspe_ = dalloc_s<float2>((size_t)S * L * svt_subspace_store_dim(d) * kSubspaceKB, stream_);
    vspe2_ = dalloc_s<float2>((size_t)S * L * svt_subspace_store_dim(d) * (d > 128 ? kSubspaceKBBig : kSubspaceKB), stream_);
    if (d > 128) {  // large-d deflation chain (level 3)
      z1pe_ = dalloc_s<float2>(dpe_elems_, stream_);
      const int sd = svt_subspace_store_dim(d);
      vdpe_ = dalloc_s<float2>((size_t)S * L * sd * sd, stream_);
      ndpe_ = dalloc_s<int>((size_t)S * L, stream_);
    }
    if (d <= 128) ycpe_ = dalloc_s<float2>((size_t)S * L * e * kSubspaceKB, stream_);
    fallback_ = dalloc_s<int>((size_t)S * L, stream_);
    diag_ = dalloc_s<int>((size_t)S * L, stream_);
    SHLR_CUDA(cudaMemsetAsync(diag_, 0, sizeof(int) * S * L, stream_));
    SHLR_CUDA(cudaMemsetAsync(fallback_, 0, sizeof(int) * S * L, stream_));
  }
  {
    const int e = std::max(cfg.Ppar, J * qpar_), d = std::min(cfg.Ppar, J * qpar_);
    decho_elems_ = (size_t)S * N * e * d;
    dp_echo_ = svt_padded_dim(d);
    decho_ = dalloc_s<float2>(decho_elems_, stream_);
    vecho_ = dalloc_s<float2>((size_t)S * N * dp_echo_ * dp_echo_, stream_);
  }
  SHLR_CUDA(cudaMemcpyAsync(dg_, dg.data(), dg.size() * sizeof(float), cudaMemcpyHostToDevice, stream_));
  SHLR_CUDA(cudaMemcpyAsync(hpe0_, hpe0.data(), N * sizeof(float2), cudaMemcpyHostToDevice, stream_));
  SHLR_CUDA(cudaMemcpyAsync(hecho0_, hecho0.data(), L * sizeof(float), cudaMemcpyHostToDevice, stream_));
  SHLR_CUDA(cudaMemcpyAsync(wcN_, wcNf.data(), N * sizeof(float2), cudaMemcpyHostToDevice, stream_));
  tN_ = make_twiddles(N, &twN_, stream_);

  // ---- data: y (fp64) -> complex64; dataset: iFFT along FE (parammap.cpp:32);
  // then the masked PE k-space x0 and lambda * x0
  // (a dataset plan may own only FE slices [s0, s0 + S) of the M_full in y:
  // the FE transform mixes every line, so it runs over all of them)
  {
    const int Mf = cfg.dataset ? std::max(cfg.M_full, S) : S;
    const size_t nel_in = (size_t)Mf * L * N * J;
    double* y_d = dalloc_s<double>(2 * nel_in, stream_);
    float2* a_d = dalloc_s<float2>(nel_in, stream_);
    float2* b_d = cfg.dataset && !cfg.hybrid_input ? dalloc_s<float2>(nel_in, stream_) : nullptr;
    uint8_t* m_d = dalloc_s<uint8_t>((size_t)N * L, stream_);
    SHLR_CUDA(cudaMemcpyAsync(y_d, y, 2 * nel_in * sizeof(double), cudaMemcpyHostToDevice, stream_));
    SHLR_CUDA(cudaMemcpyAsync(m_d, mask, (size_t)N * L, cudaMemcpyHostToDevice, stream_));
    k_p_from_double<<<grid_for(nel_in), kThreads, 0, stream_>>>(y_d, a_d, nel_in);
    SHLR_LAUNCH_CHECK();
    const float2* hyb = a_d;
    float2* twM = nullptr;
    if (cfg.dataset && cfg.hybrid_input) {
      hyb = a_d + (size_t)cfg.s0 * N * L * J;
    } else if (cfg.dataset) {
      FftTwiddles tM = make_twiddles(Mf, &twM, stream_);
      const long long inner = (long long)N * L * J;
      StridedCopyOp op{a_d, b_d, 0, inner, 1};
      launch_fft_axis<StridedCopyOp, true>(op, tM, 1, (int)inner, 16, stream_);
      hyb = b_d + (size_t)cfg.s0 * N * L * J;
    }
    k_p_prep<<<grid_for(nel_), kThreads, 0, stream_>>>(hyb, m_d, S, N, L, J, (float)cfg.lambda, x0_, yk_);
    SHLR_LAUNCH_CHECK();
    SHLR_CUDA(cudaFreeAsync(y_d, stream_));
    SHLR_CUDA(cudaFreeAsync(a_d, stream_));
    if (b_d) SHLR_CUDA(cudaFreeAsync(b_d, stream_));
    SHLR_CUDA(cudaFreeAsync(m_d, stream_));
    if (twM) SHLR_CUDA(cudaFreeAsync(twM, stream_));
    SHLR_CUDA(cudaStreamSynchronize(stream_));
  }
  SHLR_CUDA(cudaFuncSetAttribute(k_p_cg, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
  reset();
  SHLR_CUDA(cudaStreamSynchronize(stream_));
}

ParamPlan::~ParamPlan() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph_) cudaGraphDestroy(graph_);
  void* bufs[] = {x0_, yk_, x_, xold_, r_, p_, bk_, hpe_, ximg_, hecho_, dg_, hpe0_, hecho0_, wcN_, twN_,
                  dpe_, decho_, vpe_, vecho_, vspe_, vspe2_, ycpe_, z1pe_, vdpe_, ndpe_, fallback_, diag_, halt_, have_v_, ctl_, log_};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, stream_);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (evA_) cudaEventDestroy(evA_);
  if (evB_) cudaEventDestroy(evB_);
  if (stream_) cudaStreamDestroy(stream_);
}

void ParamPlan::reset() {
  const int S = cfg_.S;
  k_p_copy<<<grid_for(nel_), kThreads, 0, stream_>>>(x_, x0_, nel_);
  k_p_fill<<<grid_for(dpe_elems_), kThreads, 0, stream_>>>(dpe_, dpe_elems_, make_float2(1.f, 0.f));
  k_p_fill<<<grid_for(decho_elems_), kThreads, 0, stream_>>>(decho_, decho_elems_, make_float2(1.f, 0.f));
  k_p_init_h<<<grid_for(nel_), kThreads, 0, stream_>>>(hpe_, hecho_, hpe0_, hecho0_, S, cfg_.N, cfg_.L,
                                                        cfg_.J);
  k_p_reset<<<(S + 255) / 256, 256, 0, stream_>>>(ctl_, halt_, have_v_, S);
  SHLR_CUDA(cudaMemsetAsync(log_, 0, 3 * sizeof(double) * S * std::max(cfg_.max_outer, 1), stream_));
  SHLR_CUDA(cudaMemsetAsync(fallback_, 0, sizeof(int) * S * cfg_.L, stream_));  // solver levels
  SHLR_LAUNCH_CHECK();
  iter_ = 0;
  subspace_used_ = false;
}

SvtParams ParamPlan::svt_params(bool pe) const {
  const int S = cfg_.S, N = cfg_.N, L = cfg_.L, J = cfg_.J;
  SvtParams sp{};
  sp.nfam = 1;
  sp.inv_beta = (float)(1.0 / cfg_.beta);
  sp.tau_dual = (float)cfg_.tau;
  sp.max_sweeps = 20;
  sp.s2_tail = kS2Tail;
  sp.s2_tol_abs = kS2TolAbs;
  sp.warm = have_v_;
  sp.q_cold = 6;
  sp.q_warm = 1;
  sp.inner_norm = 1;
  SvtFamily& F = sp.fam[0];
  F.J = J;
  F.halt = halt_;
  F.s_n = J;
  F.s_j = 1;
  F.o_n = J;
  F.o_j = 1;
  if (pe) {  // Q_l: weighted lift along PE of (slice, echo) (solvers.cpp:284-288)
    sp.mode = SVT_ADMM_WEIGHTED;
    sp.thresh = (float)(1.0 / cfg_.beta);
    F.count = S * L;
    F.len = N;
    F.P = cfg_.Ppe;
    F.q = qpe_;
    F.B = Bpe_;
    F.vc = cfg_.vc ? 1 : 0;
    F.spec = x_;
    F.s_mat = (long long)N * J;
    F.out = hpe_;
    F.wc = wcN_;
    F.D = dpe_;
    F.V = vpe_;
    F.Vs = vspe_;
    F.fallback = fallback_;
    F.halt_div = L;
    sp.ycache = ycpe_;
  } else {   // P_n: plain lift along echoes of (slice, PE row) (solvers.cpp:279-283)
    sp.mode = SVT_ADMM_PLAIN;
    sp.thresh = (float)(cfg_.lambda2 / cfg_.beta);
    F.count = S * N;
    F.len = L;
    F.P = cfg_.Ppar;
    F.q = qpar_;
    F.B = J;
    F.vc = 0;
    F.spec = ximg_;
    F.s_mat = (long long)L * J;
    F.out = hecho_;
    F.wc = nullptr;
    F.D = decho_;
    F.V = vecho_;
    F.halt_div = N;
  }
  F.o_mat = F.s_mat;
  F.wide = (F.B * F.q > F.P) ? 1 : 0;
  F.e = std::max(F.P, F.B * F.q);
  F.d = std::min(F.P, F.B * F.q);
  return sp;
}

void ParamPlan::enqueue_iteration(bool record_events) {
  const int S = cfg_.S, N = cfg_.N, L = cfg_.L, J = cfg_.J;
  const int LJ = L * J;
  const int F = std::min(16, LJ);
  // ---- RHS: b^ = lambda y^ + beta (hpe + F_PE hecho)
  {
    ParamRhsOp op{hecho_, hpe_, yk_, bk_, N, L, J, (float)cfg_.beta, halt_};
    launch_fft_axis<ParamRhsOp, false>(op, tN_, S, LJ, F, stream_);
    ++launch_count_;
  }
  // ---- X-update: per-slice capped CG (solvers.cpp:276-277)
  k_p_cg<<<S, kCgThreads, 0, stream_>>>(bk_, dg_, x_, xold_, r_, p_, L * N * J, J, ctl_, halt_,
                                          cfg_.cg_max, cfg_.cg_tol);
  SHLR_LAUNCH_CHECK();
  ++launch_count_;
  // ---- image-domain x for the echo lifts
  {
    ParamToImageOp op{x_, ximg_, N, L, J, halt_};
    launch_fft_axis<ParamToImageOp, true>(op, tN_, S, LJ, F, stream_);
    ++launch_count_;
  }
  if (record_events) SHLR_CUDA(cudaEventRecord(evA_, stream_));
  // ---- Z/D updates and the next RHS adjoints: PE family, then echo family
  {
    SvtParams sp = svt_params(true);
    sp.sweeps_out = diag_;
    sp.fam[0].Vs2 = vspe2_;
    sp.fam[0].Z1 = z1pe_;
    sp.fam[0].Vd = vdpe_;
    sp.fam[0].ndefl = ndpe_;
    int nl = 0;
    // PE lifts are low rank (mean 15-17 above the threshold at config 4):
    // a 32-column level 1, 48-column level 2, then the full solver
    if ((nl = launch_hankel_svt_levels(sp, sp.fam[0].count, stream_, kSubspaceKB1)) > 0) {
      subspace_used_ = true;
      launch_count_ += nl;
    } else {
      if (subspace_used_) sp.warm = nullptr;
      launch_hankel_svt(sp, sp.fam[0].count, stream_);
      ++launch_count_;
    }
  }
  {
    // echo lifts (P x J(L-P+1), 5 x 32 at config 4): one thread per matrix
    // when they are that small, else the general kernel
    SvtParams sp = svt_params(false);
    if (!launch_small_svt(sp, stream_)) launch_hankel_svt(sp, sp.fam[0].count, stream_);
    ++launch_count_;
  }
  if (record_events) SHLR_CUDA(cudaEventRecord(evB_, stream_));
  // ---- stop rule + log
  k_p_relchange<<<S, 512, 0, stream_>>>(x_, xold_, L * N * J, ctl_, halt_, have_v_, log_, cfg_.tol,
                                         cfg_.max_outer);
  SHLR_LAUNCH_CHECK();
  ++launch_count_;
}

void ParamPlan::build_graph() {
  launch_count_ = 0;
  SHLR_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  enqueue_iteration(false);
  SHLR_CUDA(cudaStreamEndCapture(stream_, &graph_));
  SHLR_CUDA(cudaGraphInstantiate(&graph_exec_, graph_, 0));
  launches_per_iter_ = launch_count_;
}

void ParamPlan::run(size_t iters) {
  const size_t todo = std::min(iters, (size_t)std::max(0, cfg_.max_outer - iter_));
  svt_ms_ = 0;
  const bool use_graph = !timing_ && !std::getenv("SHLR_NO_GRAPH");
  if (use_graph && !graph_exec_) build_graph();
  SHLR_CUDA(cudaEventRecord(ev0_, stream_));
  for (size_t i = 0; i < todo; ++i) {
    if (use_graph) {
      SHLR_CUDA(cudaGraphLaunch(graph_exec_, stream_));
    } else {
      launch_count_ = 0;
      enqueue_iteration(timing_);
      launches_per_iter_ = launch_count_;
      if (timing_) {
        SHLR_CUDA(cudaEventSynchronize(evB_));
        float ms = 0;
        SHLR_CUDA(cudaEventElapsedTime(&ms, evA_, evB_));
        svt_ms_ += ms;
        if (std::getenv("SHLR_RANK_DIAG")) {  // Ritz values above the threshold per PE lift
          const int n = cfg_.S * cfg_.L;
          std::vector<int> h(n);
          SHLR_CUDA(cudaMemcpy(h.data(), diag_, n * sizeof(int), cudaMemcpyDeviceToHost));
          int mx = 0;
          double mean = 0;
          for (int v : h) {
            mx = std::max(mx, v / 1000);
            mean += v / 1000;
          }
          std::fprintf(stderr, "param iter %d: PE rank above threshold max %d mean %.1f\n", iter_ + 1, mx,
                       mean / n);
        }
      }
    }
    ++iter_;
  }
  SHLR_CUDA(cudaEventRecord(ev1_, stream_));
}

void ParamPlan::sync() {
  SHLR_CUDA(cudaStreamSynchronize(stream_));
  float ms = 0;
  if (cudaEventElapsedTime(&ms, ev0_, ev1_) == cudaSuccess) total_ms_ = ms;
}

void ParamPlan::download(double* x_out, std::vector<int>* outer, std::vector<double>* final_rel,
                         std::vector<std::string>* log_lines, int* error) {
  const int S = cfg_.S, N = cfg_.N, L = cfg_.L, J = cfg_.J;
  // scratch of its own: a download between run() calls leaves the plan's state alone
  float2* s1 = dalloc_s<float2>(nel_, stream_);
  ParamToImageOp op{x_, s1, N, L, J, nullptr};
  launch_fft_axis<ParamToImageOp, true>(op, tN_, S, L * J, std::min(16, L * J), stream_);
  double* xd = dalloc_s<double>(2 * nel_, stream_);
  k_p_to_double<<<grid_for(nel_), kThreads, 0, stream_>>>(s1, xd, nel_);
  SHLR_LAUNCH_CHECK();
  SHLR_CUDA(cudaFreeAsync(s1, stream_));
  std::vector<ParamSliceCtl> hc(S);
  const int mo = std::max(cfg_.max_outer, 1);
  std::vector<double> lg((size_t)S * mo * 3);
  SHLR_CUDA(cudaMemcpyAsync(x_out, xd, 2 * nel_ * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  SHLR_CUDA(cudaMemcpyAsync(hc.data(), ctl_, S * sizeof(ParamSliceCtl), cudaMemcpyDeviceToHost, stream_));
  SHLR_CUDA(cudaMemcpyAsync(lg.data(), log_, lg.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  SHLR_CUDA(cudaStreamSynchronize(stream_));
  SHLR_CUDA(cudaFreeAsync(xd, stream_));
  *error = 0;
  if (outer) outer->assign(S, 0);
  if (final_rel) final_rel->assign(S, 1.0);
  if (log_lines) log_lines->clear();
  for (int s = 0; s < S; ++s) {
    if (outer) (*outer)[s] = hc[s].outer;
    if (final_rel) (*final_rel)[s] = hc[s].outer > 0 ? hc[s].relchange : 1.0;
    if (!*error && hc[s].error) *error = hc[s].error;
    if (log_lines)
      for (int k = 0; k < hc[s].outer && k < cfg_.max_outer; ++k) {
        const double* l = &lg[((size_t)s * mo + k) * 3];
        char buf[160];
        std::snprintf(buf, sizeof buf, "iter=%d relchange=%.3e cg_iters=%d cg_res=%.3e", k + 1, l[0],
                      (int)l[1], l[2]);
        log_lines->push_back(buf);
      }
  }
  if (!*error && dp_pe_ > 128 && subspace_used_) {
    // large-d PE lifts: a matrix left with more singular values above the
    // threshold than the subspace levels hold is reported (as PiPlan does)
    std::vector<int> fl((size_t)S * L);
    SHLR_CUDA(cudaMemcpy(fl.data(), fallback_, fl.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int f : fl)
      if (f == kLevelOverflow) *error = 3;
  }
}

}  // namespace shlr_b200
