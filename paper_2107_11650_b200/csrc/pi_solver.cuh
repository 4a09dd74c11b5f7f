// Parallel-imaging ADMM (shlr_pi_reconstruct, proj/src/solvers.cpp:95-191)
// on one B200, in centred 2D k-space.
#pragma once

#include <string>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "hankel_svt.cuh"

namespace shlr_b200 {

struct CgState {
  double bnorm, rho, denom, alpha, gamma, rel, rho_next, pad0;
  int it, done, zero_b;
  int pending;  // SPIRiT CG: x += alpha p, r -= alpha A p of the last iteration not yet applied
                // (fused into the next iteration's row stage, or flushed by k_cg_flush)
};

struct SolverCtl {
  CgState cg;
  double relchange;
  int stopped;   // ADMM stop rule fired (solvers.cpp:187)
  int error;     // 1: non-finite residual, 2: operator not positive definite
  int outer;     // completed outer iterations
  int have_v;    // the SVT eigenvector store holds a warm start
  unsigned int arrive[8];
};

struct PiConfig {
  int M, N, J;
  int Pr, Pc;            // pencils: rows use pencil_for(N), columns pencil_for(M)
  bool vc, spirit;
  double lambda, lambda1, beta, tau, tol, cg_tol;
  int max_outer, cg_max;
  int debug_sv_iter;
};

class PiPlan {
 public:
  PiPlan(const PiConfig& cfg, const double* y, const uint8_t* mask, size_t mask_rows,
         const double* taps, size_t ntaps, const double* spirit_w, size_t spirit_k);
  ~PiPlan();
  PiPlan(const PiPlan&) = delete;
  PiPlan& operator=(const PiPlan&) = delete;

  void reset();                  // state back to iteration 0 (re-uploads nothing)
  void run(size_t iters);        // enqueue iters outer iterations
  void sync();
  void download(double* x_out, size_t* outer_iters, double* final_rel,
                std::vector<std::string>* log_lines, int* error);
  void download_sv(double* sv_out);   // debug hook (debug_sv_iter)
  // test hook: out = A x in the image domain with the plan's X-update operator
  void debug_normal_apply(const double* x_img, double* out_img);
  double svt_ms() const { return svt_ms_; }
  double total_ms() const { return total_ms_; }
  int launches_per_iter() const { return launches_per_iter_; }
  void set_timing(bool on) { timing_ = on; }
  void set_warm_start(bool on) { warm_start_ = on; }
  // per-matrix Jacobi sweeps (stage1 * 100 + stage2) of the last SVT launch
  void debug_sweeps(int* out, int n);
  void debug_levels(int* out, int n);
  // subspace-solver phase clocks of the last SVT launch (8 per matrix; needs
  // SHLR_PHASE_CLK in the environment at plan creation)
  void debug_phases(long long* out, int n);
  cudaStream_t stream() const { return stream_; }
  const PiConfig& config() const { return cfg_; }

 private:
  void enqueue_iteration(int k, bool record_events);
  void build_graph();
  void cg_apply_spirit(float2* in_vec, float2* out_ap, bool init);

  PiConfig cfg_;
  cudaStream_t stream_ = nullptr;
  size_t nel_ = 0;   // M*N*J
  int qr_ = 0, qc_ = 0, B_ = 0;
  int red_blocks_ = 0;

  // device buffers
  float2* x0_ = nullptr;  // masked y (k-space x0)
  float2 *yk_ = nullptr, *x_ = nullptr, *xold_ = nullptr, *r_ = nullptr, *p_ = nullptr,
         *ap_ = nullptr, *bk_ = nullptr, *tmp_ = nullptr, *tmp2_ = nullptr;
  float* dg_ = nullptr;
  float2 *srow_ = nullptr, *scol_ = nullptr, *hrow_ = nullptr, *hcol_ = nullptr;
  float2 *hrow0_ = nullptr, *hcol0_ = nullptr;
  float2 *drow_ = nullptr, *dcol_ = nullptr;
  float2 *vrow_ = nullptr, *vcol_ = nullptr;  // SVT eigenvector stores (warm start)
  bool cg_fused_ = true;      // SPIRiT CG: vector update fused into the row stages (SHLR_CG_UNFUSED=1: off)
  float2* ycache_ = nullptr;  // Ahat V of the Rayleigh-Ritz pass, kept for the Z pass (SvtParams::ycache)
  float2 *vsrow_ = nullptr, *vscol_ = nullptr;  // subspace-solver block stores (warm start)
  float2 *vs2row_ = nullptr, *vs2col_ = nullptr;  // large-d level-2 block stores
  float2 *z1row_ = nullptr, *z1col_ = nullptr;    // large-d level-2 Z1 (level-3 deflation)
  float2 *vdrow_ = nullptr, *vdcol_ = nullptr;    // large-d deflation chain bases
  int* ndefl_ = nullptr;
  int cg_grid_ = 0;         // persistent SPIRiT CG loop: cooperative grid (0: per-stage kernels)
  size_t cg_smem_ = 0;                          // deflated columns per matrix (rows, then columns)
  int* fallback_ = nullptr;                     // per-matrix subspace -> full fallback flags
  int q_cold_ = 6, q_warm_ = 1;
  int kb1_ = kSubspaceKB;  // level-1 block of the subspace SVT (d <= 128); SHLR_KB1 overrides
  bool subspace_ = true;
  float rr_tol_rel_ = 0.f, rr_tol_abs_ = 0.f;  // 0 = kernel defaults
  float rr_tail_ = 0.f;
  bool subspace_used_ = false;                // an earlier iteration ran the subspace solver
  int* sweeps_ = nullptr;                     // diagnostics
  long long* phase_clk_ = nullptr;            // diagnostics
  bool warm_start_ = true;
  int svt_dp_ = 0;
  float2 *wcN_ = nullptr, *wcM_ = nullptr;
  float2* pmat_ = nullptr;  // SPIRiT (G-I)^H(G-I) per pixel, [M][N][J][J]
  int* rank_prev_ = nullptr;  // Ritz values above the threshold per lifted matrix, previous iteration
  float2* ppack_ = nullptr;  // 8 coils: its packed Hermitian form, [N][M][36] (k_spirit_cols_bulk)
  size_t cols_bulk_smem_ = 0;
  float2 *twM_ = nullptr, *twN_ = nullptr;
  float* sv_ = nullptr;     // debug singular values
  double* partials_ = nullptr;
  SolverCtl* ctl_ = nullptr;
  double* log_ = nullptr;   // max_outer x 3
  FftTwiddles tM_, tN_;
  size_t d_row_elems_ = 0, d_col_elems_ = 0;
  int d_sv_ = 0;

  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr, evA_ = nullptr, evB_ = nullptr;
  bool timing_ = false;
  double svt_ms_ = 0, total_ms_ = 0;
  int launches_per_iter_ = 0;
  int launch_count_ = 0;
  int iter_ = 0;
};

// Standalone helpers used by the C ABI.
void hankel_svt_batched_device(const float2* vecs, int batch, int nc, int n, int p, float tau,
                               float2* out, float* sv, cudaStream_t stream,
                               int* sweeps_out = nullptr);
void fft_along_axis_host(double* data, const size_t* dims, int ndim, int axis, bool inverse);
double fp32_peak_probe();

}  // namespace shlr_b200
