// Parameter-imaging ADMM (SHLR-P / SHLR-VP, Algorithm S2) on one B200:
// shlr_param_reconstruct_slice (proj/src/solvers.cpp:193-298) for every
// frequency-encode slice of recon_param_dataset (proj/src/parammap.cpp:21-54)
// at once.  The slices are independent ADMM problems; they run batched in
// the same launches, each with its own CG scalars and its own early stop.
#pragma once

#include <string>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "hankel_svt.cuh"

namespace shlr_b200 {

// Per-slice solver state (one per FE slice).
struct ParamSliceCtl {
  double relchange;
  double cg_rel;
  int cg_it;
  int outer;     // completed outer iterations
  int stopped;   // early-stop rule fired (solvers.cpp:294)
  int error;     // 1: non-finite residual, 2: operator not positive definite
};

struct ParamConfig {
  int S;                 // slices batched (M FE lines, or 1 for a single slice)
  int N, L, J;           // phase encodes, echoes, coils of one slice
  int Ppe, Ppar;         // pencil_for(N), pencil_for_param(L) (hankel.cpp:10-29)
  bool vc;
  bool dataset;          // y is M x N x L x J k-space: iFFT along FE first (parammap.cpp:32)
  int M_full;            // dataset: FE lines of y (the plan solves slices [s0, s0 + S))
  bool hybrid_input;     // dataset: y is already iFFT'd along FE (the caller did parammap.cpp:32)
  int s0;
  double lambda, lambda2, beta, tau, tol, cg_tol;
  int max_outer, cg_max;
};

class ParamPlan {
 public:
  // y: dataset M x N x L x J (k-space) or slice N x L x J (hybrid: FE image,
  // PE k-space), interleaved complex128.  mask: N x L uint8 (row = phase
  // encode, column = echo; sampling.hpp:33-52).
  ParamPlan(const ParamConfig& cfg, const double* y, const uint8_t* mask, const double* taps,
            size_t ntaps);
  ~ParamPlan();
  ParamPlan(const ParamPlan&) = delete;
  ParamPlan& operator=(const ParamPlan&) = delete;

  void reset();
  void run(size_t iters);
  void sync();
  // x_out: S x N x L x J interleaved complex128 (image domain along PE);
  // per-slice iteration counts / final relative changes and the log lines
  // of every slice in slice order (the order recon_param_dataset logs them).
  void download(double* x_out, std::vector<int>* outer, std::vector<double>* final_rel,
                std::vector<std::string>* log_lines, int* error);
  double svt_ms() const { return svt_ms_; }
  double total_ms() const { return total_ms_; }
  int launches_per_iter() const { return launches_per_iter_; }
  void set_timing(bool on) { timing_ = on; }
  const ParamConfig& config() const { return cfg_; }

 private:
  void enqueue_iteration(bool record_events);
  void build_graph();
  SvtParams svt_params(bool pe) const;

  ParamConfig cfg_;
  cudaStream_t stream_ = nullptr;
  size_t nel_ = 0;        // S * L * N * J
  int qpe_ = 0, qpar_ = 0, Bpe_ = 0;

  // k-space state [S][L][N][J]
  float2 *x0_ = nullptr, *yk_ = nullptr, *x_ = nullptr, *xold_ = nullptr, *r_ = nullptr,
         *p_ = nullptr, *bk_ = nullptr, *hpe_ = nullptr;
  // image-domain (along PE) [S][N][L][J]
  float2 *ximg_ = nullptr, *hecho_ = nullptr;
  float* dg_ = nullptr;              // [L][N] diagonal of the X-update operator
  float2 *hpe0_ = nullptr, *wcN_ = nullptr, *twN_ = nullptr;
  float* hecho0_ = nullptr;          // [L] -counts_par / beta
  float2 *dpe_ = nullptr, *decho_ = nullptr;    // duals (Ahat orientation)
  float2 *vpe_ = nullptr, *vecho_ = nullptr;    // full-solver eigenvector stores
  float2* vspe_ = nullptr;                      // subspace-solver block store (PE family)
  float2* vspe2_ = nullptr;                     // its level-2 store
  float2* ycpe_ = nullptr;                      // Ahat V of the Rayleigh-Ritz pass (SvtParams::ycache)
  float2* z1pe_ = nullptr;                      // PE d > 128: Z1 of the deflated level 3
  float2* vdpe_ = nullptr;                      // PE d > 128: deflation chain bases
  int* ndpe_ = nullptr;                         // PE d > 128: deflated columns per matrix
  int* fallback_ = nullptr;
  int* diag_ = nullptr;              // per-PE-lift diagnostics (sweeps_out of the SVT launch)
  int* halt_ = nullptr;              // [S] stopped || error
  int* have_v_ = nullptr;            // warm-start flag (after the first iteration)
  ParamSliceCtl* ctl_ = nullptr;     // [S]
  double* log_ = nullptr;            // [S][max_outer][3]
  FftTwiddles tN_;
  size_t dpe_elems_ = 0, decho_elems_ = 0;
  int dp_pe_ = 0, dp_echo_ = 0;
  bool subspace_used_ = false;

  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr, evA_ = nullptr, evB_ = nullptr;
  bool timing_ = false;
  double svt_ms_ = 0, total_ms_ = 0;
  int launches_per_iter_ = 0, launch_count_ = 0, iter_ = 0;
};

}  // namespace shlr_b200
