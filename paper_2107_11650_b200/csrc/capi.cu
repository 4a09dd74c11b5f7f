// extern "C" boundary (include/shlr_cuda.h).  Every entry point converts C++
// exceptions into return codes; no CPU fallback exists anywhere behind it.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/shlr_cuda.h"
#include "metrics.cuh"
#include "param_solver.cuh"
#include "pi_solver.cuh"

namespace shlr_b200 {
bool spirit_calibrate_device(const double* acs, size_t a, size_t b, size_t j, size_t k, double tikhonov,
                             double* weights_out);
}

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <class Fn>
int guarded(Fn&& fn) {
  g_last_error.clear();
  try {
    return fn();
  } catch (const shlr_b200::InvalidArg& e) {
    return fail(SHLR_EINVAL, e.what());
  } catch (const shlr_b200::Unsupported& e) {
    return fail(SHLR_EUNSUPPORTED, e.what());
  } catch (const shlr_b200::CudaError& e) {
    return fail(SHLR_ECUDA, e.what());
  } catch (const std::exception& e) {
    return fail(SHLR_ECUDA, e.what());
  }
}

int require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw shlr_b200::CudaError("no CUDA device visible: the SHLR B200 path has no CPU fallback");
  }
  return n;
}

// Mirrors AdmmConfig::validate (solvers.hpp:29-33) and the argument checks
// of shlr_pi_reconstruct (solvers.cpp:101-123).
void validate_pi(const shlr_pi_args* a) {
  using shlr_b200::InvalidArg;
  if (!a) throw InvalidArg("shlr_pi_reconstruct: null args");
  if (a->lambda <= 0 || a->lambda1 < 0 || a->beta <= 0 || a->tau <= 0 || a->tol <= 0 ||
      a->cg_tol <= 0)
    throw InvalidArg("AdmmConfig: invalid parameter");
  if (a->m == 0 || a->n == 0 || a->j == 0 || !a->y)
    throw InvalidArg("shlr_pi_reconstruct: expected M x N x J");
  if (a->enable_spirit && !a->spirit_weights)
    throw InvalidArg("shlr_pi_reconstruct: spirit enabled without kernels");
  if (!a->mask || (a->mask_rows != 1 && a->mask_rows != a->m))
    throw InvalidArg("shlr_pi_reconstruct: mask dims mismatch");
  if (a->pencil_row < 1 || a->pencil_row > a->n || a->pencil_col < 1 || a->pencil_col > a->m)
    throw InvalidArg("HankelConfig: pencil exceeds signal length");
  if (!a->taps || a->ntaps == 0 || a->ntaps > a->n || a->ntaps > a->m)
    throw InvalidArg("weights_from_filter: taps invalid");
  if (a->enable_spirit && (a->spirit_k % 2 == 0 || a->spirit_k == 0))
    throw InvalidArg("SpiritKernels: kernel size must be odd");
}

shlr_b200::PiConfig config_of(const shlr_pi_args* a) {
  shlr_b200::PiConfig c{};
  c.M = (int)a->m;
  c.N = (int)a->n;
  c.J = (int)a->j;
  c.Pr = (int)a->pencil_row;
  c.Pc = (int)a->pencil_col;
  c.vc = a->enable_vc != 0;
  // solvers.cpp:118-119: lambda1 is used only with SPIRiT enabled and > 0.
  c.spirit = a->enable_spirit != 0 && a->lambda1 > 0.0;
  c.lambda = a->lambda;
  c.lambda1 = c.spirit ? a->lambda1 : 0.0;
  c.beta = a->beta;
  c.tau = a->tau;
  c.tol = a->tol;
  c.cg_tol = a->cg_tol;
  c.max_outer = (int)a->max_outer;
  c.cg_max = (int)a->cg_max;
  c.debug_sv_iter = a->debug_sv_iter;
  return c;
}

// Mirrors AdmmConfig::validate and the checks of shlr_param_reconstruct_slice
// (solvers.cpp:199-206) / recon_param_dataset (parammap.cpp:27-30).
void validate_param(const shlr_param_args* a) {
  using shlr_b200::InvalidArg;
  if (!a) throw InvalidArg("shlr_param_reconstruct_slice: null args");
  if (a->lambda <= 0 || a->lambda2 < 0 || a->beta <= 0 || a->tau <= 0 || a->tol <= 0 ||
      a->cg_tol <= 0)
    throw InvalidArg("AdmmConfig: invalid parameter");
  if (a->n == 0 || a->l == 0 || a->j == 0 || !a->y)
    throw InvalidArg("shlr_param_reconstruct_slice: expected N x L x J");
  if (!a->mask) throw InvalidArg("shlr_param_reconstruct_slice: mask dims mismatch");
  if (a->pencil_pe < 1 || a->pencil_pe > a->n)
    throw InvalidArg("HankelConfig: pencil exceeds signal length");
  if (a->pencil_par < 1 || a->pencil_par > a->l)
    throw InvalidArg("HankelConfig: parameter pencil exceeds signal length");
  if (!a->taps || a->ntaps == 0 || a->ntaps > a->n)
    throw InvalidArg("weights_from_filter: taps invalid");
  if (a->slice_end != 0 || a->slice_begin != 0) {
    if (a->m == 0) throw InvalidArg("recon_param_dataset: a slice range needs a dataset");
    if (a->slice_begin >= a->slice_end || a->slice_end > a->m)
      throw InvalidArg("recon_param_dataset: slice range outside the dataset");
  }
}

shlr_b200::ParamConfig param_config_of(const shlr_param_args* a) {
  shlr_b200::ParamConfig c{};
  const bool shard = a->slice_end > a->slice_begin;
  c.S = a->m ? (shard ? (int)(a->slice_end - a->slice_begin) : (int)a->m) : 1;
  c.dataset = a->m != 0;
  c.M_full = (int)a->m;
  c.s0 = shard ? (int)a->slice_begin : 0;
  c.hybrid_input = a->m && a->hybrid_input;
  c.N = (int)a->n;
  c.L = (int)a->l;
  c.J = (int)a->j;
  c.Ppe = (int)a->pencil_pe;
  c.Ppar = (int)a->pencil_par;
  c.vc = a->enable_vc != 0;
  c.lambda = a->lambda;
  c.lambda2 = a->lambda2;
  c.beta = a->beta;
  c.tau = a->tau;
  c.tol = a->tol;
  c.cg_tol = a->cg_tol;
  c.max_outer = (int)a->max_outer;
  c.cg_max = (int)a->cg_max;
  return c;
}

}  // namespace

struct shlr_param_plan {
  shlr_b200::ParamPlan* impl;
};

struct shlr_pi_plan {
  shlr_b200::PiPlan* impl;
};

extern "C" {

int shlr_cuda_abi_version(void) { return SHLR_ABI_VERSION; }

const char* shlr_cuda_last_error(void) { return g_last_error.c_str(); }

int shlr_cuda_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int shlr_cuda_pi_plan_create(const shlr_pi_args* args, shlr_pi_plan** out) {
  return guarded([&] {
    validate_pi(args);
    if (!out) throw shlr_b200::InvalidArg("null plan pointer");
    require_device();
    auto cfg = config_of(args);
    auto* impl = new shlr_b200::PiPlan(cfg, args->y, args->mask, args->mask_rows, args->taps,
                                       args->ntaps, cfg.spirit ? args->spirit_weights : nullptr,
                                       args->spirit_k);
    *out = new shlr_pi_plan{impl};
    return SHLR_OK;
  });
}

int shlr_cuda_debug_normal_apply(const shlr_pi_args* args, const double* x_img, double* out_img) {
  return guarded([&] {
    validate_pi(args);
    if (!x_img || !out_img) throw shlr_b200::InvalidArg("normal_apply: null buffer");
    require_device();
    auto cfg = config_of(args);
    shlr_b200::PiPlan plan(cfg, args->y, args->mask, args->mask_rows, args->taps, args->ntaps,
                           cfg.spirit ? args->spirit_weights : nullptr, args->spirit_k);
    plan.debug_normal_apply(x_img, out_img);
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_reset(shlr_pi_plan* plan) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->reset();
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_run(shlr_pi_plan* plan, size_t iters) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->run(iters);
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_sync(shlr_pi_plan* plan) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->sync();
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_timing(shlr_pi_plan* plan, double* svt_ms, double* total_ms,
                             int* launches_per_iter) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    if (svt_ms) *svt_ms = plan->impl->svt_ms();
    if (total_ms) *total_ms = plan->impl->total_ms();
    if (launches_per_iter) *launches_per_iter = plan->impl->launches_per_iter();
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_download(shlr_pi_plan* plan, double* x_out, shlr_stats* stats,
                               shlr_log_fn log_cb, void* log_ctx) {
  return guarded([&] {
    if (!plan || !x_out) throw shlr_b200::InvalidArg("null plan/output");
    size_t outer = 0;
    double rel = 0;
    int err = 0;
    std::vector<std::string> lines;
    plan->impl->download(x_out, &outer, &rel, &lines, &err);
    if (log_cb)
      for (const auto& l : lines) log_cb(log_ctx, l.c_str());
    if (stats) {
      stats->outer_iters = outer;
      stats->final_rel_change = rel;
    }
    if (err == 1) return fail(SHLR_EDIVERGE, "cg_solve: non-finite residual");
    if (err == 2) return fail(SHLR_EDIVERGE, "cg_solve: operator not positive definite");
    if (err == 3)
      return fail(SHLR_EUNSUPPORTED,
                  "hankel_svt: a lifted matrix with min(m, n) > 128 has more than 118 singular values "
                  "above the threshold (large-d subspace levels 2 + 3 hold 56 + 62)");
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_set_warm_start(shlr_pi_plan* plan, int on) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->set_warm_start(on != 0);
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_debug_phases(shlr_pi_plan* plan, long long* out, int n) {
  return guarded([&] {
    if (!plan || !out) throw shlr_b200::InvalidArg("null plan/output");
    plan->impl->debug_phases(out, n);
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_debug_sweeps(shlr_pi_plan* plan, int* out, int n) {
  return guarded([&] {
    if (!plan || !out) throw shlr_b200::InvalidArg("null plan/output");
    plan->impl->debug_sweeps(out, n);
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_debug_levels(shlr_pi_plan* plan, int* out, int n) {
  return guarded([&] {
    if (!plan || !out) throw shlr_b200::InvalidArg("null plan/output");
    plan->impl->debug_levels(out, n);
    return SHLR_OK;
  });
}

int shlr_cuda_pi_plan_set_timing(shlr_pi_plan* plan, int on) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->set_timing(on != 0);
    return SHLR_OK;
  });
}

int shlr_cuda_fp32_peak_tflops(double* tflops) {
  return guarded([&] {
    if (!tflops) throw shlr_b200::InvalidArg("null output");
    require_device();
    *tflops = shlr_b200::fp32_peak_probe();
    return SHLR_OK;
  });
}

void shlr_cuda_pi_plan_destroy(shlr_pi_plan* plan) {
  if (!plan) return;
  delete plan->impl;
  delete plan;
}

int shlr_cuda_pi_reconstruct(const shlr_pi_args* args, double* x_out, double* sv_out,
                             shlr_stats* stats, shlr_log_fn log_cb, void* log_ctx) {
  shlr_pi_plan* plan = nullptr;
  int rc = shlr_cuda_pi_plan_create(args, &plan);
  if (rc != SHLR_OK) return rc;
  rc = shlr_cuda_pi_plan_run(plan, args->max_outer);
  if (rc == SHLR_OK) rc = shlr_cuda_pi_plan_sync(plan);
  if (rc == SHLR_OK) rc = shlr_cuda_pi_plan_download(plan, x_out, stats, log_cb, log_ctx);
  if ((rc == SHLR_OK || rc == SHLR_EDIVERGE) && sv_out && args->debug_sv_iter > 0) {
    const int rc2 = guarded([&] {
      plan->impl->download_sv(sv_out);
      return SHLR_OK;
    });
    if (rc == SHLR_OK) rc = rc2;
  }
  std::string err = g_last_error;
  shlr_cuda_pi_plan_destroy(plan);
  g_last_error = err;
  return rc;
}

int shlr_cuda_hankel_svt_batched(const void* vecs, int batch, int nc, int n, int p, float tau,
                                 void* out, float* sv_out, void* stream) {
  return guarded([&] {
    if (batch < 0 || nc < 1 || n < 1 || p < 1 || p > n || tau < 0 || !vecs || !out)
      throw shlr_b200::InvalidArg("hankel_svt_batched: invalid arguments");
    {
      const size_t bytes = (size_t)batch * nc * n * sizeof(float2);
      const char* a = static_cast<const char*>(vecs);
      const char* b = static_cast<const char*>(out);
      if (bytes && a < b + bytes && b < a + bytes)
        throw shlr_b200::InvalidArg("hankel_svt_batched: out overlaps vecs");
    }
    require_device();
    shlr_b200::hankel_svt_batched_device(static_cast<const float2*>(vecs), batch, nc, n, p, tau,
                                         static_cast<float2*>(out), sv_out,
                                         static_cast<cudaStream_t>(stream));
    return SHLR_OK;
  });
}

int shlr_cuda_hankel_svt_batched_host(const double* vecs, int batch, int nc, int n, int p,
                                      double tau, double* out, double* sv_out) {
  return guarded([&] {
    if (batch < 0 || nc < 1 || n < 1 || p < 1 || p > n || tau < 0 || !vecs || !out)
      throw shlr_b200::InvalidArg("hankel_svt_batched: invalid arguments");
    require_device();
    const size_t tot = (size_t)batch * nc * n;
    const int q = n - p + 1;
    const int d = std::min(p, nc * q);
    std::vector<float2> h(tot);
    for (size_t i = 0; i < tot; ++i) h[i] = make_float2((float)vecs[2 * i], (float)vecs[2 * i + 1]);
    float2 *dv = nullptr, *dout = nullptr;
    float* dsv = nullptr;
    SHLR_CUDA(cudaMalloc(&dv, std::max<size_t>(tot, 1) * sizeof(float2)));
    SHLR_CUDA(cudaMalloc(&dout, std::max<size_t>(tot, 1) * sizeof(float2)));
    if (sv_out) SHLR_CUDA(cudaMalloc(&dsv, std::max<size_t>((size_t)batch * d, 1) * sizeof(float)));
    SHLR_CUDA(cudaMemcpy(dv, h.data(), tot * sizeof(float2), cudaMemcpyHostToDevice));
    shlr_b200::hankel_svt_batched_device(dv, batch, nc, n, p, (float)tau, dout, dsv, nullptr);
    SHLR_CUDA(cudaMemcpy(h.data(), dout, tot * sizeof(float2), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < tot; ++i) {
      out[2 * i] = h[i].x;
      out[2 * i + 1] = h[i].y;
    }
    if (sv_out) {
      std::vector<float> s((size_t)batch * d);
      SHLR_CUDA(cudaMemcpy(s.data(), dsv, s.size() * sizeof(float), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < s.size(); ++i) sv_out[i] = s[i];
    }
    cudaFree(dv);
    cudaFree(dout);
    if (dsv) cudaFree(dsv);
    return SHLR_OK;
  });
}

int shlr_cuda_debug_svt_sweeps(const void* vecs, int batch, int nc, int n, int p, float tau,
                               void* out, int* sweeps_dev) {
  return guarded([&] {
    if (batch < 0 || nc < 1 || n < 1 || p < 1 || p > n || tau < 0 || !vecs || !out || !sweeps_dev)
      throw shlr_b200::InvalidArg("debug_svt_sweeps: invalid arguments");
    require_device();
    shlr_b200::hankel_svt_batched_device(static_cast<const float2*>(vecs), batch, nc, n, p, tau,
                                         static_cast<float2*>(out), nullptr, nullptr, sweeps_dev);
    return SHLR_OK;
  });
}

int shlr_cuda_lift_index_map_path(int n, int p, int coils, int vc, int path, int32_t* map) {
  return guarded([&] {
    if (n < 1 || p < 1 || p > n || coils < 1 || !map || path < 0 || path > 2)
      throw shlr_b200::InvalidArg("lift_index_map: invalid arguments");
    require_device();
    shlr_b200::lift_index_map_device(n, p, coils, vc, path, map);
    return SHLR_OK;
  });
}

int shlr_cuda_lift_index_map(int n, int p, int coils, int vc, int32_t* map) {
  return shlr_cuda_lift_index_map_path(n, p, coils, vc, 1, map);
}

int shlr_cuda_ssos(const double* x, size_t m, size_t n, size_t j, double* out) {
  return guarded([&] {
    if (!x || !out || m == 0 || n == 0 || j == 0) throw shlr_b200::InvalidArg("ssos: expected an M x N x J tensor");
    require_device();
    shlr_b200::ssos_host(x, m, n, j, out);
    return SHLR_OK;
  });
}

int shlr_cuda_rlne(const double* ref, const double* rec, size_t count, double* out) {
  return guarded([&] {
    if (!ref || !rec || !out || count == 0) throw shlr_b200::InvalidArg("rlne: dimension mismatch");
    require_device();
    *out = shlr_b200::rlne_host(ref, rec, count);
    return SHLR_OK;
  });
}

int shlr_cuda_mssim(const double* ref, const double* rec, size_t rows, size_t cols, double* out) {
  return guarded([&] {
    if (!ref || !rec || !out) throw shlr_b200::InvalidArg("mssim: dimension mismatch");
    if (rows < 11 || cols < 11) throw shlr_b200::InvalidArg("mssim: image smaller than the 11x11 window");
    require_device();
    *out = shlr_b200::mssim_host(ref, rec, rows, cols);
    return SHLR_OK;
  });
}

int shlr_cuda_fft_along_axis(double* data, const size_t* dims, int ndim, int axis, int inverse) {
  return guarded([&] {
    if (!data || !dims || ndim < 1) throw shlr_b200::InvalidArg("fft: invalid arguments");
    for (int i = 0; i < ndim; ++i)
      if (dims[i] == 0) throw shlr_b200::InvalidArg("fft: empty input");
    require_device();
    shlr_b200::fft_along_axis_host(data, dims, ndim, axis, inverse != 0);
    return SHLR_OK;
  });
}

int shlr_cuda_param_plan_create(const shlr_param_args* args, shlr_param_plan** out) {
  return guarded([&] {
    validate_param(args);
    if (!out) throw shlr_b200::InvalidArg("null plan pointer");
    require_device();
    auto* impl = new shlr_b200::ParamPlan(param_config_of(args), args->y, args->mask, args->taps,
                                          args->ntaps);
    *out = new shlr_param_plan{impl};
    return SHLR_OK;
  });
}

int shlr_cuda_param_plan_reset(shlr_param_plan* plan) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->reset();
    return SHLR_OK;
  });
}

int shlr_cuda_param_plan_run(shlr_param_plan* plan, size_t iters) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->run(iters);
    return SHLR_OK;
  });
}

int shlr_cuda_param_plan_sync(shlr_param_plan* plan) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->sync();
    return SHLR_OK;
  });
}

int shlr_cuda_param_plan_set_timing(shlr_param_plan* plan, int on) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    plan->impl->set_timing(on != 0);
    return SHLR_OK;
  });
}

int shlr_cuda_param_plan_timing(shlr_param_plan* plan, double* svt_ms, double* total_ms,
                                int* launches_per_iter) {
  return guarded([&] {
    if (!plan) throw shlr_b200::InvalidArg("null plan");
    if (svt_ms) *svt_ms = plan->impl->svt_ms();
    if (total_ms) *total_ms = plan->impl->total_ms();
    if (launches_per_iter) *launches_per_iter = plan->impl->launches_per_iter();
    return SHLR_OK;
  });
}

int shlr_cuda_param_plan_download(shlr_param_plan* plan, double* x_out, shlr_stats* stats,
                                  shlr_log_fn log_cb, void* log_ctx) {
  return guarded([&] {
    if (!plan || !x_out) throw shlr_b200::InvalidArg("null plan/output");
    std::vector<int> outer;
    std::vector<double> rel;
    std::vector<std::string> lines;
    int err = 0;
    plan->impl->download(x_out, &outer, &rel, log_cb ? &lines : nullptr, &err);
    if (log_cb)
      for (const auto& l : lines) log_cb(log_ctx, l.c_str());
    if (stats) {
      size_t total = 0;
      for (int o : outer) total += (size_t)o;
      stats->outer_iters = total;
      stats->final_rel_change = rel.empty() ? 1.0 : rel.back();
    }
    if (err == 1) return fail(SHLR_EDIVERGE, "cg_solve: non-finite residual");
    if (err == 2) return fail(SHLR_EDIVERGE, "cg_solve: operator not positive definite");
    if (err == 3)
      return fail(SHLR_EUNSUPPORTED,
                  "shlr_param_reconstruct_slice: more singular values above the threshold than the "
                  "large-d subspace levels hold");
    return SHLR_OK;
  });
}

void shlr_cuda_param_plan_destroy(shlr_param_plan* plan) {
  if (!plan) return;
  delete plan->impl;
  delete plan;
}

int shlr_cuda_param_reconstruct(const shlr_param_args* args, double* x_out, shlr_stats* stats,
                                shlr_log_fn log_cb, void* log_ctx) {
  shlr_param_plan* plan = nullptr;
  int rc = shlr_cuda_param_plan_create(args, &plan);
  if (rc != SHLR_OK) return rc;
  rc = shlr_cuda_param_plan_run(plan, args->max_outer);
  if (rc == SHLR_OK) rc = shlr_cuda_param_plan_sync(plan);
  if (rc == SHLR_OK) rc = shlr_cuda_param_plan_download(plan, x_out, stats, log_cb, log_ctx);
  std::string err = g_last_error;
  shlr_cuda_param_plan_destroy(plan);
  g_last_error = err;
  return rc;
}

int shlr_cuda_spirit_calibrate(const double* acs, size_t a, size_t b, size_t j, size_t k, double tikhonov,
                               double* weights_out) {
  return guarded([&] {
    // spirit.cpp:24-38: the reference's argument checks
    if (!acs || !weights_out || j == 0 || k == 0 || k % 2 == 0 || tikhonov < 0)
      throw shlr_b200::InvalidArg("spirit_calibrate: invalid arguments");
    if (a <= k || b <= k) throw shlr_b200::InvalidArg("spirit_calibrate: ACS region too small");
    double energy = 0.0;
    for (size_t i = 0; i < 2 * a * b * j; ++i) energy += acs[i] * acs[i];
    if (energy == 0.0) throw shlr_b200::InvalidArg("spirit_calibrate: all-zero ACS");
    require_device();
    if (!shlr_b200::spirit_calibrate_device(acs, a, b, j, k, tikhonov, weights_out))
      throw shlr_b200::InvalidArg("spirit_calibrate: normal matrix not positive definite");
    return SHLR_OK;
  });
}

}  // extern "C"
