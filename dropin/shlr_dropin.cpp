// The reference-side drop-in: the bodies a maintainer swaps
// into the reference library so that its own API -- and every caller of it
// (tools/shlr_cli.cpp, tests/test_*.cpp, tests/acceptance.cpp) -- runs the
// B200 path.  Compiled in namespace shlr against the reference's own headers
// (proj/include/shlr/*.hpp, read in place) and linked with the reference's
// other translation units, whose definitions of these entry points are made
// weak (dropin/Makefile), and with libshlr_b200.so through the C-ABI of
// include/shlr_cuda.h.
//
// Replaced entry points (reference file:line of the body each one replaces):
//   shlr_pi_reconstruct           proj/src/solvers.cpp:95-191
//   shlr_param_reconstruct_slice  proj/src/solvers.cpp:193-298
//   recon_param_dataset           proj/src/parammap.cpp:21-54 (its host FE transform,
//                                 then all FE slices batched in one device call)
//   ssos                          proj/src/io.cpp:105-117
//   rlne, mssim                   proj/src/metrics.cpp:9-75
// Each keeps the reference's argument validation, in the reference's order
// and with its exception types, before the device call.
#include <ostream>
#include <stdexcept>
#include <string>

#include "shlr/fft.hpp"
#include "shlr/io.hpp"
#include "shlr/metrics.hpp"
#include "shlr/parammap.hpp"
#include "shlr/solvers.hpp"
#include "shlr_cuda.h"

namespace shlr {

namespace {

void log_line(void* ctx, const char* line) {
  if (ctx) *static_cast<std::ostream*>(ctx) << line << "\n";
}

// C-ABI return code -> the reference's exception types
void check(int rc) {
  if (rc == SHLR_OK) return;
  const std::string msg = shlr_cuda_last_error();
  if (rc == SHLR_EINVAL) throw std::invalid_argument(msg);
  if (rc == SHLR_EDIVERGE) throw DivergenceError(msg);  // solvers.cpp:36,45,53
  throw std::runtime_error(msg);                        // CUDA error / geometry outside this build
}

shlr_param_args param_args(const ComplexTensor& y, std::size_t m, std::size_t n, std::size_t l, std::size_t j,
                           const SamplingMask& mask, const HankelConfig& cfg, const AdmmConfig& acfg) {
  shlr_param_args a{};
  a.m = m;
  a.n = n;
  a.l = l;
  a.j = j;
  a.y = reinterpret_cast<const double*>(y.data());
  a.mask = mask.bits.data();
  a.taps = reinterpret_cast<const double*>(cfg.filter_taps.data());
  a.ntaps = cfg.filter_taps.size();
  a.pencil_pe = cfg.pencil_for(n);       // hankel.cpp:10-18 (throws as the reference does)
  a.pencil_par = cfg.pencil_for_param(l);  // hankel.cpp:20-29
  a.lambda = acfg.lambda;
  a.lambda2 = acfg.lambda2;
  a.beta = acfg.beta;
  a.tau = acfg.tau;
  a.tol = acfg.tol;
  a.cg_tol = acfg.cg_tol;
  a.max_outer = acfg.max_outer;
  a.cg_max = acfg.cg_max;
  a.enable_vc = acfg.enable_vc ? 1 : 0;
  return a;
}

}  // namespace

ComplexTensor shlr_pi_reconstruct(const ComplexTensor& y, const SamplingMask& mask, const SpiritKernels* g,
                                  const HankelConfig& hcfg, const AdmmConfig& acfg, std::ostream* log,
                                  SolveStats* stats) {
  // solvers.cpp:101-121, same order and messages
  acfg.validate();
  if (y.rank() != 3) throw std::invalid_argument("shlr_pi_reconstruct: expected M x N x J");
  if (acfg.enable_spirit && !g) throw std::invalid_argument("shlr_pi_reconstruct: spirit enabled without kernels");
  const std::size_t m = y.dim(0), n = y.dim(1), j = y.dim(2);
  if (mask.cols != n || (mask.rows != 1 && mask.rows != m))
    throw std::invalid_argument("shlr_pi_reconstruct: mask dims mismatch");
  HankelConfig cfg = hcfg;
  cfg.virtual_coil = acfg.enable_vc;  // solvers.cpp:112
  const std::size_t p_row = cfg.pencil_for(n);
  const std::size_t p_col = cfg.pencil_for(m);
  const double lambda1 = acfg.enable_spirit ? acfg.lambda1 : 0.0;  // solvers.cpp:118
  const bool use_spirit = acfg.enable_spirit && lambda1 > 0.0;
  if (use_spirit && g->coils() != j) throw std::invalid_argument("shlr_pi_reconstruct: kernel coil mismatch");

  shlr_pi_args a{};
  a.m = m;
  a.n = n;
  a.j = j;
  a.y = reinterpret_cast<const double*>(y.data());
  a.mask = mask.bits.data();
  a.mask_rows = mask.rows;
  a.spirit_weights = use_spirit ? reinterpret_cast<const double*>(g->raw().data()) : nullptr;
  a.spirit_k = use_spirit ? g->kernel_size() : 0;
  a.taps = reinterpret_cast<const double*>(cfg.filter_taps.data());
  a.ntaps = cfg.filter_taps.size();
  a.pencil_row = p_row;
  a.pencil_col = p_col;
  a.lambda = acfg.lambda;
  a.lambda1 = acfg.lambda1;
  a.beta = acfg.beta;
  a.tau = acfg.tau;
  a.tol = acfg.tol;
  a.cg_tol = acfg.cg_tol;
  a.max_outer = acfg.max_outer;
  a.cg_max = acfg.cg_max;
  a.enable_spirit = acfg.enable_spirit ? 1 : 0;
  a.enable_vc = acfg.enable_vc ? 1 : 0;
  ComplexTensor x({m, n, j});
  shlr_stats st{};
  const int rc = shlr_cuda_pi_reconstruct(&a, reinterpret_cast<double*>(x.data()), nullptr, &st,
                                          log ? log_line : nullptr, log);
  if (stats) *stats = {st.outer_iters, st.final_rel_change};
  check(rc);
  return x;
}

ComplexTensor shlr_param_reconstruct_slice(const ComplexTensor& y_m, const SamplingMask& mask,
                                           const HankelConfig& hcfg, const AdmmConfig& acfg, std::ostream* log,
                                           SolveStats* stats) {
  // solvers.cpp:199-206
  acfg.validate();
  if (y_m.rank() != 3) throw std::invalid_argument("shlr_param_reconstruct_slice: expected N x L x J");
  const std::size_t n = y_m.dim(0), l = y_m.dim(1), j = y_m.dim(2);
  if (mask.rows != n || mask.cols != l) throw std::invalid_argument("shlr_param_reconstruct_slice: mask dims mismatch");
  HankelConfig cfg = hcfg;
  cfg.virtual_coil = acfg.enable_vc;  // solvers.cpp:209
  const shlr_param_args a = param_args(y_m, 0, n, l, j, mask, cfg, acfg);
  ComplexTensor x({n, l, j});
  shlr_stats st{};
  const int rc =
      shlr_cuda_param_reconstruct(&a, reinterpret_cast<double*>(x.data()), &st, log ? log_line : nullptr, log);
  if (stats) *stats = {st.outer_iters, st.final_rel_change};
  check(rc);
  return x;
}

ParameterDataset recon_param_dataset(const ParameterDataset& y, const SamplingMask& mask, const HankelConfig& hcfg,
                                     const AdmmConfig& acfg, std::ostream* log, std::size_t* total_iters) {
  // parammap.cpp:25-30; each slice's own checks (solvers.cpp:199-206) once for all
  y.validate();
  const std::size_t m = y.fe(), n = y.pe(), l = y.echoes(), j = y.coils();
  if (mask.rows != n || mask.cols != l) throw std::invalid_argument("recon_param_dataset: mask dims mismatch");
  acfg.validate();
  HankelConfig cfg = hcfg;
  cfg.virtual_coil = acfg.enable_vc;
  // the reference's own setup transform (parammap.cpp:32, host FP64), then
  // every FE slice's ADMM batched on the device in one call
  const ComplexTensor hybrid = fft_along_axis(y.data, 0, true);
  shlr_param_args a = param_args(hybrid, m, n, l, j, mask, cfg, acfg);
  a.hybrid_input = 1;
  ParameterDataset out;
  out.tes_ms = y.tes_ms;
  out.data = ComplexTensor({m, n, l, j});
  shlr_stats st{};
  const int rc = shlr_cuda_param_reconstruct(&a, reinterpret_cast<double*>(out.data.data()), &st,
                                             log ? log_line : nullptr, log);
  if (total_iters) *total_iters = st.outer_iters;
  check(rc);
  return out;
}

RealImage ssos(const ComplexTensor& x) {
  if (x.rank() != 3) throw std::invalid_argument("ssos: expected an M x N x J tensor");  // io.cpp:106-107
  RealImage out(x.dim(0), x.dim(1));
  check(shlr_cuda_ssos(reinterpret_cast<const double*>(x.data()), x.dim(0), x.dim(1), x.dim(2), out.data()));
  return out;
}

double rlne(const RealImage& ref, const RealImage& rec) {
  if (ref.rows() != rec.rows() || ref.cols() != rec.cols())  // metrics.cpp:10-11
    throw std::invalid_argument("rlne: dimension mismatch");
  double v = 0.0;
  check(shlr_cuda_rlne(ref.data(), rec.data(), ref.size(), &v));
  return v;
}

double mssim(const RealImage& ref, const RealImage& rec) {
  if (ref.rows() != rec.rows() || ref.cols() != rec.cols())  // metrics.cpp:24-25
    throw std::invalid_argument("mssim: dimension mismatch");
  double v = 0.0;
  check(shlr_cuda_mssim(ref.data(), rec.data(), ref.rows(), ref.cols(), &v));
  return v;
}

}  // namespace shlr
