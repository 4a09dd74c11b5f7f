// shlr_b200/shlr.hpp -- C++ host mirror of the reference reconstruction API
// (proj/include/shlr/{tensor,sampling,hankel,spirit,solvers}.hpp) over the
// C-ABI in include/shlr_cuda.h.  Same type names, field meanings, defaults,
// argument validation order and exception types as the reference, so code
// written against shlr:: compiles against shlr_b200:: unchanged for the
// reconstruction path:
//
//   shlr_pi_reconstruct     solvers.hpp:64-70   (validation solvers.cpp:101-123)
//   shlr_param_reconstruct_slice                solvers.hpp:74-79   (validation solvers.cpp:199-206)
//   ParameterDataset, recon_param_dataset       parammap.hpp:11-40  (validation parammap.cpp:10-30)
//   AdmmConfig / validate   solvers.hpp:16-34
//   SolveStats, DivergenceError                 solvers.hpp:36-43
//   HankelConfig::pencil_for                    hankel.hpp:15-25, hankel.cpp:10-18
//   SamplingMask, mask_gauss_cartesian, mask_random2d, acs_range
//                                               sampling.hpp:33-68
//   SpiritKernels, spirit_calibrate             spirit.hpp:12-64
//   ComplexTensor (row-major, coil fastest)     tensor.hpp:16-119
//
// All numerical work runs on the GPU through libshlr_b200.so; there is no CPU
// fallback (a host without a device gets shlr_b200::CudaError).
#pragma once

#include <complex>
#include <cstddef>
#include <cstdint>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../shlr_cuda.h"

namespace shlr_b200 {

using cplx = std::complex<double>;

struct DivergenceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CalibrationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc, const char* what) {
  if (rc == SHLR_OK) return;
  const std::string msg = std::string(what) + ": " + shlr_cuda_last_error();
  if (rc == SHLR_EINVAL) throw std::invalid_argument(msg);
  if (rc == SHLR_EDIVERGE) throw DivergenceError(msg);
  if (rc == SHLR_EUNSUPPORTED) throw std::domain_error(msg);
  throw CudaError(msg);
}
}  // namespace detail

/// N-dimensional complex tensor, row-major (last dimension fastest).
class ComplexTensor {
 public:
  ComplexTensor() = default;
  explicit ComplexTensor(std::vector<std::size_t> dims) : dims_(std::move(dims)) {
    if (dims_.empty()) throw std::invalid_argument("ComplexTensor: rank must be >= 1");
    std::size_t n = 1;
    for (auto d : dims_) {
      if (d == 0) throw std::invalid_argument("ComplexTensor: all dims must be >= 1");
      n *= d;
    }
    data_.assign(n, cplx{0.0, 0.0});
  }
  ComplexTensor(std::vector<std::size_t> dims, std::vector<cplx> data) : ComplexTensor(std::move(dims)) {
    if (data.size() != data_.size())
      throw std::invalid_argument("ComplexTensor: data size does not match dims");
    data_ = std::move(data);
  }
  const std::vector<std::size_t>& dims() const { return dims_; }
  std::size_t rank() const { return dims_.size(); }
  std::size_t dim(std::size_t i) const { return dims_.at(i); }
  std::size_t size() const { return data_.size(); }
  cplx* data() { return data_.data(); }
  const cplx* data() const { return data_.data(); }
  cplx& operator[](std::size_t i) { return data_[i]; }
  const cplx& operator[](std::size_t i) const { return data_[i]; }
  cplx& at(std::size_t i0, std::size_t i1, std::size_t i2) {
    return data_[(i0 * dims_[1] + i1) * dims_[2] + i2];
  }
  const cplx& at(std::size_t i0, std::size_t i1, std::size_t i2) const {
    return data_[(i0 * dims_[1] + i1) * dims_[2] + i2];
  }

 private:
  std::vector<std::size_t> dims_;
  std::vector<cplx> data_;
};

struct SamplingMask {
  std::size_t rows = 0, cols = 0;
  std::vector<std::uint8_t> bits;  // rows * cols, row-major
  std::string generator;
  std::uint64_t seed = 0;
  double rate = 0.0;
  std::size_t acs = 0;
  double pf = 1.0;
  bool at(std::size_t r, std::size_t c) const { return bits[r * cols + c] != 0; }
  bool sampled(std::size_t r, std::size_t c) const { return bits[(rows == 1 ? 0 : r) * cols + c] != 0; }
  std::size_t count() const {
    std::size_t c = 0;
    for (auto b : bits) c += b != 0;
    return c;
  }
};

inline std::pair<std::size_t, std::size_t> acs_range(std::size_t n, std::size_t acs) {
  std::size_t a0 = 0, a1 = 0;
  if (shlr_acs_range(n, acs, &a0, &a1) != SHLR_OK)
    throw std::invalid_argument("acs_range: acs block does not fit");
  return {a0, a1};
}

inline SamplingMask mask_gauss_cartesian(std::size_t n, double rate, std::size_t acs, std::uint64_t seed) {
  SamplingMask m;
  m.rows = 1;
  m.cols = n;
  m.bits.assign(n, 0);
  if (shlr_mask_gauss_cartesian(n, rate, acs, seed, m.bits.data()) != SHLR_OK)
    throw std::invalid_argument("mask_gauss_cartesian: invalid arguments");
  m.generator = "gauss_cartesian";
  m.seed = seed;
  m.rate = rate;
  m.acs = acs;
  return m;
}

inline SamplingMask mask_random2d(std::size_t rows, std::size_t cols, double rate, std::size_t center,
                                  std::uint64_t seed) {
  SamplingMask m;
  m.rows = rows;
  m.cols = cols;
  m.bits.assign(rows * cols, 0);
  if (shlr_mask_random2d(rows, cols, rate, center, seed, m.bits.data()) != SHLR_OK)
    throw std::invalid_argument("mask_random2d: invalid arguments");
  m.generator = "random2d";
  m.seed = seed;
  m.rate = rate;
  m.acs = center;
  return m;
}

struct HankelConfig {
  std::size_t pencil = 0;
  std::size_t pencil_param = 0;
  std::vector<cplx> filter_taps = {cplx{1, 0}, cplx{-1, 0}};
  bool virtual_coil = false;
  std::size_t pencil_for(std::size_t len) const {
    const std::size_t p = shlr_pencil_for(pencil, len);
    if (p == 0) throw std::invalid_argument("HankelConfig: pencil exceeds signal length");
    return p;
  }
  std::size_t pencil_for_param(std::size_t len) const {
    const std::size_t p = shlr_pencil_for_param(pencil_param, len);
    if (p == 0) throw std::invalid_argument("HankelConfig: parameter pencil exceeds signal length");
    return p;
  }
};

struct AdmmConfig {
  double lambda = 1e4;
  double lambda1 = 1e2;
  double lambda2 = 2.0;
  double beta = 1.0;
  double tau = 1.0;
  std::size_t max_outer = 50;
  double tol = 1e-6;
  std::size_t cg_max = 15;
  double cg_tol = 1e-8;
  bool enable_spirit = false;
  bool enable_vc = false;
  void validate() const {
    if (lambda <= 0 || lambda1 < 0 || lambda2 < 0 || beta <= 0 || tau <= 0 || tol <= 0 || cg_tol <= 0)
      throw std::invalid_argument("AdmmConfig: invalid parameter");
  }
};

struct SolveStats {
  std::size_t outer_iters = 0;
  double final_rel_change = 0.0;
};

class SpiritKernels {
 public:
  SpiritKernels() = default;
  SpiritKernels(std::size_t kernel_size, std::size_t coils, std::vector<cplx> weights)
      : k_(kernel_size), j_(coils), weights_(std::move(weights)) {
    if (k_ % 2 == 0 || k_ == 0) throw std::invalid_argument("SpiritKernels: kernel size must be odd");
    if (weights_.size() != k_ * k_ * j_ * j_) throw std::invalid_argument("SpiritKernels: weight size mismatch");
    for (std::size_t j = 0; j < j_; ++j)
      if (weight(0, 0, j, j) != cplx{0, 0})
        throw std::invalid_argument("SpiritKernels: self center tap must be zero");
  }
  std::size_t kernel_size() const { return k_; }
  std::size_t coils() const { return j_; }
  cplx weight(long di, long dj, std::size_t src, std::size_t dst) const {
    const long h = static_cast<long>(k_) / 2;
    return weights_[((static_cast<std::size_t>(di + h) * k_ + static_cast<std::size_t>(dj + h)) * j_ + src) *
                        j_ + dst];
  }
  const std::vector<cplx>& raw() const { return weights_; }

 private:
  std::size_t k_ = 0, j_ = 0;
  std::vector<cplx> weights_;
};

inline SpiritKernels spirit_calibrate(const ComplexTensor& acs, std::size_t kernel_size = 5,
                                      double tikhonov = 1e-4) {
  if (acs.rank() != 3) throw std::invalid_argument("spirit_calibrate: expected a x b x J ACS");
  if (kernel_size % 2 == 0 || kernel_size == 0)
    throw std::invalid_argument("spirit_calibrate: kernel size must be odd");
  if (acs.dim(0) <= kernel_size || acs.dim(1) <= kernel_size)
    throw CalibrationError("spirit_calibrate: ACS region too small");
  if (tikhonov < 0) throw std::invalid_argument("spirit_calibrate: negative tikhonov");
  const std::size_t j = acs.dim(2);
  std::vector<cplx> w(kernel_size * kernel_size * j * j);
  const int rc = shlr_spirit_calibrate(reinterpret_cast<const double*>(acs.data()), acs.dim(0), acs.dim(1), j,
                                       kernel_size, tikhonov, reinterpret_cast<double*>(w.data()));
  if (rc != SHLR_OK) throw CalibrationError("spirit_calibrate: calibration failed");
  return SpiritKernels(kernel_size, j, std::move(w));
}

// The same calibration in FP64 on the device (shlr_cuda_spirit_calibrate).
inline SpiritKernels spirit_calibrate_device(const ComplexTensor& acs, std::size_t kernel_size = 5,
                                             double tikhonov = 1e-4) {
  if (acs.rank() != 3) throw std::invalid_argument("spirit_calibrate: expected a x b x J ACS");
  if (kernel_size % 2 == 0 || kernel_size == 0)
    throw std::invalid_argument("spirit_calibrate: kernel size must be odd");
  if (acs.dim(0) <= kernel_size || acs.dim(1) <= kernel_size)
    throw CalibrationError("spirit_calibrate: ACS region too small");
  if (tikhonov < 0) throw std::invalid_argument("spirit_calibrate: negative tikhonov");
  const std::size_t j = acs.dim(2);
  std::vector<cplx> w(kernel_size * kernel_size * j * j);
  const int rc = shlr_cuda_spirit_calibrate(reinterpret_cast<const double*>(acs.data()), acs.dim(0), acs.dim(1),
                                            j, kernel_size, tikhonov, reinterpret_cast<double*>(w.data()));
  if (rc == SHLR_EINVAL) throw CalibrationError(std::string("spirit_calibrate: ") + shlr_cuda_last_error());
  detail::check(rc, "spirit_calibrate");
  return SpiritKernels(kernel_size, j, std::move(w));
}

// Parallel-imaging ADMM (SHLR / SHLR-S / SHLR-V / SHLR-SV) on the GPU.
inline ComplexTensor shlr_pi_reconstruct(const ComplexTensor& y, const SamplingMask& mask,
                                         const SpiritKernels* g, const HankelConfig& hcfg,
                                         const AdmmConfig& acfg, std::ostream* log = nullptr,
                                         SolveStats* stats = nullptr) {
  acfg.validate();
  if (y.rank() != 3) throw std::invalid_argument("shlr_pi_reconstruct: expected M x N x J");
  if (acfg.enable_spirit && !g)
    throw std::invalid_argument("shlr_pi_reconstruct: spirit enabled without kernels");
  const std::size_t m = y.dim(0), n = y.dim(1), j = y.dim(2);
  if (mask.cols != n || (mask.rows != 1 && mask.rows != m))
    throw std::invalid_argument("shlr_pi_reconstruct: mask dims mismatch");
  const double lambda1 = acfg.enable_spirit ? acfg.lambda1 : 0.0;
  const bool use_spirit = acfg.enable_spirit && lambda1 > 0.0;
  if (use_spirit && g->coils() != j)
    throw std::invalid_argument("shlr_pi_reconstruct: kernel coil mismatch");

  shlr_pi_args a{};
  a.m = m;
  a.n = n;
  a.j = j;
  a.y = reinterpret_cast<const double*>(y.data());
  a.mask = mask.bits.data();
  a.mask_rows = mask.rows;
  a.spirit_weights = use_spirit ? reinterpret_cast<const double*>(g->raw().data()) : nullptr;
  a.spirit_k = use_spirit ? g->kernel_size() : 0;
  a.taps = reinterpret_cast<const double*>(hcfg.filter_taps.data());
  a.ntaps = hcfg.filter_taps.size();
  a.pencil_row = hcfg.pencil_for(n);
  a.pencil_col = hcfg.pencil_for(m);
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
  a.debug_sv_iter = 0;

  ComplexTensor x({m, n, j});
  shlr_stats st{};
  auto cb = [](void* ctx, const char* line) {
    if (ctx) *static_cast<std::ostream*>(ctx) << line << "\n";
  };
  const int rc = shlr_cuda_pi_reconstruct(&a, reinterpret_cast<double*>(x.data()), nullptr, &st, cb, log);
  if (stats) *stats = {st.outer_iters, st.final_rel_change};
  detail::check(rc, "shlr_pi_reconstruct");
  return x;
}

namespace detail {
inline shlr_param_args param_args(const ComplexTensor& y, std::size_t m, std::size_t n, std::size_t l,
                                  std::size_t j, const SamplingMask& mask, const HankelConfig& hcfg,
                                  const AdmmConfig& acfg) {
  shlr_param_args a{};
  a.m = m;
  a.n = n;
  a.l = l;
  a.j = j;
  a.y = reinterpret_cast<const double*>(y.data());
  a.mask = mask.bits.data();
  a.taps = reinterpret_cast<const double*>(hcfg.filter_taps.data());
  a.ntaps = hcfg.filter_taps.size();
  a.pencil_pe = hcfg.pencil_for(n);
  a.pencil_par = hcfg.pencil_for_param(l);
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
inline void log_line(void* ctx, const char* line) {
  if (ctx) *static_cast<std::ostream*>(ctx) << line << "\n";
}
}  // namespace detail

// Parameter-imaging ADMM on one PE x echo plane (SHLR-P / SHLR-VP), on the GPU.
inline ComplexTensor shlr_param_reconstruct_slice(const ComplexTensor& y_m, const SamplingMask& mask,
                                                  const HankelConfig& hcfg, const AdmmConfig& acfg,
                                                  std::ostream* log = nullptr, SolveStats* stats = nullptr) {
  acfg.validate();
  if (y_m.rank() != 3) throw std::invalid_argument("shlr_param_reconstruct_slice: expected N x L x J");
  const std::size_t n = y_m.dim(0), l = y_m.dim(1), j = y_m.dim(2);
  if (mask.rows != n || mask.cols != l)
    throw std::invalid_argument("shlr_param_reconstruct_slice: mask dims mismatch");
  const shlr_param_args a = detail::param_args(y_m, 0, n, l, j, mask, hcfg, acfg);
  ComplexTensor x({n, l, j});
  shlr_stats st{};
  const int rc = shlr_cuda_param_reconstruct(&a, reinterpret_cast<double*>(x.data()), &st,
                                             log ? detail::log_line : nullptr, log);
  if (stats) *stats = {st.outer_iters, st.final_rel_change};
  detail::check(rc, "shlr_param_reconstruct_slice");
  return x;
}

/// Multi-echo multi-coil dataset: FE x PE x echoes x coils plus echo times.
struct ParameterDataset {
  ComplexTensor data;  // M x N x L x J
  std::vector<double> tes_ms;
  void validate() const {
    if (data.rank() != 4) throw std::invalid_argument("ParameterDataset: expected M x N x L x J");
    if (tes_ms.size() != data.dim(2)) throw std::invalid_argument("ParameterDataset: TE count != L");
    for (std::size_t i = 0; i < tes_ms.size(); ++i)
      if (tes_ms[i] <= 0 || (i > 0 && tes_ms[i] <= tes_ms[i - 1]))
        throw std::invalid_argument("ParameterDataset: TEs must be positive and strictly increasing");
  }
  std::size_t fe() const { return data.dim(0); }
  std::size_t pe() const { return data.dim(1); }
  std::size_t echoes() const { return data.dim(2); }
  std::size_t coils() const { return data.dim(3); }
};

// Per-FE-slice reconstruction (iFFT along FE, then every slice's ADMM with
// its own early stop): all slices batched on the GPU.
inline ParameterDataset recon_param_dataset(const ParameterDataset& y, const SamplingMask& mask,
                                            const HankelConfig& hcfg, const AdmmConfig& acfg,
                                            std::ostream* log = nullptr, std::size_t* total_iters = nullptr) {
  y.validate();
  const std::size_t m = y.fe(), n = y.pe(), l = y.echoes(), j = y.coils();
  if (mask.rows != n || mask.cols != l) throw std::invalid_argument("recon_param_dataset: mask dims mismatch");
  acfg.validate();
  const shlr_param_args a = detail::param_args(y.data, m, n, l, j, mask, hcfg, acfg);
  ParameterDataset out;
  out.tes_ms = y.tes_ms;
  out.data = ComplexTensor({m, n, l, j});
  shlr_stats st{};
  const int rc =
      shlr_cuda_param_reconstruct(&a, reinterpret_cast<double*>(out.data.data()), &st,
                                  log ? detail::log_line : nullptr, log);
  if (total_iters) *total_iters = st.outer_iters;
  detail::check(rc, "recon_param_dataset");
  return out;
}

// FE slices [begin, end) of recon_param_dataset only (the slices are
// independent: parammap.cpp:37-51) -- the unit of work of one rank in a
// multi-GPU job.  Returns the end - begin reconstructed slices.
inline ParameterDataset recon_param_dataset_shard(const ParameterDataset& y, const SamplingMask& mask,
                                                  const HankelConfig& hcfg, const AdmmConfig& acfg,
                                                  std::size_t begin, std::size_t end, std::ostream* log = nullptr,
                                                  std::size_t* total_iters = nullptr) {
  y.validate();
  const std::size_t m = y.fe(), n = y.pe(), l = y.echoes(), j = y.coils();
  if (mask.rows != n || mask.cols != l) throw std::invalid_argument("recon_param_dataset: mask dims mismatch");
  if (begin > end || end > m) throw std::invalid_argument("recon_param_dataset: slice range outside the dataset");
  acfg.validate();
  if (begin == end) {  // empty shard (more ranks than FE slices): nothing to solve; the
                       // C-ABI reads slice range (0, 0) as "all slices", so it is not called
    if (total_iters) *total_iters = 0;
    ParameterDataset empty;
    empty.tes_ms = y.tes_ms;
    empty.data = ComplexTensor({0, n, l, j});
    return empty;
  }
  shlr_param_args a = detail::param_args(y.data, m, n, l, j, mask, hcfg, acfg);
  a.slice_begin = begin;
  a.slice_end = end;
  ParameterDataset out;
  out.tes_ms = y.tes_ms;
  out.data = ComplexTensor({end - begin, n, l, j});
  shlr_stats st{};
  const int rc =
      shlr_cuda_param_reconstruct(&a, reinterpret_cast<double*>(out.data.data()), &st,
                                  log ? detail::log_line : nullptr, log);
  if (total_iters) *total_iters = st.outer_iters;
  detail::check(rc, "recon_param_dataset");
  return out;
}

// Centred unitary FFT along one axis (fft.hpp:11-30), on the device.
inline ComplexTensor fft_along_axis(const ComplexTensor& x, std::size_t axis, bool inverse) {
  ComplexTensor out = x;
  detail::check(shlr_cuda_fft_along_axis(reinterpret_cast<double*>(out.data()), x.dims().data(),
                                         static_cast<int>(x.rank()), static_cast<int>(axis), inverse ? 1 : 0),
                "fft_along_axis");
  return out;
}

inline ComplexTensor ifft2d_centered(const ComplexTensor& x) {
  return fft_along_axis(fft_along_axis(x, 0, true), 1, true);
}
inline ComplexTensor fft2d_centered(const ComplexTensor& x) {
  return fft_along_axis(fft_along_axis(x, 0, false), 1, false);
}

}  // namespace shlr_b200
