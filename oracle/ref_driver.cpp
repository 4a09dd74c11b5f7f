// ref_driver: a command-line driver over the REFERENCE library's own public
// API (proj/include/shlr/*.hpp), linked against the unmodified reference
// sources built by oracle/Makefile.  TEST INFRASTRUCTURE ONLY: it generates
// golden outputs for the parity tests and times the reference CPU path for
// bench.py's cpu_baseline / --impl reference leg.  It never runs inside the
// product path.
//
// Usage: ref_driver <mode> key=value ...
//   pi     y= mask= out= [kernels=] [spirit=0] [vc=0] [pencil=0] [acs=0]
//          [kernel=5] [tikhonov=1e-4] [max_outer=50] [tol=1e-6] [lambda=1e4]
//          [lambda1=1e2] [beta=1] [tau=1] [cg_max=15] [cg_tol=1e-8]
//          [sv_iters=] (comma list of 1-based iterations whose singular values
//          of L + D/beta are dumped; uses the instrumented replay below)
//          [x_iters=] (comma list of 1-based iterations whose image x is
//          dumped to out.x<k>.cplx; also uses the replay)
//          [replay=0] [time=0]  (time=1 without the replay: the stock
//          shlr_pi_reconstruct timed per iteration through its log lines)
//   param  y= mask= out= [vc=0] [pencil=0] [pencil_param=0] ...admm keys
//          (y is N x L x J -> shlr_param_reconstruct_slice, or M x N x L x J
//          -> recon_param_dataset)
//   svt    vecs= p= tau= out= [time=0] [limit=0]
//          vecs is B x Nc x N: lift_plain -> svt -> adjoint_lift_plain per
//          matrix (solvers.cpp:264-268,280-282 composition)
//   mask   kind=gauss|random2d|uniform n= [m=] rate= acs= seed= out=
//   calib  y= mask= acs= [kernel=5] [tikhonov=1e-4] out=
//   metrics [x= (M x N x J) -> out.ssos.cplx] [ref= rec= (real, rank 2) -> rlne / mssim on stdout]
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <Eigen/SVD>

#include "shlr/fft.hpp"
#include "shlr/hankel.hpp"
#include "shlr/io.hpp"
#include "shlr/metrics.hpp"
#include "shlr/operators.hpp"
#include "shlr/parammap.hpp"
#include "shlr/sampling.hpp"
#include "shlr/solvers.hpp"
#include "shlr/spirit.hpp"

using namespace shlr;

namespace {

using Args = std::map<std::string, std::string>;

std::string get(const Args& a, const std::string& k, const std::string& def = "") {
  auto it = a.find(k);
  if (it == a.end()) {
    if (def == "\x01") throw std::invalid_argument("missing argument " + k);
    return def;
  }
  return it->second;
}
double getd(const Args& a, const std::string& k, double def) {
  auto s = get(a, k);
  return s.empty() ? def : std::stod(s);
}
std::size_t getu(const Args& a, const std::string& k, std::size_t def) {
  auto s = get(a, k);
  return s.empty() ? def : static_cast<std::size_t>(std::stoull(s));
}

double g_t0 = 0.0;

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

AdmmConfig admm_from(const Args& a) {
  AdmmConfig c;
  c.lambda = getd(a, "lambda", c.lambda);
  c.lambda1 = getd(a, "lambda1", c.lambda1);
  c.lambda2 = getd(a, "lambda2", c.lambda2);
  c.beta = getd(a, "beta", c.beta);
  c.tau = getd(a, "tau", c.tau);
  c.max_outer = getu(a, "max_outer", c.max_outer);
  c.tol = getd(a, "tol", c.tol);
  c.cg_max = getu(a, "cg_max", c.cg_max);
  c.cg_tol = getd(a, "cg_tol", c.cg_tol);
  c.enable_spirit = getu(a, "spirit", 0) != 0;
  c.enable_vc = getu(a, "vc", 0) != 0;
  return c;
}

HankelConfig hankel_from(const Args& a) {
  HankelConfig h;
  h.pencil = getu(a, "pencil", 0);
  h.pencil_param = getu(a, "pencil_param", 0);
  return h;
}

void write_sv(const std::vector<std::vector<double>>& rows, const std::string& path) {
  std::size_t width = 0;
  for (auto& r : rows) width = std::max(width, r.size());
  ComplexTensor t({rows.size(), std::max<std::size_t>(width, 1)});
  for (std::size_t i = 0; i < rows.size(); ++i)
    for (std::size_t k = 0; k < rows[i].size(); ++k) t.at(i, k) = cplx{rows[i][k], 0};
  write_cplx(t, path);
}

std::vector<double> singular_values(const CMatrix& m) {
  Eigen::JacobiSVD<CMatrix> svd(m);
  const auto& s = svd.singularValues();
  std::vector<double> out(static_cast<std::size_t>(s.size()));
  for (Eigen::Index i = 0; i < s.size(); ++i) out[static_cast<std::size_t>(i)] = s(i);
  return out;
}

SpiritKernels calibrate_from(const ComplexTensor& y_masked, std::size_t acs,
                             std::size_t kernel, double tikhonov) {
  // ACS block = all rows x acs_range(N, acs) columns (shlr_cli.cpp:390-396).
  auto [a0, a1] = acs_range(y_masked.dim(1), acs);
  ComplexTensor block({y_masked.dim(0), a1 - a0, y_masked.dim(2)});
  for (std::size_t r = 0; r < y_masked.dim(0); ++r)
    for (std::size_t c = a0; c < a1; ++c)
      for (std::size_t j = 0; j < y_masked.dim(2); ++j)
        block.at(r, c - a0, j) = y_masked.at(r, c, j);
  return spirit_calibrate(block, kernel, tikhonov);
}

SpiritKernels read_kernels(const std::string& path) {
  ComplexTensor t = read_cplx(path);
  if (t.rank() != 4 || t.dim(0) != t.dim(1) || t.dim(2) != t.dim(3))
    throw std::invalid_argument("kernels file must be k x k x J x J");
  std::vector<cplx> w(t.data(), t.data() + t.size());
  return SpiritKernels(t.dim(0), t.dim(2), std::move(w));
}

void write_kernels(const SpiritKernels& g, const std::string& path) {
  const std::size_t k = g.kernel_size(), j = g.coils();
  ComplexTensor t({k, k, j, j}, g.raw());
  write_cplx(t, path);
}

// Instrumented replay of shlr_pi_reconstct's loop (solvers.cpp:95-191) built
// from the same public primitives in the same order, so it is bitwise equal
// to the library call; it additionally dumps the singular values of
// L + D/beta (the SVT input) at the requested iterations.
ComplexTensor pi_replay(const ComplexTensor& y, const SamplingMask& mask,
                        const SpiritKernels* g, const HankelConfig& hcfg,
                        const AdmmConfig& acfg, std::ostream* log, SolveStats* stats,
                        const std::vector<std::size_t>& sv_iters,
                        const std::string& sv_prefix, bool print_times = false,
                        const std::vector<std::size_t>& x_iters = {}) {
  acfg.validate();
  const std::size_t m = y.dim(0), n = y.dim(1), j = y.dim(2);
  HankelConfig cfg = hcfg;
  cfg.virtual_coil = acfg.enable_vc;
  const std::size_t p_row = cfg.pencil_for(n);
  const std::size_t p_col = cfg.pencil_for(m);
  const std::size_t blocks = j * (acfg.enable_vc ? 2 : 1);
  std::optional<SpiritImageOp> gop;
  const double lambda1 = acfg.enable_spirit ? acfg.lambda1 : 0.0;
  if (acfg.enable_spirit && lambda1 > 0.0) gop.emplace(*g, m, n);
  const ComplexTensor y_masked = apply_mask(y, mask);
  const ComplexTensor fid_rhs = ifft2d_centered(y_masked);
  std::vector<CMatrix> z_row(m), d_row(m), z_col(n), d_col(n);
  for (std::size_t r = 0; r < m; ++r) {
    z_row[r] = CMatrix::Zero(static_cast<Eigen::Index>(p_row),
                             static_cast<Eigen::Index>(blocks * (n - p_row + 1)));
    d_row[r] = CMatrix::Ones(z_row[r].rows(), z_row[r].cols());
  }
  for (std::size_t c = 0; c < n; ++c) {
    z_col[c] = CMatrix::Zero(static_cast<Eigen::Index>(p_col),
                             static_cast<Eigen::Index>(blocks * (m - p_col + 1)));
    d_col[c] = CMatrix::Ones(z_col[c].rows(), z_col[c].cols());
  }
  ComplexTensor x = ifft2d_centered(y_masked);
  const double beta = acfg.beta;
  const auto apply_a = [&](const ComplexTensor& v) {
    return normal_apply(v, mask, gop ? &*gop : nullptr, cfg, acfg.lambda, lambda1, beta);
  };
  std::size_t iters = 0;
  double relchange = 1.0;
  const std::vector<std::size_t> dims = {m, n, j};
  if (print_times) std::printf("setup_seconds=%.6f\n", now_s() - g_t0);
  for (std::size_t k = 0; k < acfg.max_outer; ++k) {
    const double t_it = now_s();
    ComplexTensor b({m, n, j});
    b += fid_rhs;
    b *= cplx{acfg.lambda, 0};
    for (std::size_t r = 0; r < m; ++r) {
      CMatrix t = z_row[r] - d_row[r] / beta;
      ComplexTensor adj = adjoint_lift_rows(t, dims, r, cfg);
      adj *= cplx{beta, 0};
      b += adj;
    }
    for (std::size_t c = 0; c < n; ++c) {
      CMatrix t = z_col[c] - d_col[c] / beta;
      ComplexTensor adj = adjoint_lift_cols(t, dims, c, cfg);
      adj *= cplx{beta, 0};
      b += adj;
    }
    CgResult cg;
    ComplexTensor x_new = cg_solve(apply_a, b, x, acfg.cg_max, acfg.cg_tol, &cg);
    const bool dump = std::find(sv_iters.begin(), sv_iters.end(), k + 1) != sv_iters.end();
    std::vector<std::vector<double>> svs;
    for (std::size_t r = 0; r < m; ++r) {
      CMatrix lifted = lift_rows(x_new, r, cfg);
      if (dump) svs.push_back(singular_values(lifted + d_row[r] / beta));
      z_row[r] = svt(lifted + d_row[r] / beta, 1.0 / beta);
      d_row[r] += acfg.tau * (lifted - z_row[r]);
    }
    for (std::size_t c = 0; c < n; ++c) {
      CMatrix lifted = lift_cols(x_new, c, cfg);
      if (dump) svs.push_back(singular_values(lifted + d_col[c] / beta));
      z_col[c] = svt(lifted + d_col[c] / beta, 1.0 / beta);
      d_col[c] += acfg.tau * (lifted - z_col[c]);
    }
    if (dump) write_sv(svs, sv_prefix + ".sv" + std::to_string(k + 1) + ".cplx");
    if (std::find(x_iters.begin(), x_iters.end(), k + 1) != x_iters.end())
      write_cplx(x_new, sv_prefix + ".x" + std::to_string(k + 1) + ".cplx");
    // rel_change_sq (solvers.cpp:80-87)
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < x_new.size(); ++i) {
      num += std::norm(x_new[i] - x[i]);
      den += std::norm(x[i]);
    }
    relchange = den > 0.0 ? num / den : (num > 0.0 ? 1.0 : 0.0);
    if (print_times) {
      std::printf("iter_seconds=%.6f\n", now_s() - t_it);
      std::fflush(stdout);
    }
    x = std::move(x_new);
    iters = k + 1;
    if (log)
      (*log) << "iter=" << iters << " relchange=" << std::scientific
             << std::setprecision(3) << relchange << " cg_iters=" << cg.iterations
             << " cg_res=" << cg.relative_residual << "\n"
             << std::defaultfloat;
    if (relchange < acfg.tol) break;
  }
  if (stats) *stats = {iters, relchange};
  return x;
}

// Log sink that stamps every line the STOCK shlr_pi_reconstruct writes
// (solvers.cpp:71-78, one line per outer iteration): prints
// first_iter_seconds= (call start -> first line, includes the solver's setup)
// and then iter_seconds= per further iteration, so the unmodified library
// call is timed per iteration without replaying its loop.
class StampBuf : public std::streambuf {
 public:
  StampBuf(std::streambuf* sink, double t0) : sink_(sink), last_(t0) {}

 protected:
  int overflow(int c) override {
    if (c == traits_type::eof()) return traits_type::not_eof(c);
    if (sink_->sputc(static_cast<char>(c)) == traits_type::eof()) return traits_type::eof();
    if (c == '\n') {
      const double t = now_s();
      std::printf("%s=%.6f\n", first_ ? "first_iter_seconds" : "iter_seconds", t - last_);
      std::fflush(stdout);
      first_ = false;
      last_ = t;
    }
    return c;
  }
  int sync() override { return sink_->pubsync(); }

 private:
  std::streambuf* sink_;
  double last_;
  bool first_ = true;
};

std::vector<std::size_t> parse_list(const std::string& s) {
  std::vector<std::size_t> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(static_cast<std::size_t>(std::stoull(item)));
  return out;
}

void write_stats(const std::string& path, const SolveStats& st, double secs) {
  std::ofstream os(path);
  os << std::setprecision(17) << "outer_iters=" << st.outer_iters << "\n"
     << "final_rel_change=" << st.final_rel_change << "\n"
     << "seconds=" << secs << "\n";
}

int cmd_pi(const Args& a) {
  ComplexTensor y = read_cplx(get(a, "y", "\x01"));
  SamplingMask mask = read_mask(get(a, "mask", "\x01"));
  const std::string out = get(a, "out", "\x01");
  AdmmConfig acfg = admm_from(a);
  HankelConfig hcfg = hankel_from(a);
  ComplexTensor ym = apply_mask(y, mask);
  SpiritKernels g;
  if (acfg.enable_spirit) {
    if (!get(a, "kernels").empty()) {
      g = read_kernels(get(a, "kernels"));
    } else {
      const std::size_t acs = getu(a, "acs", mask.acs);
      g = calibrate_from(ym, acs, getu(a, "kernel", 5), getd(a, "tikhonov", 1e-4));
      write_kernels(g, out + ".kernels.cplx");
    }
  }
  const auto sv_iters = parse_list(get(a, "sv_iters"));
  const auto x_iters = parse_list(get(a, "x_iters"));
  std::ofstream log(out + ".log");
  SolveStats st;
  const double t0 = now_s();
  g_t0 = t0;
  const bool replay = !sv_iters.empty() || !x_iters.empty() || getu(a, "replay", 0);
  // stock call timed per iteration through its own log lines (time=1)
  StampBuf stamp(log.rdbuf(), t0);
  std::ostream stamped(&stamp);
  std::ostream* log_out = (!replay && getu(a, "time", 0)) ? &stamped : &log;
  ComplexTensor x =
      replay ? pi_replay(ym, mask, acfg.enable_spirit ? &g : nullptr, hcfg, acfg, &log, &st,
                         sv_iters, out, getu(a, "time", 0) != 0, x_iters)
             : shlr_pi_reconstruct(ym, mask, acfg.enable_spirit ? &g : nullptr, hcfg, acfg,
                                   log_out, &st);
  log_out->flush();
  const double secs = now_s() - t0;
  write_cplx(x, out + ".x.cplx");
  write_stats(out + ".stats", st, secs);
  if (getu(a, "time", 0))
    std::printf("pi seconds=%.6f iters=%zu\n", secs, st.outer_iters);
  return 0;
}

int cmd_param(const Args& a) {
  ComplexTensor y = read_cplx(get(a, "y", "\x01"));
  SamplingMask mask = read_mask(get(a, "mask", "\x01"));
  const std::string out = get(a, "out", "\x01");
  AdmmConfig acfg = admm_from(a);
  HankelConfig hcfg = hankel_from(a);
  std::ofstream log(out + ".log");
  const double t0 = now_s();
  if (y.rank() == 3) {
    SolveStats st;
    ComplexTensor x = shlr_param_reconstruct_slice(y, mask, hcfg, acfg, &log, &st);
    write_cplx(x, out + ".x.cplx");
    write_stats(out + ".stats", st, now_s() - t0);
  } else {
    ParameterDataset ds;
    ds.data = y;
    for (std::size_t e = 0; e < y.dim(2); ++e) ds.tes_ms.push_back(10.0 * static_cast<double>(e + 1));
    std::size_t total = 0;
    ParameterDataset rec = recon_param_dataset(ds, mask, hcfg, acfg, &log, &total);
    write_cplx(rec.data, out + ".x.cplx");
    write_stats(out + ".stats", SolveStats{total, 0.0}, now_s() - t0);
  }
  if (getu(a, "time", 0)) std::printf("param seconds=%.6f\n", now_s() - t0);
  return 0;
}

int cmd_svt(const Args& a) {
  ComplexTensor v = read_cplx(get(a, "vecs", "\x01"));
  if (v.rank() != 3) throw std::invalid_argument("vecs must be B x Nc x N");
  const std::size_t bsz = v.dim(0), nc = v.dim(1), n = v.dim(2);
  const std::size_t p = getu(a, "p", 0);
  const double tau = getd(a, "tau", 1.0);
  const std::size_t limit = getu(a, "limit", 0);
  const std::size_t nb = limit ? std::min(limit, bsz) : bsz;
  const std::string out = get(a, "out");
  ComplexTensor adj({nb, nc, n});
  std::vector<std::vector<double>> svs;
  const double t0 = now_s();
  double t_svt = 0;
  for (std::size_t b = 0; b < nb; ++b) {
    std::vector<std::vector<cplx>> vecs(nc, std::vector<cplx>(n));
    for (std::size_t c = 0; c < nc; ++c)
      for (std::size_t i = 0; i < n; ++i) vecs[c][i] = v.at(b, c, i);
    CMatrix l = lift_plain(vecs, p);
    const double ts = now_s();
    CMatrix z = svt(l, tau);
    t_svt += now_s() - ts;
    auto back = adjoint_lift_plain(z, n, nc);
    for (std::size_t c = 0; c < nc; ++c)
      for (std::size_t i = 0; i < n; ++i) adj.at(b, c, i) = back[c][i];
    if (!out.empty()) svs.push_back(singular_values(l));
  }
  const double secs = now_s() - t0;
  if (!out.empty()) {
    write_cplx(adj, out + ".adj.cplx");
    write_sv(svs, out + ".sv.cplx");
  }
  if (getu(a, "time", 0))
    std::printf("svt matrices=%zu seconds=%.6f svt_seconds=%.6f\n", nb, secs, t_svt);
  return 0;
}

int cmd_mask(const Args& a) {
  const std::string kind = get(a, "kind", "gauss");
  const std::size_t n = getu(a, "n", 0);
  SamplingMask m;
  if (kind == "gauss")
    m = mask_gauss_cartesian(n, getd(a, "rate", 0.25), getu(a, "acs", 0), getu(a, "seed", 0));
  else if (kind == "random2d")
    m = mask_random2d(getu(a, "m", n), n, getd(a, "rate", 0.25), getu(a, "acs", 0),
                      getu(a, "seed", 0));
  else if (kind == "uniform")
    m = mask_uniform(n, getu(a, "r", 1), getu(a, "acs", 0));
  else
    throw std::invalid_argument("unknown mask kind " + kind);
  write_mask(m, get(a, "out", "\x01"));
  return 0;
}

// x= (M x N x J) -> out.ssos.cplx; with ref= and rec= (real images stored as
// rank-2 .cplx): rlne and mssim printed with 17 digits
int cmd_metrics(const Args& a) {
  const std::string out = get(a, "out");
  if (!get(a, "x").empty()) {
    RealImage s = ssos(read_cplx(get(a, "x")));
    ComplexTensor t({s.rows(), s.cols()});
    for (std::size_t i = 0; i < s.size(); ++i) t[i] = cplx{s[i], 0.0};
    write_cplx(t, out + ".ssos.cplx");
  }
  if (!get(a, "ref").empty()) {
    auto to_real = [](const ComplexTensor& t) {
      RealImage r(t.dim(0), t.dim(1));
      for (std::size_t i = 0; i < r.size(); ++i) r[i] = t[i].real();
      return r;
    };
    RealImage ref = to_real(read_cplx(get(a, "ref"))), rec = to_real(read_cplx(get(a, "rec", "\x01")));
    std::printf("rlne=%.17g\nmssim=%.17g\n", rlne(ref, rec), mssim(ref, rec));
  }
  return 0;
}

int cmd_calib(const Args& a) {
  ComplexTensor y = read_cplx(get(a, "y", "\x01"));
  SamplingMask mask = read_mask(get(a, "mask", "\x01"));
  ComplexTensor ym = apply_mask(y, mask);
  SpiritKernels g = calibrate_from(ym, getu(a, "acs", mask.acs), getu(a, "kernel", 5),
                                   getd(a, "tikhonov", 1e-4));
  write_kernels(g, get(a, "out", "\x01"));
  return 0;
}

} // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver pi|param|svt|mask|calib key=value...\n");
    return 3;
  }
  Args a;
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    auto eq = s.find('=');
    if (eq == std::string::npos) {
      std::fprintf(stderr, "bad argument %s\n", argv[i]);
      return 3;
    }
    a[s.substr(0, eq)] = s.substr(eq + 1);
  }
  const std::string mode = argv[1];
  try {
    if (mode == "pi") return cmd_pi(a);
    if (mode == "param") return cmd_param(a);
    if (mode == "svt") return cmd_svt(a);
    if (mode == "mask") return cmd_mask(a);
    if (mode == "calib") return cmd_calib(a);
    if (mode == "metrics") return cmd_metrics(a);
    std::fprintf(stderr, "unknown mode %s\n", mode.c_str());
    return 3;
  } catch (const DivergenceError& e) {
    std::fprintf(stderr, "divergence: %s\n", e.what());
    return 4;
  } catch (const IoError& e) {
    std::fprintf(stderr, "io: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
