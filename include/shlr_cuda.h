/*
 * shlr_cuda.h -- C-ABI boundary of the B200-native SHLR hot path.
 *
 * This is the drop-in boundary for the per-iteration separable-Hankel ADMM
 * step of arXiv 2107.11650's reference C++ library.  A maintainer keeps the
 * reference's public C++ API (proj/include/shlr/solvers.hpp) and replaces the
 * bodies of its solver entry points with calls into the functions below
 * (the C++ mirror in include/shlr_b200/ does exactly
 * that).  Plain pointers and sizes only -- no torch, no C++ types.
 *
 * Conventions (mirroring the reference):
 *   - complex data is interleaved (re, im) IEEE double, row-major, last
 *     dimension fastest, exactly as shlr::ComplexTensor stores
 *     std::complex<double> (proj/include/shlr/tensor.hpp:16-119);
 *   - masks are uint8 rows x cols, rows == 1 for line masks that broadcast
 *     along dim 0 (proj/include/shlr/sampling.hpp:33-52);
 *   - every call is synchronous with respect to the host, runs on its own
 *     stream/device state, and holds no global mutable state besides the
 *     last-error string (thread-local);
 *   - return codes: SHLR_OK, SHLR_EINVAL (-> std::invalid_argument),
 *     SHLR_EDIVERGE (-> shlr::DivergenceError), SHLR_ECUDA (CUDA failure,
 *     including "no device"), SHLR_EUNSUPPORTED (valid for the reference but
 *     outside what this build implements; never a silent CPU fallback).
 */
#ifndef SHLR_CUDA_H
#define SHLR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SHLR_OK 0
#define SHLR_EINVAL 1
#define SHLR_EDIVERGE 4
#define SHLR_ECUDA 5
#define SHLR_EUNSUPPORTED 6

#define SHLR_ABI_VERSION 1

/* Library/ABI identification. */
int shlr_cuda_abi_version(void);
/* Last error message of the calling thread ("" if none). */
const char* shlr_cuda_last_error(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int shlr_cuda_device_count(void);

/* Progress callback: one call per outer iteration with the exact text the
 * reference writes (proj/src/solvers.cpp:71-78, without the newline). */
typedef void (*shlr_log_fn)(void* ctx, const char* line);

typedef struct shlr_stats {
  size_t outer_iters;       /* SolveStats::outer_iters  (solvers.hpp:36-39) */
  double final_rel_change;  /* SolveStats::final_rel_change */
} shlr_stats;

/* Arguments of shlr_pi_reconstruct (proj/include/shlr/solvers.hpp:64-70)
 * after the host-side validation the reference does (solvers.cpp:101-123).
 * Pencils are already resolved with HankelConfig::pencil_for
 * (proj/src/hankel.cpp:10-18): pencil_row = pencil_for(N), pencil_col =
 * pencil_for(M). */
typedef struct shlr_pi_args {
  size_t m, n, j;              /* y is m x n x j                              */
  const double* y;             /* interleaved complex, m*n*j                  */
  const uint8_t* mask;         /* mask_rows x n                               */
  size_t mask_rows;            /* 1 (line mask) or m                          */
  const double* spirit_weights;/* k*k*j*j interleaved complex, the flat index
                                  of SpiritKernels::raw() (spirit.hpp:21-29),
                                  or NULL when enable_spirit == 0             */
  size_t spirit_k;             /* kernel size (odd)                           */
  const double* taps;          /* HankelConfig::filter_taps, interleaved      */
  size_t ntaps;
  size_t pencil_row, pencil_col;
  double lambda, lambda1, beta, tau, tol, cg_tol;
  size_t max_outer, cg_max;
  int enable_spirit, enable_vc;
  int debug_sv_iter;           /* >0: record singular values of L + D/beta at
                                  this 1-based outer iteration (parity hook)  */
} shlr_pi_args;

/* Full parallel-imaging reconstruction, host buffers in and out.
 * x_out: m*n*j interleaved complex (image domain, like the reference).
 * sv_out (optional, with debug_sv_iter > 0): (m + n) * d doubles, rows first
 * then columns, each row of d sorted descending, d = min(p, blocks*q) of that
 * direction (row and column matrices must then share d).  log_cb may be NULL. */
int shlr_cuda_pi_reconstruct(const shlr_pi_args* args, double* x_out,
                             double* sv_out, shlr_stats* stats,
                             shlr_log_fn log_cb, void* log_ctx);

/* Resident-plan API: the same computation split into setup / iterate /
 * download so that a caller (bench.py, a serving loop) keeps every buffer in
 * HBM.  plan_run executes `iters` outer iterations (bounded by max_outer and
 * the early-stop rule) on the plan's stream; it does not synchronise. */
typedef struct shlr_pi_plan shlr_pi_plan;
int shlr_cuda_pi_plan_create(const shlr_pi_args* args, shlr_pi_plan** out);
int shlr_cuda_pi_plan_reset(shlr_pi_plan* plan);          /* back to iteration 0 */
int shlr_cuda_pi_plan_run(shlr_pi_plan* plan, size_t iters);
int shlr_cuda_pi_plan_sync(shlr_pi_plan* plan);
/* Device time (ms) of the Hankel-SVT kernel over the last plan_run call
 * (CUDA events on the plan's stream; 0 if not measured). */
int shlr_cuda_pi_plan_timing(shlr_pi_plan* plan, double* svt_ms, double* total_ms,
                             int* launches_per_iter);
/* Timing mode: plan_run launches kernels directly (no CUDA graph) and times
 * the Hankel-SVT launch of every iteration with CUDA events. */
int shlr_cuda_pi_plan_set_timing(shlr_pi_plan* plan, int on);
/* Eigen-solver warm start across outer iterations (default on): each row /
 * column matrix starts its Jacobi refinement from the eigenvectors it had in
 * the previous iteration.  The result is the same spectral function either
 * way; only the sweep count changes. */
int shlr_cuda_pi_plan_set_warm_start(shlr_pi_plan* plan, int on);
/* Diagnostics: Jacobi sweeps (stage1 * 100 + stage2) per matrix of the last
 * Hankel-SVT launch, rows first then columns; n = m + n entries. */
int shlr_cuda_pi_plan_debug_sweeps(shlr_pi_plan* plan, int* out, int n);
/* Diagnostics: the solver level each lifted matrix ended the last outer
 * iteration at, rows first then columns; n = m + n entries.  0: level 1;
 * 1: handed to the next level and redone there; 2: beyond the last level's
 * block (d > 128 without a deflation buffer: reported on download); 3: kept
 * at level 2; 4 / 5: large d, solved by the deflation chain (4 only while a
 * chain is in flight). */
int shlr_cuda_pi_plan_debug_levels(shlr_pi_plan* plan, int* out, int n);
/* Diagnostics: per-matrix clock64 stamps of the subspace solver's phases
 * (8 per matrix) of the last launch; zeros unless SHLR_PHASE_CLK was set in
 * the environment when the plan was created. */
int shlr_cuda_pi_plan_debug_phases(shlr_pi_plan* plan, long long* out, int n);
int shlr_cuda_pi_plan_download(shlr_pi_plan* plan, double* x_out, shlr_stats* stats,
                               shlr_log_fn log_cb, void* log_ctx);
void shlr_cuda_pi_plan_destroy(shlr_pi_plan* plan);

/* ------------------------------------------------------------------------
 * Parameter imaging (SHLR-P / SHLR-VP, Algorithm S2).
 *
 * Arguments of shlr_param_reconstruct_slice (proj/include/shlr/solvers.hpp:74-79)
 * and recon_param_dataset (proj/include/shlr/parammap.hpp:35-40) after the
 * host-side validation the reference does (solvers.cpp:199-206,
 * parammap.cpp:27-30).  Pencils are resolved with HankelConfig::pencil_for(n)
 * and HankelConfig::pencil_for_param(l) (proj/src/hankel.cpp:10-29).
 *   m == 0: y is one N x L x J slice (FE image, PE k-space), the input of
 *           shlr_param_reconstruct_slice;
 *   m >= 1: y is an M x N x L x J dataset (k-space in FE and PE), the input
 *           of recon_param_dataset: iFFT along FE, then every FE slice is an
 *           independent ADMM with its own early stop -- all of them run
 *           batched on the device.
 * mask is N x L (row = phase encode, column = echo). */
typedef struct shlr_param_args {
  size_t m, n, l, j;
  const double* y;             /* interleaved complex                          */
  const uint8_t* mask;         /* n x l                                        */
  const double* taps;          /* HankelConfig::filter_taps, interleaved       */
  size_t ntaps;
  size_t pencil_pe, pencil_par;
  double lambda, lambda2, beta, tau, tol, cg_tol;
  size_t max_outer, cg_max;
  int enable_vc;
  /* Dataset mode only: solve FE slices [slice_begin, slice_end) of the M
   * (the FE transform still runs over all M lines); x_out then holds
   * slice_end - slice_begin slices.  0, 0 = all.  The slices are independent
   * problems (parammap.cpp:37-51): ranks of a multi-GPU job each take a range,
   * with no collective. */
  size_t slice_begin, slice_end;
  /* Dataset mode only: 1 = y is already the hybrid (FE image, PE k-space) the
   * reference's recon_param_dataset computes first (fft_along_axis(y, 0,
   * inverse), parammap.cpp:32): the device skips its FE transform.  A caller
   * that keeps the reference's own host FFT for that setup step (the drop-in,
   * dropin/shlr_dropin.cpp) gets per-slice results bitwise equal to
   * shlr_param_reconstruct_slice on the same hybrid planes. */
  int hybrid_input;
} shlr_param_args;

/* Full parameter reconstruction, host buffers in and out.  x_out: (m ? m : 1)
 * x n x l x j interleaved complex (image domain along FE and PE, like the
 * reference).  stats (nullable): for a slice, SolveStats of the slice; for a
 * dataset, outer_iters = total outer iterations over all slices (the
 * reference's *total_iters, parammap.cpp:52) and final_rel_change of the last
 * slice.  log_cb receives every slice's per-iteration lines in slice order. */
int shlr_cuda_param_reconstruct(const shlr_param_args* args, double* x_out, shlr_stats* stats,
                                shlr_log_fn log_cb, void* log_ctx);

/* Resident-plan API of the parameter path (same contract as the PI plan). */
typedef struct shlr_param_plan shlr_param_plan;
int shlr_cuda_param_plan_create(const shlr_param_args* args, shlr_param_plan** out);
int shlr_cuda_param_plan_reset(shlr_param_plan* plan);
int shlr_cuda_param_plan_run(shlr_param_plan* plan, size_t iters);
int shlr_cuda_param_plan_sync(shlr_param_plan* plan);
int shlr_cuda_param_plan_set_timing(shlr_param_plan* plan, int on);
int shlr_cuda_param_plan_timing(shlr_param_plan* plan, double* svt_ms, double* total_ms,
                                int* launches_per_iter);
int shlr_cuda_param_plan_download(shlr_param_plan* plan, double* x_out, shlr_stats* stats,
                                  shlr_log_fn log_cb, void* log_ctx);
void shlr_cuda_param_plan_destroy(shlr_param_plan* plan);

/* Batched Hankel-SVT unit (BASELINE config 5): for each of `batch` matrices,
 * lift_plain (proj/src/operators.cpp:93-103) the nc vectors of length n with
 * pencil p, svt with threshold tau (solvers.cpp:11-21), adjoint_lift_plain
 * (operators.cpp:105-119).  All pointers are DEVICE pointers to complex64
 * (float2) data: vecs and out are batch x nc x n; sv_out (nullable) is
 * batch x d floats, descending.  stream is a cudaStream_t (NULL = default).
 * out must not overlap vecs (SHLR_EINVAL): tall large-d lifts accumulate the
 * adjoint in the zeroed output while the lift source is still being read. */
int shlr_cuda_hankel_svt_batched(const void* vecs, int batch, int nc, int n, int p,
                                 float tau, void* out, float* sv_out, void* stream);
/* Same, host complex128 buffers in and out (the e2e path). */
int shlr_cuda_hankel_svt_batched_host(const double* vecs, int batch, int nc, int n, int p,
                                      double tau, double* out, double* sv_out);

/* Test hook: the X-update operator of shlr_pi_reconstruct alone, out = A x
 * with A the reference's normal_apply (proj/src/operators.cpp:213-248) for
 * the configuration in args (mask, taps, pencils, virtual coils, lambda,
 * lambda1, beta, SPIRiT kernels), evaluated by the device's k-space operator
 * (exact diagonal + F2D P F2D^-1).  x_img and out_img: m x n x j interleaved
 * complex, image domain. */
int shlr_cuda_debug_normal_apply(const shlr_pi_args* args, const double* x_img, double* out_img);

/* Diagnostics: the device-pointer batched SVT that also writes, per matrix,
 * the number of Jacobi sweeps the eigen-solver used (sweeps_dev: device int
 * array of batch entries). */
int shlr_cuda_debug_svt_sweeps(const void* vecs, int batch, int nc, int n, int p, float tau,
                               void* out, int* sweeps_dev);

/* Hankel lift index map used by the device kernels, for bit-exact parity of
 * the lift (operators.cpp:25-58, hankel.cpp:31-41,99-113).  For a p x
 * (blocks*q) matrix built from `coils` vectors of length n (blocks = coils *
 * (vc ? 2 : 1)), writes for every element (i, c), row-major, three int32:
 * source coil, source index into that coil's spectrum, conj flag (1 for the
 * conjugate-flipped virtual-coil blocks).  map must hold p*blocks*q*3 ints.
 * Computed by running the kernels' own lift stage (spectra staging, offset
 * table, chunk builder) on index-encoded spectra s_j[n] = (j+1) + i(n+1) with
 * unit weights and decoding the lifted elements: path 0 = the full solver's
 * load_chunk / lift_elem, 1 = the subspace solver's build_chunk / lift_tab,
 * 2 = the large-d variants' build_chunk_big / lift_global (d <= 256 here).
 * shlr_cuda_lift_index_map is path 1. */
int shlr_cuda_lift_index_map(int n, int p, int coils, int vc, int32_t* map);
int shlr_cuda_lift_index_map_path(int n, int p, int coils, int vc, int path, int32_t* map);

/* Centered unitary FFT along one axis of a host complex128 tensor
 * (proj/src/fft.cpp:100-128), computed on the device in complex64.
 * dims has ndim entries; data is transformed in place. */
int shlr_cuda_fft_along_axis(double* data, const size_t* dims, int ndim, int axis,
                             int inverse);

/* Measured FP32 CUDA-core peak of the current device (TFLOP/s): a
 * register-resident FMA chain over all SMs, timed with CUDA events.  Used as
 * the roofline denominator of the FP32 Hankel-SVT kernel. */
int shlr_cuda_fp32_peak_tflops(double* tflops);

/* Image-quality metrics on the device in FP64, host
 * buffers in and out, synchronous.
 *   shlr_cuda_ssos   -- ssos (proj/src/io.cpp:105-117): x is m x n x j
 *                       interleaved complex, out m x n; bitwise the reference's
 *                       (same operation order, round-to-nearest, no FMA).
 *   shlr_cuda_rlne   -- rlne (proj/src/metrics.cpp:9-21) over `count` pixels;
 *                       SHLR_EINVAL for an identically zero reference.
 *   shlr_cuda_mssim  -- mssim (metrics.cpp:23-75): mean SSIM over all 11 x 11
 *                       Gaussian windows (sigma 1.5), C1/C2 from max(ref);
 *                       SHLR_EINVAL for an image smaller than the window.
 * The dimension checks of the reference's callers (RealImage shapes) stay on
 * the host; the final sums are deterministic tree reductions. */
int shlr_cuda_ssos(const double* x, size_t m, size_t n, size_t j, double* out);
int shlr_cuda_rlne(const double* ref, const double* rec, size_t count, double* out);
int shlr_cuda_mssim(const double* ref, const double* rec, size_t rows, size_t cols, double* out);

/* Host-side helpers of the boundary (no GPU needed): the reference's mask
 * generators (proj/src/sampling.cpp:31-173), bit-exact. */
int shlr_mask_gauss_cartesian(size_t n, double rate, size_t acs, uint64_t seed,
                              uint8_t* bits_out);
int shlr_mask_random2d(size_t rows, size_t cols, double rate, size_t center,
                       uint64_t seed, uint8_t* bits_out);
int shlr_acs_range(size_t n, size_t acs, size_t* start, size_t* end);
size_t shlr_pencil_for(size_t pencil, size_t len);
/* HankelConfig::pencil_for_param (proj/src/hankel.cpp:20-29); 0 = invalid. */
size_t shlr_pencil_for_param(size_t pencil_param, size_t len);
/* SPIRiT kernel calibration (proj/src/spirit.cpp:22-94) on an a x b x j ACS
 * block (interleaved complex, row-major): the Tikhonov filter
 * s / (s^2 + mu^2), mu = tikhonov * s_max, computed as the equivalent ridge
 * solve in FP64 on the host.  weights_out: k*k*j*j interleaved complex in
 * SpiritKernels::raw() order.  Setup only (not on the per-iteration path). */
int shlr_spirit_calibrate(const double* acs, size_t a, size_t b, size_t j, size_t k,
                          double tikhonov, double* weights_out);

/* The same calibration on the device in FP64: the
 * augmented patch-matrix Gram in tiles, then per target coil the power
 * iteration for s_max^2, the ridge shift and a Cholesky solve -- the
 * restatement shlr_spirit_calibrate runs on the host.  Same arguments and
 * result layout; SHLR_ECUDA without a device. */
int shlr_cuda_spirit_calibrate(const double* acs, size_t a, size_t b, size_t j, size_t k,
                               double tikhonov, double* weights_out);

#ifdef __cplusplus
}
#endif

#endif /* SHLR_CUDA_H */
