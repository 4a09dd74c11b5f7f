"""Python mirror of the reference's reconstruction API over the C-ABI.

Same names, argument meaning and error behaviour as ``proj/include/shlr``:

* ``HankelConfig``   -- ``hankel.hpp:15-25`` (``pencil_for``: ``hankel.cpp:10-18``)
* ``AdmmConfig``     -- ``solvers.hpp:16-34`` (``validate``: ``:29-33``)
* ``SamplingMask``   -- ``sampling.hpp:33-52``
* ``SpiritKernels``  -- ``spirit.hpp:12-36`` (weights ``(k, k, J, J)`` =
  the flat index ``((di+h)*k + (dj+h))*J + src)*J + dst``)
* ``shlr_pi_reconstruct`` -- ``solvers.hpp:64-70``; raises ``ValueError``
  where the reference throws ``std::invalid_argument`` and
  ``DivergenceError`` for ``shlr::DivergenceError``.
* ``shlr_param_reconstruct_slice`` -- ``solvers.hpp:74-79`` and
  ``recon_param_dataset`` / ``ParameterDataset`` -- ``parammap.hpp:11-40``
  (all FE slices of a dataset run batched on the device).
* ``hankel_svt_batched`` -- the config-5 lift_plain -> svt -> adjoint unit.

Everything numerical runs in ``lib/libshlr_b200.so`` on the GPU; this module
only marshals arrays.  Complex inputs are complex128 (the reference's
``std::complex<double>``); the device computes in complex64.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from ._lib import (LOG_FN, SHLR_EDIVERGE, SHLR_EINVAL, SHLR_EUNSUPPORTED, SHLR_OK, ShlrParamArgs,
                   ShlrPiArgs, ShlrStats, last_error, lib)


class DivergenceError(RuntimeError):
    """``shlr::DivergenceError`` (``solvers.hpp:41-43``)."""


class CudaError(RuntimeError):
    """CUDA failure or no device (the product path has no CPU fallback)."""


def _check(rc: int, what: str) -> None:
    if rc == SHLR_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == SHLR_EINVAL:
        raise ValueError(msg)
    if rc == SHLR_EDIVERGE:
        raise DivergenceError(msg)
    if rc == SHLR_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise CudaError(msg)


def device_count() -> int:
    return int(lib.shlr_cuda_device_count())


@dataclass
class HankelConfig:
    pencil: int = 0
    pencil_param: int = 0
    filter_taps: Sequence[complex] = (1.0 + 0j, -1.0 + 0j)
    virtual_coil: bool = False

    def pencil_for(self, length: int) -> int:
        p = int(lib.shlr_pencil_for(self.pencil, length))
        if p == 0:
            raise ValueError("HankelConfig: pencil exceeds signal length")
        return p

    def pencil_for_param(self, length: int) -> int:
        p = int(lib.shlr_pencil_for_param(self.pencil_param, length))
        if p == 0:
            raise ValueError("HankelConfig: parameter pencil exceeds signal length")
        return p


@dataclass
class AdmmConfig:
    lam: float = 1e4
    lambda1: float = 1e2
    lambda2: float = 2.0
    beta: float = 1.0
    tau: float = 1.0
    max_outer: int = 50
    tol: float = 1e-6
    cg_max: int = 15
    cg_tol: float = 1e-8
    enable_spirit: bool = False
    enable_vc: bool = False

    def validate(self) -> None:
        if (self.lam <= 0 or self.lambda1 < 0 or self.lambda2 < 0 or self.beta <= 0
                or self.tau <= 0 or self.tol <= 0 or self.cg_tol <= 0):
            raise ValueError("AdmmConfig: invalid parameter")


@dataclass
class SamplingMask:
    rows: int
    cols: int
    bits: np.ndarray  # uint8 (rows, cols)
    generator: str = ""
    seed: int = 0
    rate: float = 0.0
    acs: int = 0

    def count(self) -> int:
        return int(np.count_nonzero(self.bits))


@dataclass
class SpiritKernels:
    kernel_size: int
    coils: int
    weights: np.ndarray  # complex (k, k, J, J)


@dataclass
class SolveStats:
    outer_iters: int = 0
    final_rel_change: float = 0.0


def acs_range(n: int, acs: int) -> Tuple[int, int]:
    a0, a1 = C.c_size_t(), C.c_size_t()
    _check(lib.shlr_acs_range(n, acs, C.byref(a0), C.byref(a1)), "acs_range")
    return a0.value, a1.value


def mask_gauss_cartesian(n: int, rate: float, acs: int, seed: int) -> SamplingMask:
    bits = np.zeros(n, np.uint8)
    _check(lib.shlr_mask_gauss_cartesian(n, rate, acs, seed,
                                         bits.ctypes.data_as(C.POINTER(C.c_uint8))),
           "mask_gauss_cartesian")
    return SamplingMask(1, n, bits.reshape(1, n), "gauss_cartesian", seed, rate, acs)


def mask_random2d(rows: int, cols: int, rate: float, center: int, seed: int) -> SamplingMask:
    bits = np.zeros(rows * cols, np.uint8)
    _check(lib.shlr_mask_random2d(rows, cols, rate, center, seed,
                                  bits.ctypes.data_as(C.POINTER(C.c_uint8))), "mask_random2d")
    return SamplingMask(rows, cols, bits.reshape(rows, cols), "random2d", seed, rate, center)


def spirit_calibrate(acs: np.ndarray, kernel_size: int = 5, tikhonov: float = 1e-4,
                     device: bool = False) -> SpiritKernels:
    """``shlr::spirit_calibrate`` (``spirit.hpp:62-64``) on an a x b x J ACS block.
    Setup, not the per-iteration path: FP64 on the host by default,
    ``device=True`` runs the same FP64 restatement on the GPU
    (``shlr_cuda_spirit_calibrate``)."""
    blk = _c128(acs)
    if blk.ndim != 3:
        raise ValueError("spirit_calibrate: expected a x b x J ACS")
    a, b, j = blk.shape
    w = np.zeros((kernel_size, kernel_size, j, j), np.complex128)
    fn = lib.shlr_cuda_spirit_calibrate if device else lib.shlr_spirit_calibrate
    _check(fn(_dptr(blk), a, b, j, kernel_size, tikhonov, _dptr(w)), "spirit_calibrate")
    return SpiritKernels(kernel_size, j, w)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _pi_args(y: np.ndarray, mask: SamplingMask, g: Optional[SpiritKernels], hcfg: HankelConfig,
             acfg: AdmmConfig, debug_sv_iter: int, keep: list) -> ShlrPiArgs:
    acfg.validate()
    if y.ndim != 3:
        raise ValueError("shlr_pi_reconstruct: expected M x N x J")
    if acfg.enable_spirit and g is None:
        raise ValueError("shlr_pi_reconstruct: spirit enabled without kernels")
    m, n, j = y.shape
    if mask.cols != n or (mask.rows != 1 and mask.rows != m):
        raise ValueError("shlr_pi_reconstruct: mask dims mismatch")
    use_spirit = acfg.enable_spirit and acfg.lambda1 > 0.0
    if use_spirit and g.coils != j:
        raise ValueError("shlr_pi_reconstruct: kernel coil mismatch")
    yc = _c128(y)
    bits = np.ascontiguousarray(mask.bits, dtype=np.uint8)
    taps = _c128(list(hcfg.filter_taps))
    keep += [yc, bits, taps]
    a = ShlrPiArgs()
    a.m, a.n, a.j = m, n, j
    a.y = _dptr(yc)
    a.mask = bits.ctypes.data_as(C.POINTER(C.c_uint8))
    a.mask_rows = mask.rows
    if use_spirit:
        w = _c128(g.weights)
        keep.append(w)
        a.spirit_weights = _dptr(w)
        a.spirit_k = g.kernel_size
    a.taps = _dptr(taps)
    a.ntaps = len(hcfg.filter_taps)
    a.pencil_row = hcfg.pencil_for(n)
    a.pencil_col = hcfg.pencil_for(m)
    a.lam, a.lambda1, a.beta, a.tau = acfg.lam, acfg.lambda1, acfg.beta, acfg.tau
    a.tol, a.cg_tol = acfg.tol, acfg.cg_tol
    a.max_outer, a.cg_max = acfg.max_outer, acfg.cg_max
    a.enable_spirit, a.enable_vc = int(acfg.enable_spirit), int(acfg.enable_vc)
    a.debug_sv_iter = int(debug_sv_iter)
    return a


def shlr_pi_reconstruct(y: np.ndarray, mask: SamplingMask, g: Optional[SpiritKernels],
                        hcfg: HankelConfig, acfg: AdmmConfig,
                        log: Optional[List[str]] = None, stats: Optional[SolveStats] = None,
                        debug_sv_iter: int = 0, sv_out: Optional[list] = None,
                        out: Optional[np.ndarray] = None) -> np.ndarray:
    """``shlr::shlr_pi_reconstruct`` (``solvers.hpp:64-70``) on the GPU.
    out: optional caller-owned result buffer (complex128, C-contiguous,
    M x N x J; e.g. pinned host memory that is reused across calls)."""
    keep: list = []
    a = _pi_args(y, mask, g, hcfg, acfg, debug_sv_iter, keep)
    m, n, j = y.shape
    if out is not None:
        if out.dtype != np.complex128 or out.shape != (m, n, j) or not out.flags.c_contiguous:
            raise ValueError("shlr_pi_reconstruct: out must be a C-contiguous complex128 M x N x J array")
        x = out
    else:
        x = np.empty((m, n, j), np.complex128)
    st = ShlrStats()
    lines: List[str] = []

    @LOG_FN
    def _cb(_ctx, line):
        lines.append(line.decode())

    sv = None
    if debug_sv_iter > 0:
        qr = n - a.pencil_row + 1
        blocks = j * (2 if acfg.enable_vc else 1)
        d = min(a.pencil_row, blocks * qr)
        sv = np.zeros((m + n, d), np.float64)
    rc = lib.shlr_cuda_pi_reconstruct(C.byref(a), _dptr(x), _dptr(sv) if sv is not None else None,
                                      C.byref(st), _cb, None)
    if log is not None:
        log.extend(lines)
    if stats is not None:
        stats.outer_iters = int(st.outer_iters)
        stats.final_rel_change = float(st.final_rel_change)
    _check(rc, "shlr_pi_reconstruct")
    if sv_out is not None and sv is not None:
        sv_out.append(sv)
    return x


def debug_normal_apply(y: np.ndarray, mask: SamplingMask, g: Optional[SpiritKernels], hcfg: HankelConfig,
                       acfg: AdmmConfig, x: np.ndarray) -> np.ndarray:
    """Test hook: A x for the X-update operator of shlr_pi_reconstruct
    (normal_apply, operators.cpp:213-248) as the device evaluates it."""
    keep: list = []
    a = _pi_args(y, mask, g, hcfg, acfg, 0, keep)
    xc = _c128(x)
    if xc.shape != np.shape(y):
        raise ValueError("debug_normal_apply: x must have the shape of y")
    out = np.empty_like(xc)
    _check(lib.shlr_cuda_debug_normal_apply(C.byref(a), _dptr(xc), _dptr(out)), "normal_apply")
    return out


class PiPlan:
    """Resident plan (``shlr_cuda_pi_plan_*``): inputs uploaded once, the
    ADMM iterations run on-device, results downloaded on demand."""

    def __init__(self, y, mask, g, hcfg, acfg):
        self._keep: list = []
        self._args = _pi_args(y, mask, g, hcfg, acfg, 0, self._keep)
        self.shape = y.shape
        self._h = C.c_void_p()
        _check(lib.shlr_cuda_pi_plan_create(C.byref(self._args), C.byref(self._h)), "plan_create")

    def reset(self):
        _check(lib.shlr_cuda_pi_plan_reset(self._h), "plan_reset")

    def run(self, iters: int):
        _check(lib.shlr_cuda_pi_plan_run(self._h, iters), "plan_run")

    def sync(self):
        _check(lib.shlr_cuda_pi_plan_sync(self._h), "plan_sync")

    def set_timing(self, on: bool):
        _check(lib.shlr_cuda_pi_plan_set_timing(self._h, int(on)), "plan_set_timing")

    def set_warm_start(self, on: bool):
        _check(lib.shlr_cuda_pi_plan_set_warm_start(self._h, int(on)), "plan_set_warm_start")

    def debug_phases(self) -> np.ndarray:
        n = (self.shape[0] + self.shape[1]) * 24
        out = np.zeros(n, np.int64)
        _check(lib.shlr_cuda_pi_plan_debug_phases(self._h, out.ctypes.data_as(C.POINTER(C.c_longlong)), n),
               "plan_debug_phases")
        return out.reshape(-1, 24)

    def debug_sweeps(self) -> np.ndarray:
        n = self.shape[0] + self.shape[1]
        out = np.zeros(n, np.int32)
        _check(lib.shlr_cuda_pi_plan_debug_sweeps(self._h, out.ctypes.data_as(C.POINTER(C.c_int)), n),
               "plan_debug_sweeps")
        return out

    def debug_levels(self) -> np.ndarray:
        """Solver level of each lifted matrix after the last outer iteration
        (shlr_cuda_pi_plan_debug_levels: 0 level 1 ... 5 deflation chain)."""
        n = self.shape[0] + self.shape[1]
        out = np.zeros(n, np.int32)
        _check(lib.shlr_cuda_pi_plan_debug_levels(self._h, out.ctypes.data_as(C.POINTER(C.c_int)), n),
               "plan_debug_levels")
        return out

    def timing(self):
        s, t, n = C.c_double(), C.c_double(), C.c_int()
        _check(lib.shlr_cuda_pi_plan_timing(self._h, C.byref(s), C.byref(t), C.byref(n)), "timing")
        return s.value, t.value, n.value

    def download(self, log: Optional[List[str]] = None) -> Tuple[np.ndarray, SolveStats]:
        x = np.empty(self.shape, np.complex128)
        st = ShlrStats()
        lines: List[str] = []

        @LOG_FN
        def _cb(_ctx, line):
            lines.append(line.decode())

        rc = lib.shlr_cuda_pi_plan_download(self._h, _dptr(x), C.byref(st), _cb, None)
        if log is not None:
            log.extend(lines)
        _check(rc, "plan_download")
        return x, SolveStats(int(st.outer_iters), float(st.final_rel_change))

    def close(self):
        if self._h:
            lib.shlr_cuda_pi_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- parameter imaging
@dataclass
class ParameterDataset:
    """``shlr::ParameterDataset`` (``parammap.hpp:11-20``): data M x N x L x J
    (FE x PE x echoes x coils) plus the echo times in ms."""
    data: np.ndarray
    tes_ms: Sequence[float] = ()

    def validate(self) -> None:  # parammap.cpp:10-19
        if np.ndim(self.data) != 4:
            raise ValueError("ParameterDataset: expected M x N x L x J")
        if len(self.tes_ms) != np.shape(self.data)[2]:
            raise ValueError("ParameterDataset: TE count != L")
        for i, t in enumerate(self.tes_ms):
            if t <= 0 or (i > 0 and t <= self.tes_ms[i - 1]):
                raise ValueError("ParameterDataset: TEs must be positive and strictly increasing")


def shard_range(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced FE-slice range of `rank` among `world` ranks (the
    slices of recon_param_dataset are independent: parammap.cpp:37-51)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: invalid rank / world")
    return rank * m // world, (rank + 1) * m // world


def _param_args(y: np.ndarray, dataset: bool, mask: SamplingMask, hcfg: HankelConfig,
                acfg: AdmmConfig, keep: list, slices: Optional[Tuple[int, int]] = None) -> ShlrParamArgs:
    acfg.validate()
    if dataset:
        m, n, l, j = y.shape
    else:
        if y.ndim != 3:
            raise ValueError("shlr_param_reconstruct_slice: expected N x L x J")
        m, (n, l, j) = 0, y.shape
    if mask.rows != n or mask.cols != l:
        raise ValueError(("recon_param_dataset" if dataset else "shlr_param_reconstruct_slice")
                         + ": mask dims mismatch")
    yc = _c128(y)
    bits = np.ascontiguousarray(np.asarray(mask.bits).reshape(n, l), dtype=np.uint8)
    taps = _c128(list(hcfg.filter_taps))
    keep += [yc, bits, taps]
    a = ShlrParamArgs()
    a.m, a.n, a.l, a.j = m, n, l, j
    a.y = _dptr(yc)
    a.mask = bits.ctypes.data_as(C.POINTER(C.c_uint8))
    a.taps = _dptr(taps)
    a.ntaps = len(hcfg.filter_taps)
    a.pencil_pe = hcfg.pencil_for(n)
    a.pencil_par = hcfg.pencil_for_param(l)
    a.lam, a.lambda2, a.beta, a.tau = acfg.lam, acfg.lambda2, acfg.beta, acfg.tau
    a.tol, a.cg_tol = acfg.tol, acfg.cg_tol
    a.max_outer, a.cg_max = acfg.max_outer, acfg.cg_max
    a.enable_vc = int(acfg.enable_vc)
    if slices is not None:
        b, e = _check_slices(slices, m, dataset)
        if b == e:
            raise ValueError("recon_param_dataset: empty slice range")
        a.slice_begin, a.slice_end = b, e
    return a


def _check_slices(slices, m: int, dataset: bool = True) -> Tuple[int, int]:
    """Validated FE-slice range [begin, end) of a dataset of m slices (an
    empty range is valid: a rank with no slices).  The C-ABI reads (0, 0) as
    "all slices", so an empty range must never reach it."""
    if not dataset:
        raise ValueError("recon_param_dataset: a slice range needs a dataset")
    b, e = int(slices[0]), int(slices[1])
    if not 0 <= b <= e <= m:
        raise ValueError("recon_param_dataset: slice range outside the dataset")
    return b, e


def _run_param(a: ShlrParamArgs, out_shape, log, what: str):
    x = np.empty(out_shape, np.complex128)
    st = ShlrStats()
    lines: List[str] = []

    @LOG_FN
    def _cb(_ctx, line):
        lines.append(line.decode())

    # no callback when the caller does not want the log (12 800 lines at config 4)
    rc = lib.shlr_cuda_param_reconstruct(C.byref(a), _dptr(x), C.byref(st),
                                         _cb if log is not None else LOG_FN(), None)
    if log is not None:
        log.extend(lines)
    _check(rc, what)
    return x, st


def shlr_param_reconstruct_slice(y_m: np.ndarray, mask: SamplingMask, hcfg: HankelConfig,
                                 acfg: AdmmConfig, log: Optional[List[str]] = None,
                                 stats: Optional[SolveStats] = None) -> np.ndarray:
    """``shlr::shlr_param_reconstruct_slice`` (``solvers.hpp:74-79``) on the GPU:
    y_m is the zero-filled N x L x J plane at one FE position."""
    keep: list = []
    a = _param_args(np.asarray(y_m), False, mask, hcfg, acfg, keep)
    x, st = _run_param(a, np.shape(y_m), log, "shlr_param_reconstruct_slice")
    if stats is not None:
        stats.outer_iters = int(st.outer_iters)
        stats.final_rel_change = float(st.final_rel_change)
    return x


def recon_param_dataset(y: ParameterDataset, mask: SamplingMask, hcfg: HankelConfig,
                        acfg: AdmmConfig, log: Optional[List[str]] = None,
                        total_iters: Optional[List[int]] = None,
                        slices: Optional[Tuple[int, int]] = None) -> ParameterDataset:
    """``shlr::recon_param_dataset`` (``parammap.hpp:35-40``): iFFT along FE, then
    every FE slice's ADMM (each with its own early stop) -- all slices batched
    on the device.  ``total_iters`` (a list) receives the summed outer
    iterations, the reference's ``*total_iters``.  ``slices=(begin, end)``
    (extension for multi-GPU jobs, see ``shard_range``) solves only those FE
    slices; the result then holds end - begin slices."""
    y.validate()
    keep: list = []
    data = np.asarray(y.data)
    if mask.rows != data.shape[1] or mask.cols != data.shape[2]:
        raise ValueError("recon_param_dataset: mask dims mismatch")
    if slices is not None and _check_slices(slices, data.shape[0])[0] == slices[1]:
        # empty shard (more ranks than FE slices): nothing to solve
        if total_iters is not None:
            total_iters.append(0)
        return ParameterDataset(np.empty((0,) + data.shape[1:], np.complex128), list(y.tes_ms))
    a = _param_args(data, True, mask, hcfg, acfg, keep, slices)
    shape = data.shape if slices is None else (slices[1] - slices[0],) + data.shape[1:]
    x, st = _run_param(a, shape, log, "recon_param_dataset")
    if total_iters is not None:
        total_iters.append(int(st.outer_iters))
    return ParameterDataset(x, list(y.tes_ms))


class ParamPlan:
    """Resident plan of the parameter path (``shlr_cuda_param_plan_*``)."""

    def __init__(self, y, mask, hcfg, acfg, dataset: bool = True, slices: Optional[Tuple[int, int]] = None):
        self._keep: list = []
        y = np.asarray(y)
        self._args = _param_args(y, dataset, mask, hcfg, acfg, self._keep, slices)
        self.shape = y.shape if slices is None else (slices[1] - slices[0],) + y.shape[1:]
        self._h = C.c_void_p()
        _check(lib.shlr_cuda_param_plan_create(C.byref(self._args), C.byref(self._h)), "plan_create")

    def reset(self):
        _check(lib.shlr_cuda_param_plan_reset(self._h), "plan_reset")

    def run(self, iters: int):
        _check(lib.shlr_cuda_param_plan_run(self._h, iters), "plan_run")

    def sync(self):
        _check(lib.shlr_cuda_param_plan_sync(self._h), "plan_sync")

    def set_timing(self, on: bool):
        _check(lib.shlr_cuda_param_plan_set_timing(self._h, int(on)), "plan_set_timing")

    def timing(self):
        s, t, n = C.c_double(), C.c_double(), C.c_int()
        _check(lib.shlr_cuda_param_plan_timing(self._h, C.byref(s), C.byref(t), C.byref(n)), "timing")
        return s.value, t.value, n.value

    def download(self, log: Optional[List[str]] = None) -> Tuple[np.ndarray, SolveStats]:
        x = np.empty(self.shape, np.complex128)
        st = ShlrStats()
        lines: List[str] = []

        @LOG_FN
        def _cb(_ctx, line):
            lines.append(line.decode())

        rc = lib.shlr_cuda_param_plan_download(self._h, _dptr(x), C.byref(st), _cb, None)
        if log is not None:
            log.extend(lines)
        _check(rc, "plan_download")
        return x, SolveStats(int(st.outer_iters), float(st.final_rel_change))

    def close(self):
        if self._h:
            lib.shlr_cuda_param_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fp32_peak_tflops() -> float:
    v = C.c_double()
    _check(lib.shlr_cuda_fp32_peak_tflops(C.byref(v)), "fp32_peak")
    return v.value


def hankel_svt_batched(vecs: np.ndarray, p: int, tau: float, want_sv: bool = True):
    """Config-5 unit on host complex128 arrays: vecs (B, Nc, N) ->
    (adjoint vectors (B, Nc, N), singular values (B, d) descending, or None
    with want_sv=False -- the exact singular values need the full eigen-solver,
    which covers d <= 128; without them the subspace levels run any d up to
    496, tall or wide, with the deflation chain behind them: no rank limit)."""
    v = _c128(vecs)
    b, nc, n = v.shape
    q = n - p + 1
    d = min(p, nc * q)
    out = np.empty_like(v)
    sv = np.empty((b, d), np.float64) if want_sv else None
    _check(lib.shlr_cuda_hankel_svt_batched_host(_dptr(v), b, nc, n, p, tau, _dptr(out),
                                                 _dptr(sv) if want_sv else None),
           "hankel_svt_batched")
    return out, sv


def hankel_svt_batched_device(vecs_ptr: int, batch: int, nc: int, n: int, p: int, tau: float,
                              out_ptr: int, sv_ptr: int = 0, stream: int = 0) -> None:
    """Device-pointer variant (complex64 data already resident in HBM)."""
    _check(lib.shlr_cuda_hankel_svt_batched(C.c_void_p(vecs_ptr), batch, nc, n, p, tau,
                                            C.c_void_p(out_ptr), C.c_void_p(sv_ptr or None),
                                            C.c_void_p(stream or None)), "hankel_svt_batched")


def lift_index_map(n: int, p: int, coils: int, vc: bool, path: int = 1) -> np.ndarray:
    """(coil, source index, conj) of every element of the p x (blocks q)
    weighted lift, read back from the kernels' own lift stage run on
    index-encoded spectra: path 0 = full solver, 1 = subspace solver,
    2 = large-d variants (``shlr_cuda_lift_index_map_path``)."""
    q = n - p + 1
    blocks = coils * (2 if vc else 1)
    out = np.empty((p, blocks * q, 3), np.int32)
    _check(lib.shlr_cuda_lift_index_map_path(n, p, coils, int(vc), path,
                                             out.ctypes.data_as(C.POINTER(C.c_int32))), "lift_index_map")
    return out


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def ssos(x: np.ndarray) -> np.ndarray:
    """``shlr::ssos`` (``io.hpp:31``, ``io.cpp:105-117``) on the device: the
    root-sum-of-squares coil combination of an M x N x J image, FP64."""
    xc = _c128(x)
    if xc.ndim != 3:
        raise ValueError("ssos: expected an M x N x J tensor")
    m, n, j = xc.shape
    out = np.empty((m, n), np.float64)
    _check(lib.shlr_cuda_ssos(_dptr(xc), m, n, j, _dptr(out)), "ssos")
    return out


def rlne(ref: np.ndarray, rec: np.ndarray) -> float:
    """``shlr::rlne`` (``metrics.hpp:17``, ``metrics.cpp:9-21``) on the device."""
    a, b = _f64(ref), _f64(rec)
    if a.ndim != 2 or a.shape != b.shape:
        raise ValueError("rlne: dimension mismatch")
    out = C.c_double()
    _check(lib.shlr_cuda_rlne(_dptr(a), _dptr(b), a.size, C.byref(out)), "rlne")
    return out.value


def mssim(ref: np.ndarray, rec: np.ndarray) -> float:
    """``shlr::mssim`` (``metrics.hpp:21``, ``metrics.cpp:23-75``) on the device:
    mean SSIM over 11 x 11 Gaussian windows."""
    a, b = _f64(ref), _f64(rec)
    if a.ndim != 2 or a.shape != b.shape:
        raise ValueError("mssim: dimension mismatch")
    out = C.c_double()
    _check(lib.shlr_cuda_mssim(_dptr(a), _dptr(b), a.shape[0], a.shape[1], C.byref(out)), "mssim")
    return out.value


def fft_along_axis(x: np.ndarray, axis: int, inverse: bool) -> np.ndarray:
    a = _c128(x).copy()
    dims = (C.c_size_t * a.ndim)(*a.shape)
    _check(lib.shlr_cuda_fft_along_axis(_dptr(a), dims, a.ndim, axis, int(inverse)),
           "fft_along_axis")
    return a
