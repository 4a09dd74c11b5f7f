#!/usr/bin/env python
"""Benchmark of the B200 SHLR hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1], the headline): parallel-MRI SHLR-S on a
256 x 256 x 8-coil seeded phantom, R = 5 Gaussian Cartesian mask with 24 ACS
lines, Hankel window K = 15 (pencil 242 -> 512 lifted 242 x 120 matrices per
outer iteration), SPIRiT 5 x 5 (lambda1 = 1e2, Tikhonov 1e-4), lambda = 1e4,
beta = tau = 1, CG 15 / 1e-8, 50 outer iterations.

A "step" is one ADMM outer iteration (RHS, 15-iteration capped CG with the
SPIRiT term, lifted spectra, 512 fused Hankel-SVT + dual updates, stop rule).
`value` = outer iterations / s with every buffer resident in HBM, timed with
CUDA events on the plan's stream over exactly --steps iterations after
--warmup iterations, max over ranks.  The per-iteration working set (duals
119 MB + SPIRiT P 33.5 MB + vectors) exceeds the 126 MB L2, so no explicit
flush is done ("inputs larger than L2").

Multi-GPU: the path is one reconstruction per GPU ("replicas only",
DESIGN.md): each rank runs its own replica, `value` = N * steps / max time.

`--impl reference` times the reference C++ implementation compiled from its
own sources (oracle/_ref/ref_driver) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

CFG2 = dict(M=256, N=256, J=8, K=15, rate=0.2, acs=24, spirit=True, kernel=5, tikhonov=1e-4,
            lam=1e4, lambda1=1e2, beta=1.0, tau=1.0, cg_max=15, cg_tol=1e-8, outer=50)
WORKLOAD = ("config2: 256x256x8 coils, SHLR-S (SPIRiT 5x5, lambda1=1e2), R=5 Gaussian Cartesian "
            "+ 24 ACS lines, Hankel window K=15 (pencil 242, 512 lifted 242x120 matrices/iter), "
            "lambda=1e4, beta=tau=1, CG 15/1e-8, 50 outer iterations")


def svt_flops(e: int, d: int) -> float:
    """Algorithmic FLOPs of one Hankel-SVT matrix:
    Gram 8ed^2 + Hermitian eig 36d^3 + W 8d^3 + Z = AW 8ed^2."""
    return 16.0 * e * d * d + 44.0 * d ** 3


def make_inputs(cfg=CFG2):
    from paper_2107_11650_b200 import api as A
    from paper_2107_11650_b200 import synth
    ph = synth.pi_phantom(cfg["M"], cfg["N"], cfg["J"])
    mask = A.mask_gauss_cartesian(cfg["N"], cfg["rate"], cfg["acs"], synth.SEED_MASK)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    g = None
    if cfg["spirit"]:
        a0, a1 = A.acs_range(cfg["N"], cfg["acs"])
        g = A.spirit_calibrate(y[:, a0:a1, :], cfg["kernel"], cfg["tikhonov"])
    hcfg = A.HankelConfig(pencil=cfg["N"] - cfg["K"] + 1)
    return y, mask, g, hcfg


CFG4 = dict(M=256, N=256, L=12, J=4, K=13, rate=1.0 / 6.0, acs=16, vc=True, lam=1e4, lambda2=2.0,
            beta=1.0, tau=1.0, cg_max=15, cg_tol=1e-8, outer=50)
WORKLOAD4 = ("config4: T2 mapping 256x256, 4 coils, 12 echoes (TE=10e ms), SHLR-VP (virtual coils), "
             "per-echo R=6 Gaussian Cartesian masks (16 ACS lines, seed 11650+e), Hankel window K=13 "
             "(PE lift 244x104: 3072 per iter; echo lift 5x32: 65536 per iter), lambda2=2, "
             "256 FE slices batched, 50 outer iterations")


def make_param_inputs(cfg=CFG4, m=None):
    """Config 4 (BASELINE.json configs[3]): seeded T2 phantom k-space (M, N, L, J),
    the N x L per-echo mask (column e = mask_gauss_cartesian(N, 1/6, acs, 11650 + e),
    SURVEY 8 mapping table), zero-filled, plus the configs."""
    from paper_2107_11650_b200 import api as A
    from paper_2107_11650_b200 import synth
    M = m or cfg["M"]
    _, k, tes, _ = synth.t2_phantom(M, cfg["N"], cfg["J"], cfg["L"])
    bits = np.stack([A.mask_gauss_cartesian(cfg["N"], cfg["rate"], cfg["acs"], synth.SEED_MASK + e).bits[0]
                     for e in range(cfg["L"])], axis=1)
    mask = A.SamplingMask(cfg["N"], cfg["L"], bits, "gauss_cartesian", synth.SEED_MASK, cfg["rate"], cfg["acs"])
    y = np.where(bits[None, :, :, None].astype(bool), k, 0)
    hcfg = A.HankelConfig(pencil=cfg["N"] - cfg["K"] + 1)
    acfg = A.AdmmConfig(lam=cfg["lam"], lambda2=cfg["lambda2"], beta=cfg["beta"], tau=cfg["tau"],
                        max_outer=cfg["outer"], tol=1e-300, cg_max=cfg["cg_max"], cg_tol=cfg["cg_tol"],
                        enable_vc=cfg["vc"])
    return A.ParameterDataset(y, list(tes)), mask, hcfg, acfg


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits", "-lms", "100"],
            stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return None, 0, 1, 0
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(local)
    dist.init_process_group(backend)
    return dist, rank, world, local


def max_over_ranks(dist, value: float) -> float:
    if dist is None:
        return value
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------- CPU leg
# The reference legs never import the product API (nor load its .so): the
# image comes from the harness generator (numpy only), the mask from the
# reference's own generator (`ref_driver mask`), the SPIRiT kernels from the
# reference's own spirit_calibrate inside `ref_driver pi` (no kernels=).
def write_ref_inputs(tmp: str, cfg=CFG2) -> None:
    from paper_2107_11650_b200 import synth  # numpy-only harness generator
    from paper_2107_11650_b200.cplx_io import write_cplx
    ph = synth.pi_phantom(cfg["M"], cfg["N"], cfg["J"])
    write_cplx(ph.kspace, os.path.join(tmp, "y.cplx"))
    subprocess.run([REF_DRIVER, "mask", "kind=gauss", f"n={cfg['N']}", f"rate={cfg['rate']}",
                    f"acs={cfg['acs']}", f"seed={synth.SEED_MASK}", "out=m.cplx"], cwd=tmp, check=True)


def ref_pi_cmd(cfg, iters: int):
    """The stock shlr_pi_reconstruct (proj/src/solvers.cpp:95-191) through
    ref_driver, timed per iteration through its own log lines (time=1)."""
    cmd = [REF_DRIVER, "pi", "y=y.cplx", "mask=m.cplx", f"pencil={cfg['N'] - cfg['K'] + 1}",
           f"max_outer={iters}", "tol=1e-300", "time=1", f"lambda={cfg['lam']}", f"beta={cfg['beta']}",
           f"tau={cfg['tau']}", f"cg_max={cfg['cg_max']}", f"cg_tol={cfg['cg_tol']}"]
    if cfg.get("spirit"):
        cmd += ["spirit=1", f"acs={cfg['acs']}", f"kernel={cfg['kernel']}", f"tikhonov={cfg['tikhonov']}",
                f"lambda1={cfg['lambda1']}"]
    return cmd


def run_reference(tmp: str, procs: int, iters: int, budget_s: float, cfg=CFG2):
    """Runs `procs` concurrent reference processes, each the stock
    shlr_pi_reconstruct for up to `iters` outer iterations, stopping at
    `budget_s` once every process has timed an iteration.  Returns per-process
    lists of per-iteration seconds: iterations 2.. (setup excluded) when a
    process got that far, else its first iteration (setup included)."""
    cmd = ref_pi_cmd(cfg, iters)
    ps = []
    for i in range(procs):
        ps.append(subprocess.Popen(cmd + [f"out=ref{i}"], cwd=tmp, stdout=subprocess.PIPE,
                                   stderr=subprocess.DEVNULL, text=True,
                                   env=dict(os.environ, OMP_NUM_THREADS="1")))
    later = [[] for _ in ps]
    first = [[] for _ in ps]

    def reader(i, p):
        for line in p.stdout:
            if line.startswith("iter_seconds="):
                later[i].append(float(line.split("=")[1]))
            elif line.startswith("first_iter_seconds="):
                first[i].append(float(line.split("=")[1]))

    threads = [threading.Thread(target=reader, args=(i, p), daemon=True) for i, p in enumerate(ps)]
    for t in threads:
        t.start()
    t0 = time.time()
    while any(p.poll() is None for p in ps):
        if time.time() - t0 > budget_s and all(len(f) >= 1 for f in first):
            break
        time.sleep(0.5)
    for p in ps:
        if p.poll() is None:
            p.kill()
    for t in threads:
        t.join(timeout=5)
    return [lt if lt else f for lt, f in zip(later, first)]


def cpu_baseline(procs: int, iters: int, budget_s: float, cfg=CFG2):
    if not os.path.exists(REF_DRIVER):
        return None
    tmp = tempfile.mkdtemp(prefix="shlr_ref_")
    try:
        write_ref_inputs(tmp, cfg)
        res = run_reference(tmp, procs, iters, budget_s, cfg)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    per_proc = [statistics.mean(r) for r in res if r]
    if not per_proc:
        return None
    done = sum(len(r) for r in res)
    # throughput of `procs` concurrent single-threaded reference processes
    value = sum(1.0 / s for s in per_proc)
    return {"value": value, "unit": "iterations/s", "cores": len(per_proc), "kind": "reference",
            "sample": (f"{len(per_proc)} concurrent single-threaded processes of the stock "
                       f"shlr_pi_reconstruct (oracle/_ref/ref_driver: proj/src/*.cpp unmodified + builder "
                       f"Eigen subset; reference-generated mask, reference SPIRiT calibration), "
                       f"{done} outer iterations of config 2 timed through the solver's log lines "
                       f"(iterations 2.., setup excluded); mean {statistics.mean(per_proc):.2f} s per "
                       f"iteration per process")}


def bench_config(world: int) -> dict:
    """The `config` object of both arms (same workload, same keys)."""
    m, n, j, k = CFG2["M"], CFG2["N"], CFG2["J"], CFG2["K"]
    return {"workload": WORKLOAD, "parallelism": f"replicas x{world}",
            "l2": "inputs larger than L2: 119 MB duals + 33.5 MB SPIRiT P streamed per step",
            "lifted_matrix": f"{n - k + 1}x{j * k}", "matrices_per_step": m + n}


# ---------------------------------------------------------------- GPU arm
def gpu_arm(args, dist, rank, world, local):
    from paper_2107_11650_b200 import api as A
    if A.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device visible (the product path has no CPU fallback)")
    cfg = CFG2
    y, mask, g, hcfg = make_inputs(cfg)
    iters_total = args.warmup + args.steps
    acfg = A.AdmmConfig(lam=cfg["lam"], lambda1=cfg["lambda1"], beta=cfg["beta"], tau=cfg["tau"],
                        max_outer=max(iters_total, cfg["outer"]), tol=1e-300,
                        cg_max=cfg["cg_max"], cg_tol=cfg["cg_tol"], enable_spirit=True)
    plan = A.PiPlan(y, mask, g, hcfg, acfg)
    # warm-up iterations (graph capture happens on the first run call)
    plan.run(args.warmup)
    plan.sync()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    barrier(dist)
    plan.run(args.steps)
    plan.sync()
    _, total_ms, launches = plan.timing()
    barrier(dist)
    clocks = sampler.stop() if sampler else None
    t_max_ms = max_over_ranks(dist, total_ms)
    x, stats = plan.download()
    assert stats.outer_iters == iters_total, (stats.outer_iters, iters_total)

    # Hankel-SVT kernel alone: CUDA events around its launch in timing mode
    plan.reset()
    plan.set_timing(True)
    plan.run(1)   # one untimed iteration so the duals are not the all-ones start state
    plan.sync()
    reps = 5
    plan.run(reps)
    plan.sync()
    svt_ms_total, _, _ = plan.timing()
    svt_ms = svt_ms_total / reps
    plan.set_timing(False)
    plan.close()

    m, n, j, k = cfg["M"], cfg["N"], cfg["J"], cfg["K"]
    p = n - k + 1
    e, d = max(p, j * k), min(p, j * k)
    flops = (m + n) * svt_flops(e, d)
    fp32_peak = A.fp32_peak_tflops()
    achieved_tf = flops / (svt_ms * 1e-3) / 1e12
    # DRAM bytes of one launch of the dominant kernel from the committed ncu
    # --set full capture of this round (profiles/r02_ncu_summary.json, c2_svt)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02_ncu_summary.json")
    if os.path.exists(prof):
        with open(prof) as f:
            cap = json.load(f).get("c2_svt") or {}
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd, wr = cap.get("dram__bytes_read.sum"), cap.get("dram__bytes_write.sum")
        if rd is not None and wr is not None:
            traffic = (rd * scale.get(cap.get("dram__bytes_read.sum.unit", "byte"), 1.0)
                       + wr * scale.get(cap.get("dram__bytes_write.sum.unit", "byte"), 1.0))

    # e2e: the public call with host buffers, H2D of y and D2H of x inside
    e2e = None
    if not args.no_e2e:
        acfg_e2e = A.AdmmConfig(lam=cfg["lam"], lambda1=cfg["lambda1"], beta=cfg["beta"], tau=cfg["tau"],
                                max_outer=cfg["outer"], tol=1e-300, cg_max=cfg["cg_max"],
                                cg_tol=cfg["cg_tol"], enable_spirit=True)
        # process warm-up: one 1-iteration call on the same geometry loads the
        # kernels (lazy module loading) before the timed call
        A.shlr_pi_reconstruct(y, mask, g, hcfg, A.AdmmConfig(lam=cfg["lam"], lambda1=cfg["lambda1"],
                                                            max_outer=1, enable_spirit=True))
        # host buffers of the timed calls: pinned (page-locked) input and result
        # arrays, as a caller that reconstructs slice after slice would keep them
        import torch
        y_pin = torch.from_numpy(np.ascontiguousarray(y, dtype=np.complex128)).pin_memory().numpy()
        x_pin = torch.empty(y.shape, dtype=torch.complex128).pin_memory().numpy()
        barrier(dist)
        calls = []
        for _ in range(3):  # median of three calls (host wall clock per call)
            t0 = time.perf_counter()
            st = A.SolveStats()
            A.shlr_pi_reconstruct(y_pin, mask, g, hcfg, acfg_e2e, stats=st, out=x_pin)
            calls.append(time.perf_counter() - t0)
        t_e2e = max_over_ranks(dist, statistics.median(calls))
        # the full user flow of the reference CLI (shlr_cli.cpp:384-411): SPIRiT
        # calibration from the ACS block (on the device), then the reconstruction
        a0, a1 = A.acs_range(cfg["N"], cfg["acs"])
        cal = []
        for _ in range(3):
            t0 = time.perf_counter()
            g2 = A.spirit_calibrate(y_pin[:, a0:a1, :], cfg["kernel"], cfg["tikhonov"], device=True)
            A.shlr_pi_reconstruct(y_pin, mask, g2, hcfg, acfg_e2e, out=x_pin)
            cal.append(time.perf_counter() - t0)
        t_cal = max_over_ranks(dist, statistics.median(cal))
        e2e = {"value": world * st.outer_iters / t_e2e, "unit": "iterations/s",
               "calls_s": calls,
               "with_device_calibration": {"value": world * st.outer_iters / t_cal, "unit": "iterations/s",
                                           "calls_s": cal},
               "h2d_bytes_per_step": int(y.size * 16 + mask.bits.size + (g.weights.size * 16 if g else 0)),
               "d2h_bytes_per_step": int(y.size * 16),
               "step": "one full 50-iteration shlr_cuda_pi_reconstruct call (pinned host complex128 y, "
                       "mask, SPIRiT kernels in; pinned host complex128 x out; plan setup incl. SPIRiT "
                       "map build inside); median of 3 calls after a warm-up call"}

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(procs=1, iters=2, budget_s=args.cpu_budget)

    extra = {}
    if not args.no_extra:
        extra["config4_param"] = param_workload(args, dist, world, fp32_peak)
        if rank == 0 and not args.no_cpu:
            extra["config4_param"]["cpu_baseline"] = param_cpu_baseline()
        extra["config3_large_d"] = large_d_workload(args, dist, world, fp32_peak)
        extra["config5_sweep"] = sweep_workload(args, fp32_peak, cpu=rank == 0 and not args.no_cpu)
        extra["config2_shlr_sv"] = sv_workload(args, dist, world, fp32_peak)
        extra["config1_small"] = small_workload(args, dist, world, rank, fp32_peak)

    value = world * args.steps / (t_max_ms * 1e-3)
    out = {
        "metric": "recon iterations/sec (256x256x8 coils, SHLR-S, K=15)",
        "value": value,
        "unit": "iterations/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c64 (fp32 complex; fp64 reductions and setup)",
        "data": "synthetic: seeded BASELINE phantom (10 ellipses, smooth phase, 8 Gaussian coils, 40 dB)",
        "impl": "b200",
        "config": bench_config(world),
        "hankel_svt": {"matrices_per_s": (m + n) / (svt_ms * 1e-3), "kernel_ms": svt_ms,
                       "share_of_step": svt_ms / (t_max_ms / args.steps),
                       "solver": "subspace iteration (block 48; 1 pass per ADMM iteration warm, 6 cold), chunk contractions as 3xTF32 "
                                 "mma.sync, tensor-core Cholesky QR, Rayleigh-Ritz by tridiagonalisation/multisection, two co-located "
                                 "CTAs per SM; full two-stage Jacobi for matrices with > 40 singular values above tau"},
        "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved_tf / fp32_peak, "traffic": traffic,
                     "kernel": "svt_subspace_kernel<120,48,32,BIG,L1,2,MMA> (+ flagged-matrix hankel_svt_kernel)",
                     "bound_note": "compute-bound; the denominator is the FP32 FMA peak north_star names "
                                   "(contractions run as 3xTF32 on the tensor cores: 12 mma.sync per complex tile step)",
                     "algorithmic": f"{m + n} x (16 e d^2 + 44 d^3), e={e}, d={d}: {flops / 1e9:.2f} GFLOP/launch",
                     "peak_source": "measured FP32 FMA probe on this GPU (MEASURED_PEAKS.json has no FP32 figure)"},
        "gpu_launches": launches * args.steps,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "other_workloads": extra,
    }
    if rank == 0:
        print(json.dumps(out))


def param_workload(args, dist, world, fp32_peak):
    """BASELINE config 4 (T2 mapping, SHLR-VP) on the same GPU: resident-plan
    outer iterations/s over all 256 FE slices (each a full Algorithm-S2 step:
    RHS FFT, per-slice capped CG, 3072 PE lifts 244 x 104 + 65536 echo lifts
    5 x 32 with SVT, duals and adjoints, stop rule), the SVT launches alone, and
    an e2e recon_param_dataset call with host buffers.  Not the headline metric."""
    from paper_2107_11650_b200 import api as A
    cfg = CFG4
    ds, mask, hcfg, acfg = make_param_inputs(cfg)
    acfg.max_outer = max(cfg["outer"], args.warmup + args.steps)
    # N ranks: each takes a contiguous range of the independent FE slices
    # (parammap.cpp:37-51) -- no collective; one dataset iteration = all ranks
    rank = dist.get_rank() if dist is not None else 0
    shard = A.shard_range(cfg["M"], world, rank) if world > 1 else None
    plan = A.ParamPlan(ds.data, mask, hcfg, acfg, dataset=True, slices=shard)
    plan.run(args.warmup)
    plan.sync()
    barrier(dist)
    plan.run(args.steps)
    plan.sync()
    _, total_ms, launches = plan.timing()
    t_max_ms = max_over_ranks(dist, total_ms)
    plan.reset()
    plan.set_timing(True)
    plan.run(1)
    plan.sync()
    reps = 3
    plan.run(reps)
    plan.sync()
    svt_ms = plan.timing()[0] / reps
    plan.close()
    n, k, j = cfg["N"], cfg["K"], cfg["J"]
    p = n - k + 1
    bq = (2 if cfg["vc"] else 1) * j * k
    e, d = max(p, bq), min(p, bq)
    l = cfg["L"]
    pp = l // 3 + (1 if l % 3 else 0) + 1
    e2, d2 = max(pp, j * (l - pp + 1)), min(pp, j * (l - pp + 1))
    flops = cfg["M"] * l * svt_flops(e, d) + cfg["M"] * n * svt_flops(e2, d2)
    out = {"workload": WORKLOAD4, "value": args.steps / (t_max_ms * 1e-3), "unit": "iterations/s",
           "scaling": "strong (FE slices sharded over the ranks, no collective)" if world > 1 else "n/a",
           "ms_per_step": t_max_ms / args.steps, "gpu_launches_per_step": launches,
           "svt_ms": svt_ms, "svt_share_of_step": svt_ms / (t_max_ms / args.steps),
           "svt_roofline": {"bound": "fp32", "achieved": flops / (svt_ms * 1e-3) / 1e12, "peak": fp32_peak,
                            "unit": "TFLOP/s", "frac": flops / (svt_ms * 1e-3) / 1e12 / fp32_peak,
                            "algorithmic": f"256*12 x F({e}x{d}) + 256*256 x F({e2}x{d2}), "
                                           f"F = 16 e d^2 + 44 d^3: {flops / 1e9:.1f} GFLOP/step"}}
    if not args.no_e2e:
        acfg.max_outer = 1
        A.recon_param_dataset(ds, mask, hcfg, acfg, slices=shard)  # process warm-up (kernel loading)
        acfg.max_outer = cfg["outer"]
        barrier(dist)
        t0 = time.perf_counter()
        tot = []
        A.recon_param_dataset(ds, mask, hcfg, acfg, total_iters=tot, slices=shard)
        t_e2e = max_over_ranks(dist, time.perf_counter() - t0)
        out["e2e"] = {"value": cfg["outer"] / t_e2e, "unit": "iterations/s",
                      "h2d_bytes_per_step": int(ds.data.size * 16 + mask.bits.size),
                      "d2h_bytes_per_step": int(ds.data.size * 16),
                      "step": "one 50-iteration recon_param_dataset call (host complex128 M x N x L x J in/out, "
                              "FE iFFT and plan setup inside)", "slice_iterations": tot[0]}
    return out


def param_cpu_baseline(iters: int = 3):
    """The reference (oracle/_ref/ref_driver = proj/src unmodified) on the centre
    FE slice of config 4 for a few iterations, one core; a dataset iteration is
    256 independent slice iterations (parammap.cpp:37-51)."""
    if not os.path.exists(REF_DRIVER):
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import shlr_oracle as O
    from paper_2107_11650_b200.cplx_io import write_cplx, write_mask
    ds, mask, _, _ = make_param_inputs()
    hybrid = O.fft_along_axis(ds.data[:, :, :, :], 0, True)
    tmp = tempfile.mkdtemp(prefix="shlr_ref4_")
    try:
        write_cplx(hybrid[128], os.path.join(tmp, "s.cplx"))
        write_mask(mask.bits, os.path.join(tmp, "m.cplx"))
        out = subprocess.run([REF_DRIVER, "param", "y=s.cplx", "mask=m.cplx", "out=r", "vc=1",
                              f"pencil={CFG4['N'] - CFG4['K'] + 1}", f"max_outer={iters}", "tol=1e-300",
                              "time=1"], cwd=tmp, capture_output=True, text=True, timeout=600).stdout
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    secs = float(out.split("param seconds=")[1].split()[0])
    per_slice_iter = secs / iters
    return {"value": 1.0 / (CFG4["M"] * per_slice_iter), "unit": "iterations/s", "cores": 1, "kind": "reference",
            "sample": f"reference shlr_param_reconstruct_slice on the centre FE slice, {iters} iterations "
                      f"({per_slice_iter:.3f} s per slice-iteration), times 256 slices per dataset iteration"}


WORKLOAD3 = ("config3: 256x256x32 coils (two staggered rings), SHLR-V (virtual coils), R=6 2D random mask "
             "(mask_random2d(256,256,1/6,24): the reference's nearest generator to BASELINE's Poisson disc), "
             "Hankel window K=11 (pencil 246, 512 lifted 246x704 matrices/iter, d=246), 50 outer iterations")


def large_d_workload(args, dist, world, fp32_peak):
    """BASELINE config 3 on the same GPU (50 iterations, the reference default):
    the large-d subspace SVT path.  Timed over iterations 1-50 as a whole (the
    rank above the threshold, and with it the share of matrices at level 2
    (64 columns) and level 3 (deflated remainder), grows with the iteration)."""
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import make_c3_golden as G
    from paper_2107_11650_b200 import api as A
    iters = 50
    y, bits = G.make_inputs()
    mask = A.SamplingMask(256, 256, bits)
    hcfg = A.HankelConfig(pencil=246)
    acfg = A.AdmmConfig(max_outer=iters, tol=1e-300, enable_vc=True)
    plan = A.PiPlan(y, mask, None, hcfg, acfg)
    plan.run(1)   # graph capture + context warm-up on the first iteration
    plan.sync()
    plan.reset()
    barrier(dist)
    plan.run(iters)
    plan.sync()
    _, total_ms, launches = plan.timing()
    t_max_ms = max_over_ranks(dist, total_ms)
    plan.download()   # raises if a lifted matrix exceeded the large-d block
    plan.close()
    e, d = 704, 246
    flops = 512 * svt_flops(e, d)
    out = {"workload": WORKLOAD3, "value": world * iters / (t_max_ms * 1e-3), "unit": "iterations/s",
           "ms_per_step": t_max_ms / iters, "steps": iters, "gpu_launches_per_step": launches,
           "algorithmic_tflops": flops * iters / (t_max_ms * 1e-3) / 1e12,
           "algorithmic_frac_of_fp32_peak": flops * iters / (t_max_ms * 1e-3) / 1e12 / fp32_peak,
           "algorithmic": f"512 x F(704x246), F = 16 e d^2 + 44 d^3 = {svt_flops(e, d) / 1e9:.3f} GFLOP "
                          "per matrix (whole step counted as SVT time: upper bound on the step, lower bound "
                          "on the SVT rate)"}
    if not args.no_e2e:
        barrier(dist)
        t0 = time.perf_counter()
        st = A.SolveStats()
        A.shlr_pi_reconstruct(y, mask, None, hcfg, acfg, stats=st)
        t_e2e = max_over_ranks(dist, time.perf_counter() - t0)
        out["e2e"] = {"value": world * st.outer_iters / t_e2e, "unit": "iterations/s",
                      "h2d_bytes_per_step": int(y.size * 16 + bits.size), "d2h_bytes_per_step": int(y.size * 16),
                      "step": "one 50-iteration shlr_cuda_pi_reconstruct call with host buffers"}
    return out


def sv_workload(args, dist, world, fp32_peak):
    """SHLR-SV (SPIRiT + virtual coils, the paper's most accurate variant) on
    the config-2 inputs: 256^2 x 8 coils, K = 15 -> 512 lifted 242 x 240
    matrices per iteration (tall weighted, d = 240: the large-d subspace
    levels).  Resident-plan iterations/s over iterations 4.. (after
    --warmup), with the adaptive warm passes of the first iterations excluded
    only by the warm-up.  The reference needs ~283 s per iteration on one core
    (tests/golden/make_sv_golden.py: 12 iterations in 57 min)."""
    from paper_2107_11650_b200 import api as A
    cfg = CFG2
    y, mask, g, hcfg = make_inputs(cfg)
    acfg = A.AdmmConfig(lam=cfg["lam"], lambda1=cfg["lambda1"], beta=cfg["beta"], tau=cfg["tau"],
                        max_outer=max(50, args.warmup + args.steps), tol=1e-300, cg_max=cfg["cg_max"],
                        cg_tol=cfg["cg_tol"], enable_spirit=True, enable_vc=True)
    plan = A.PiPlan(y, mask, g, hcfg, acfg)
    plan.run(args.warmup)
    plan.sync()
    barrier(dist)
    plan.run(args.steps)
    plan.sync()
    _, total_ms, launches = plan.timing()
    t_max_ms = max_over_ranks(dist, total_ms)
    plan.download()
    plan.close()
    e, d = 242, 240
    flops = 512 * svt_flops(e, d)
    out = {"workload": "config2 inputs, SHLR-SV (SPIRiT + virtual coils): 512 lifted 242x240 matrices/iter",
           "value": world * args.steps / (t_max_ms * 1e-3), "unit": "iterations/s",
           "ms_per_step": t_max_ms / args.steps, "gpu_launches_per_step": launches,
           "algorithmic_tflops_whole_step": flops / (t_max_ms / args.steps * 1e-3) / 1e12,
           "reference_cpu": {"value": 1.0 / 283.0, "unit": "iterations/s", "cores": 1,
                             "sample": "offline: the reference's 12-iteration fixture run (make_sv_golden.py)"}}
    if not args.no_e2e:
        barrier(dist)
        acfg.max_outer = cfg["outer"]
        t0 = time.perf_counter()
        st = A.SolveStats()
        A.shlr_pi_reconstruct(y, mask, g, hcfg, acfg, stats=st)
        t_e2e = max_over_ranks(dist, time.perf_counter() - t0)
        out["e2e"] = {"value": world * st.outer_iters / t_e2e, "unit": "iterations/s",
                      "h2d_bytes_per_step": int(y.size * 16 + mask.bits.size + g.weights.size * 16),
                      "d2h_bytes_per_step": int(y.size * 16),
                      "step": "one 50-iteration shlr_cuda_pi_reconstruct call with host buffers"}
    return out


def small_workload(args, dist, world, rank, fp32_peak):
    """BASELINE config 1 (the reference's CPU-runnable case): 128^2 x 8 coils,
    SHLR (no SPIRiT, no vc), R = 4 Gaussian Cartesian with 16 ACS lines,
    K = 9 -> 256 lifted 120 x 72 matrices per iteration, 30 iterations."""
    from paper_2107_11650_b200 import api as A
    from paper_2107_11650_b200 import synth
    ph = synth.pi_phantom(128, 128, 8)
    mask = A.mask_gauss_cartesian(128, 0.25, 16, synth.SEED_MASK)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    hcfg = A.HankelConfig(pencil=120)
    acfg = A.AdmmConfig(max_outer=max(30, args.warmup + args.steps), tol=1e-300)
    plan = A.PiPlan(y, mask, None, hcfg, acfg)
    plan.run(args.warmup)
    plan.sync()
    barrier(dist)
    plan.run(args.steps)
    plan.sync()
    _, total_ms, launches = plan.timing()
    t_max_ms = max_over_ranks(dist, total_ms)
    plan.close()
    out = {"workload": "config1: 128x128x8 coils, SHLR, R=4 Gaussian Cartesian + 16 ACS lines, K=9 "
                       "(pencil 120, 256 lifted 120x72 matrices/iter), 30 outer iterations",
           "value": world * args.steps / (t_max_ms * 1e-3), "unit": "iterations/s",
           "ms_per_step": t_max_ms / args.steps, "gpu_launches_per_step": launches}
    if not args.no_e2e:
        acfg.max_outer = 30
        A.shlr_pi_reconstruct(y, mask, None, hcfg, A.AdmmConfig(max_outer=1))
        t0 = time.perf_counter()
        A.shlr_pi_reconstruct(y, mask, None, hcfg, acfg)
        t_e2e = max_over_ranks(dist, time.perf_counter() - t0)
        out["e2e"] = {"value": world * 30 / t_e2e, "unit": "iterations/s",
                      "h2d_bytes_per_step": int(y.size * 16 + mask.bits.size), "d2h_bytes_per_step": int(y.size * 16),
                      "step": "one 30-iteration shlr_cuda_pi_reconstruct call with host buffers"}
    if rank == 0 and not args.no_cpu and os.path.exists(REF_DRIVER):
        tmp = tempfile.mkdtemp(prefix="shlr_ref1_")
        try:
            from paper_2107_11650_b200.cplx_io import write_cplx, write_mask
            write_cplx(y, os.path.join(tmp, "y.cplx"))
            write_mask(mask.bits, os.path.join(tmp, "m.cplx"))
            res = subprocess.run([REF_DRIVER, "pi", "y=y.cplx", "mask=m.cplx", "out=r", "pencil=120", "max_outer=2",
                                  "tol=1e-300", "replay=1", "time=1"], cwd=tmp, capture_output=True, text=True,
                                 timeout=600).stdout
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
        its = [float(ln.split("=")[1]) for ln in res.splitlines() if ln.startswith("iter_seconds=")]
        if its:
            out["cpu_baseline"] = {"value": 1.0 / statistics.mean(its), "unit": "iterations/s", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"oracle/_ref/ref_driver, {len(its)} config-1 iterations, one core"}
    return out


SWEEP_POINTS = [(n, nc, k) for n in (128, 256, 512) for nc in (1, 8, 32) for k in (7, 15, 31)]
HBM_GBS = 6552.0  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth) on this pool's B200s


def hbm_peak() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("hbm_gbs", HBM_GBS))
    except (OSError, ValueError):
        return HBM_GBS


def sweep_cpu_rates(points, budget_s: float = 2.0):
    """Host-core reference rate of every sweep point: oracle/_ref/ref_driver
    svt (the reference's lift_plain -> svt -> adjoint_lift_plain, unmodified,
    single-threaded) on the point's first matrices, `limit` sized for about
    `budget_s` seconds from a 1.5 GFLOP/s estimate; the points run
    concurrently, one process per host core."""
    from paper_2107_11650_b200 import synth
    from paper_2107_11650_b200.cplx_io import write_cplx
    if not os.path.exists(REF_DRIVER):
        return {}
    tmp = tempfile.mkdtemp(prefix="shlr_sweep_")
    jobs = []
    try:
        for n, nc, k in points:
            p = n - k + 1
            e, d = max(p, nc * k), min(p, nc * k)
            est = svt_flops(e, d) / 1.5e9
            limit = int(max(1, min(2 * n, np.ceil(budget_s / max(est, 1e-9)))))
            name = f"v{n}_{nc}_{k}.cplx"
            write_cplx(synth.sweep_vectors(n, nc, k, limit), os.path.join(tmp, name))
            jobs.append(((n, nc, k), [REF_DRIVER, "svt", f"vecs={name}", f"p={p}",
                                      f"tau={synth.sweep_tau(n, nc, k)}", "time=1", f"limit={limit}"]))
        out, running = {}, []
        ncpu = max(1, os.cpu_count() or 1)
        queue = list(jobs)
        while queue or running:
            while queue and len(running) < ncpu:
                key, cmd = queue.pop(0)
                running.append((key, subprocess.Popen(cmd, cwd=tmp, stdout=subprocess.PIPE, text=True,
                                                      env=dict(os.environ, OMP_NUM_THREADS="1"))))
            key, proc = running.pop(0)
            txt = proc.communicate(timeout=900)[0]
            for tok in txt.split():
                if tok.startswith("matrices="):
                    mats = int(tok.split("=")[1])
                elif tok.startswith("seconds="):
                    secs = float(tok.split("=")[1])
            out[key] = {"matrices_per_s_per_core": mats / secs, "sample": f"{mats} matrices, {secs:.2f} s, 1 core"}
        return out
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def sweep_workload(args, fp32_peak, cpu: bool = True):
    """BASELINE config 5 (batched Hankel-SVT unit): all 27 points N x Nc x K,
    batch = 2N slices, slices in {1, 16}; device-resident complex64 vectors in
    and out through the device-pointer C-ABI call (lift_plain -> svt ->
    adjoint_lift_plain, cold: the unit has no warm start), CUDA events around
    the call on its stream.  slices = 16 tiles the 2N seeded matrices of slice
    0 sixteen times (every matrix is solved independently; generating 32N
    distinct seeded matrices on the host would take minutes at N = 512,
    Nc = 32).  Beside each point: matrices/s, algorithmic TFLOP/s and its
    fraction of the FP32 peak, HBM GB/s of the sweep's own bytes (16 Nc N per
    matrix: vectors in, adjoint out) and its fraction of the measured copy
    bandwidth, and the host-core reference rate."""
    import torch
    from paper_2107_11650_b200 import api as A
    from paper_2107_11650_b200 import synth
    hbm = hbm_peak()
    cpu_rates = sweep_cpu_rates(SWEEP_POINTS) if cpu else {}
    ncpu = os.cpu_count() or 1
    out = []
    for n, nc, k in SWEEP_POINTS:
        p = n - k + 1
        e, d = max(p, nc * k), min(p, nc * k)
        v1 = synth.sweep_vectors(n, nc, k, 2 * n).astype(np.complex64)
        tau = synth.sweep_tau(n, nc, k)
        base = torch.from_numpy(v1).cuda()
        for slices in (1, 16):
            batch = 2 * n * slices
            rec = {"N": n, "Nc": nc, "K": k, "slices": slices, "matrix": f"{p}x{nc * k}", "batch": batch}
            try:
                dv = base.repeat(slices, 1, 1) if slices > 1 else base
                do = torch.empty_like(dv)
                st = torch.cuda.Stream()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st):
                    A.hankel_svt_batched_device(dv.data_ptr(), batch, nc, n, p, tau, do.data_ptr(), 0,
                                                st.cuda_stream)
                    st.synchronize()
                    reps = 3 if slices == 1 else 1
                    e0.record(st)
                    for _ in range(reps):
                        A.hankel_svt_batched_device(dv.data_ptr(), batch, nc, n, p, tau, do.data_ptr(), 0,
                                                    st.cuda_stream)
                    e1.record(st)
                    st.synchronize()
                ms = e0.elapsed_time(e1) / reps
                tf = batch * svt_flops(e, d) / (ms * 1e-3) / 1e12
                gbs = batch * 16.0 * nc * n / (ms * 1e-3) / 1e9
                rec.update({"ms": ms, "matrices_per_s": batch / (ms * 1e-3), "algorithmic_tflops": tf,
                            "frac_of_fp32_peak": tf / fp32_peak, "hbm_gbs": gbs, "frac_of_hbm": gbs / hbm,
                            "bound": "fp32" if tf / fp32_peak >= gbs / hbm else "hbm"})
                c = cpu_rates.get((n, nc, k))
                if c:
                    rec["cpu_reference"] = dict(c, all_cores_matrices_per_s=c["matrices_per_s_per_core"] * ncpu,
                                                cores=ncpu)
                    rec["speedup_vs_all_host_cores"] = rec["matrices_per_s"] / (c["matrices_per_s_per_core"] * ncpu)
                del dv, do
            except Exception as exc:  # geometry outside this build
                rec["unsupported"] = str(exc)[:160]
            out.append(rec)
        del base
        torch.cuda.empty_cache()
    return {"workload": "config5: batched Hankel-SVT unit, all 27 points N in {128,256,512} x Nc in {1,8,32} x "
                        "K in {7,15,31}, CN(0,1) + rank-K/2 exponentials, tau = sqrt(m)+sqrt(n), batch 2N x "
                        "slices, slices in {1,16}, cold solves",
            "host_cores": ncpu, "points": out}


def reference_arm(args, dist, rank, world):
    """The reference's own CPU implementation (stock shlr_pi_reconstruct, the
    unmodified proj/src compiled by oracle/Makefile) on the host cores: up to
    --ref-procs concurrent single-threaded processes (the reference has no
    threading; concurrent calls are safe).  Rank 0 only."""
    if rank != 0:
        return
    if not os.path.exists(REF_DRIVER):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/ref_driver not built (run __graft_entry__.build())"}))
        return
    procs = max(1, min(os.cpu_count() or 1, args.ref_procs))
    tmp = tempfile.mkdtemp(prefix="shlr_ref_")
    try:
        write_ref_inputs(tmp, CFG2)
        iters = max(2, min(args.steps, 50))
        res = run_reference(tmp, procs, iters, args.cpu_budget, CFG2)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    per_proc = [statistics.mean(r) for r in res if r]
    done = sum(len(r) for r in res)
    value = sum(1.0 / s for s in per_proc) if per_proc else 0.0
    out = {
        "metric": "recon iterations/sec (256x256x8 coils, SHLR-S, K=15)",
        "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 / value if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (fp64)",
        "data": "synthetic: seeded BASELINE phantom (10 ellipses, smooth phase, 8 Gaussian coils, 40 dB)",
        "impl": "reference",
        "config": bench_config(world),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": len(per_proc),
                         "kind": "reference",
                         "sample": f"{len(per_proc)} concurrent single-threaded processes of the stock "
                                   f"shlr_pi_reconstruct, {done} outer iterations timed through its log "
                                   f"lines (iterations 2.., setup excluded), budget {args.cpu_budget:.0f} s"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def relaunch_distributed(n: int) -> int:
    """`bench.py --gpus N` (N > 1) outside torchrun: launch N ranks on this
    node with torch.distributed.run (127.0.0.1 rendezvous) and wait."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config-3/4 side workloads")
    ap.add_argument("--cpu-budget", type=float, default=150.0)
    ap.add_argument("--ref-procs", type=int, default=16)
    args = ap.parse_args()
    if args.warmup < 1 or args.steps < 1:
        raise SystemExit("need --steps >= 1 and --warmup >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch_distributed(args.gpus))
    dist, rank, world, local = dist_setup()
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; timing {world} rank(s)", file=sys.stderr)
    try:
        if args.impl == "reference":
            reference_arm(args, dist, rank, world)
        else:
            gpu_arm(args, dist, rank, world, local)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
