"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself:
oracle/_ref/ref_driver is the reference's own proj/src/*.cpp (unmodified,
compiled against the builder's Eigen subset by oracle/Makefile).  Run in the
build container (needs oracle/_ref built):

    python tests/golden/make_golden.py

Each .npz holds the seeded inputs and the reference outputs (image, per-
iteration log lines, singular values of L + D/beta at the dumped iterations,
masks, SPIRiT kernels).  Small sizes only: the fixtures are committed.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2107_11650_b200.cplx_io import read_cplx, write_cplx, write_mask  # noqa: E402

DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def run(args, cwd):
    subprocess.run([DRIVER] + args, cwd=cwd, check=True, stdout=subprocess.DEVNULL)


def pi_case(name, m, n, j, pencil, vc, spirit, seed, max_outer=4, sv_iters=(1, 4), rate=0.5,
            acs=6, kernel=3):
    rng = np.random.default_rng(seed)
    y = rng.standard_normal((m, n, j)) + 1j * rng.standard_normal((m, n, j))
    with tempfile.TemporaryDirectory() as tmp:
        run(["mask", "kind=gauss", f"n={n}", f"rate={rate}", f"acs={acs}", f"seed={seed}",
             "out=m.cplx"], tmp)
        bits = read_cplx(os.path.join(tmp, "m.cplx")).real.astype(np.uint8)
        write_cplx(y, os.path.join(tmp, "y.cplx"))
        args = ["pi", "y=y.cplx", "mask=m.cplx", "out=o", f"vc={int(vc)}", f"spirit={int(spirit)}",
                f"pencil={pencil}", f"max_outer={max_outer}", "tol=1e-300", f"acs={acs}",
                f"kernel={kernel}", "sv_iters=" + ",".join(map(str, sv_iters))]
        run(args, tmp)
        out = dict(y=y, mask=bits, pencil=pencil, vc=vc, spirit=spirit, max_outer=max_outer,
                   sv_iters=np.array(sv_iters), acs=acs, kernel=kernel, rate=rate, seed=seed,
                   x=read_cplx(os.path.join(tmp, "o.x.cplx")),
                   log=np.array(open(os.path.join(tmp, "o.log")).read().splitlines()))
        for it in sv_iters:
            out[f"sv{it}"] = read_cplx(os.path.join(tmp, f"o.sv{it}.cplx")).real
        if spirit:
            out["kernels"] = read_cplx(os.path.join(tmp, "o.kernels.cplx"))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def svt_case(name, b, nc, n, p, tau, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((b, nc, n)) + 1j * rng.standard_normal((b, nc, n))
    # low-rank signal so the threshold bites
    t = np.arange(n)
    for r in range(3):
        w = rng.uniform(0, 2 * np.pi, size=(b, 1, 1))
        v += 4 * (rng.standard_normal((b, nc, 1)) + 1j * rng.standard_normal((b, nc, 1))) * np.exp(1j * w * t)
    with tempfile.TemporaryDirectory() as tmp:
        write_cplx(v, os.path.join(tmp, "v.cplx"))
        run(["svt", "vecs=v.cplx", f"p={p}", f"tau={tau!r}", "out=o"], tmp)
        out = dict(vecs=v, p=p, tau=tau, adj=read_cplx(os.path.join(tmp, "o.adj.cplx")),
                   sv=read_cplx(os.path.join(tmp, "o.sv.cplx")).real)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def param_masks(n, l, rate, acs, seed):
    """N x L parameter-imaging mask: echo e's column is mask_gauss_cartesian(n, rate, acs,
    seed + e) from the reference's own generator (SURVEY 8 mapping table, config 4)."""
    cols = []
    with tempfile.TemporaryDirectory() as tmp:
        for e in range(l):
            run(["mask", "kind=gauss", f"n={n}", f"rate={rate!r}", f"acs={acs}", f"seed={seed + e}",
                 "out=m.cplx"], tmp)
            cols.append(read_cplx(os.path.join(tmp, "m.cplx")).real.astype(np.uint8).reshape(-1))
    return np.stack(cols, axis=1)


def param_case(name, shape, vc, seed, max_outer=4, pencil=0, pencil_param=0, tol=1e-300, rate=0.4,
               acs=4, extra=()):
    """shape (N, L, J) -> shlr_param_reconstruct_slice; (M, N, L, J) -> recon_param_dataset."""
    rng = np.random.default_rng(seed)
    y = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    n, l = shape[-3], shape[-2]
    bits = param_masks(n, l, rate, acs, seed)
    with tempfile.TemporaryDirectory() as tmp:
        write_cplx(y, os.path.join(tmp, "y.cplx"))
        write_mask(bits, os.path.join(tmp, "m.cplx"))
        args = ["param", "y=y.cplx", "mask=m.cplx", "out=o", f"vc={int(vc)}", f"pencil={pencil}",
                f"pencil_param={pencil_param}", f"max_outer={max_outer}", f"tol={tol!r}"] + list(extra)
        run(args, tmp)
        stats = dict(ln.split("=", 1) for ln in open(os.path.join(tmp, "o.stats")).read().split()
                     if "=" in ln)
        out = dict(y=y, mask=bits, pencil=pencil, pencil_param=pencil_param, vc=vc, max_outer=max_outer,
                   tol=tol, seed=seed, extra=np.array(list(extra), dtype=object),
                   x=read_cplx(os.path.join(tmp, "o.x.cplx")),
                   log=np.array(open(os.path.join(tmp, "o.log")).read().splitlines()),
                   outer_iters=int(stats.get("outer_iters", -1)))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def mask_case():
    specs = [("gauss", 256, 0.2, 24, 11650), ("gauss", 128, 0.25, 16, 11650),
             ("gauss", 256, 0.34, 22, 42), ("gauss", 256, 1.0 / 6.0, 16, 11651),
             ("random2d", 64, 0.18, 12, 7), ("random2d", 256, 1.0 / 6.0, 24, 11650)]
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for i, (kind, n, rate, acs, seed) in enumerate(specs):
            run(["mask", f"kind={kind}", f"n={n}", f"rate={rate!r}", f"acs={acs}", f"seed={seed}",
                 f"out=m{i}.cplx"], tmp)
            out[f"bits{i}"] = read_cplx(os.path.join(tmp, f"m{i}.cplx")).real.astype(np.uint8)
            out[f"spec{i}"] = np.array([kind, n, rate, acs, seed], dtype=object)
    np.savez_compressed(os.path.join(HERE, "masks.npz"), **out)


def main():
    if not os.path.exists(DRIVER):
        raise SystemExit("build oracle/_ref first (make -C oracle)")
    if sys.argv[1:] == ["param"]:
        return param_cases()
    for vc in (0, 1):
        for sp in (0, 1):
            pi_case(f"pi_24x24x3_p9_vc{vc}_s{sp}", 24, 24, 3, 9, vc, sp, seed=10 + 2 * vc + sp)
    pi_case("pi_24x24x2_p18_tall", 24, 24, 2, 18, 0, 0, seed=21)
    pi_case("pi_32x32x2_default_pencil", 32, 32, 2, 0, 1, 0, seed=22, sv_iters=(1, 3), max_outer=3)
    pi_case("pi_15x15x2_odd", 15, 15, 2, 6, 1, 1, seed=23, acs=5, rate=0.6)
    pi_case("pi_64x64x4_long", 64, 64, 4, 49, 0, 1, seed=24, max_outer=12, sv_iters=(1, 12),
            rate=0.4, acs=12, kernel=5)
    svt_case("svt_tall_40_3_p31", 6, 3, 40, 31, 3.0, seed=31)
    svt_case("svt_wide_64_4_p20", 5, 4, 64, 20, 6.0, seed=32)
    svt_case("svt_120x120_sq", 4, 8, 134, 120, 20.0, seed=33)
    mask_case()
    param_cases()
    print("golden fixtures written to", HERE)


def param_cases():
    param_case("param_slice_24x8x2_vc0", (24, 8, 2), 0, seed=41, pencil=17)
    param_case("param_slice_24x8x2_vc1", (24, 8, 2), 1, seed=42, pencil=17)
    param_case("param_slice_20x12x3_default", (20, 12, 3), 1, seed=43, max_outer=3)
    param_case("param_slice_16x9x2_early_stop", (16, 9, 2), 0, seed=44, max_outer=40, tol=1e-3,
               pencil=11)
    param_case("param_dataset_5x20x9x2_vc1", (5, 20, 9, 2), 1, seed=45, max_outer=3, pencil=14)
    param_case("param_dataset_4x16x10x2_stop", (4, 16, 10, 2), 0, seed=46, max_outer=30, tol=2e-3,
               pencil=11, extra=("lambda2=0.5",))


if __name__ == "__main__":
    main()
