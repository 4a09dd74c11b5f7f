"""SHLR-SV (SPIRiT + virtual coils) at the headline geometry against the
reference library's own run (tests/golden/sv_ref12.npz, make_sv_golden.py).

256 x 256 x 8 coils, K = 15: the lifted matrices are 242 x 240 -- tall
weighted lifts with d = 240, which run on the large-d subspace levels with
the adjoint weighting conj(wc) and the virtual-coil dagger applied to each
chunk's partial anti-diagonal sums (adjoint_lift_weighted,
operators.cpp:60-91).  The reference's kernels (its own calibration) feed
the run; images within 1e-4 relative L2 at every dumped iteration."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-4
ITERS = (1, 2, 5, 12)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "sv_ref12.npz")))


@pytest.fixture(scope="module")
def inputs(api, golden):
    import bench
    from paper_2107_11650_b200 import synth
    cfg = bench.CFG2
    ph = synth.pi_phantom(cfg["M"], cfg["N"], cfg["J"])
    mask = api.mask_gauss_cartesian(cfg["N"], cfg["rate"], cfg["acs"], synth.SEED_MASK)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    g = api.SpiritKernels(cfg["kernel"], cfg["J"], golden["kernels"])
    return y, mask, g, api.HankelConfig(pencil=cfg["N"] - cfg["K"] + 1)


def worst(x, golden, it):
    coils = [int(c) for c in golden["coils"]]
    return max(rel(x[:, :, coils], golden[f"x{it}_coils"]),
               rel(np.sqrt((np.abs(x) ** 2).sum(axis=2)), golden[f"rss{it}"]))


@pytest.mark.gpu
def test_sv_headline_geometry_drift_trace(gpu, golden, inputs):
    y, mask, g, hcfg = inputs
    A = gpu
    acfg = A.AdmmConfig(max_outer=12, tol=1e-300, enable_spirit=True, enable_vc=True)
    plan = A.PiPlan(y, mask, g, hcfg, acfg)
    done, errs = 0, {}
    for it in ITERS:
        plan.run(it - done)
        plan.sync()
        done = it
        x, st = plan.download()
        errs[it] = worst(x, golden, it)
    print("SHLR-SV drift trace", {k: f"{v:.2e}" for k, v in errs.items()})
    assert max(errs.values()) < TOL, errs


@pytest.mark.gpu
def test_sv_headline_geometry_public_call(gpu, golden, inputs):
    y, mask, g, hcfg = inputs
    A = gpu
    log = []
    x = A.shlr_pi_reconstruct(y, mask, g, hcfg,
                              A.AdmmConfig(max_outer=12, tol=1e-300, enable_spirit=True, enable_vc=True), log=log)
    assert worst(x, golden, 12) < TOL
    ref = [str(l) for l in golden["log"]]
    assert [l.split()[2] for l in log] == [l.split()[2] for l in ref]  # cg_iters
