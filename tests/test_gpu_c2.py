"""BASELINE config 2 at full size against the reference library's own run.

tests/golden/c2_ref50.npz holds the unmodified reference (oracle/_ref +
oracle/ref_driver, see tests/golden/make_c2_golden.py) run for 50 ADMM
iterations on 256 x 256 x 8 coils, R = 5, K = 15 (242 x 120 block-Hankel
matrices, 512 per sweep), SPIRiT, with every input made without the product:
the mask by the reference's generator, the SPIRiT kernels by the reference's
own spirit_calibrate.  It keeps the image and the singular values of
L + D/beta after iterations 1, 2, 5, 10 and 50 (the per-iteration drift trace)
and the reference's kernels.

Bars (BASELINE north_star): image and singular values within 1e-4 relative
L2; the mask bit-exact; the calibrations (setup, FP64) within 1e-7 of the
reference's kernels (ridge-by-Cholesky against the reference's SVD Tikhonov
filter: 3.8e-9 measured)."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-4
CAL_TOL = 1e-7
ITERS = (1, 2, 5, 10, 50)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "c2_ref50.npz")))


@pytest.fixture(scope="module")
def inputs(api, golden):
    """Config-2 inputs with the REFERENCE's kernels (the run's own)."""
    import bench
    from paper_2107_11650_b200 import synth
    cfg = bench.CFG2
    A = api
    ph = synth.pi_phantom(cfg["M"], cfg["N"], cfg["J"])
    mask = A.mask_gauss_cartesian(cfg["N"], cfg["rate"], cfg["acs"], synth.SEED_MASK)
    y = np.where(mask.bits[0][None, :, None].astype(bool), ph.kspace, 0)
    g = A.SpiritKernels(cfg["kernel"], cfg["J"], golden["kernels"])
    return y, mask, g, A.HankelConfig(pencil=cfg["N"] - cfg["K"] + 1)


def check_image(x, golden, it):
    coils = [int(c) for c in golden["coils"]]
    if it == 50 and "x50" in golden:
        assert rel(x, golden["x50"]) < TOL
    assert rel(x[:, :, coils], golden[f"x{it}_coils"]) < TOL
    assert rel(np.sqrt((np.abs(x) ** 2).sum(axis=2)), golden[f"rss{it}"]) < TOL


def test_c2_mask_is_the_reference_mask(api, golden, inputs):
    assert np.array_equal(inputs[1].bits.reshape(-1), golden["mask"])


def test_c2_host_calibration_matches_reference(api, golden, inputs):
    """Host FP64 calibration (the product's setup path) against the kernels the
    reference's own spirit_calibrate produced for this run (spirit.cpp:22-94)."""
    import bench
    y, _, _, _ = inputs
    a0, a1 = api.acs_range(256, bench.CFG2["acs"])
    g = api.spirit_calibrate(y[:, a0:a1, :], 5, 1e-4)
    err = float(np.abs(g.weights - golden["kernels"]).max() / np.abs(golden["kernels"]).max())
    assert err < CAL_TOL, err


def test_c2_oracle_calibration_matches_reference(golden, inputs):
    """The oracle's restatement of spirit_calibrate is pinned to the reference too."""
    import shlr_oracle as O
    y = inputs[0]
    a0, a1 = O.acs_range(256, 24)
    g = O.spirit_calibrate(y[:, a0:a1, :], 5, 1e-4)
    err = float(np.abs(g.weights - golden["kernels"]).max() / np.abs(golden["kernels"]).max())
    assert err < CAL_TOL, err


@pytest.mark.gpu
def test_c2_device_calibration_matches_reference(gpu, golden, inputs):
    """SPIRiT calibration on the device (FP64, shlr_cuda_spirit_calibrate)
    against the reference's own kernels."""
    y = inputs[0]
    a0, a1 = gpu.acs_range(256, 24)
    g = gpu.spirit_calibrate(y[:, a0:a1, :], 5, 1e-4, device=True)
    err = float(np.abs(g.weights - golden["kernels"]).max() / np.abs(golden["kernels"]).max())
    assert err < CAL_TOL, err


@pytest.mark.gpu
@pytest.mark.parametrize("it", ITERS)
def test_c2_parity_vs_reference(gpu, golden, inputs, it):
    """One-shot public call for `it` iterations: the image and (debug hook:
    the full eigen-solver at that iteration) the singular values of L + D/beta."""
    if f"x{it}_coils" not in golden:
        pytest.fail(f"c2_ref50.npz has no iteration {it}")
    y, mask, g, hcfg = inputs
    A = gpu
    acfg = A.AdmmConfig(max_outer=it, tol=1e-300, enable_spirit=True)
    log, svs = [], []
    x = A.shlr_pi_reconstruct(y, mask, g, hcfg, acfg, log=log, debug_sv_iter=it, sv_out=svs)
    assert rel(svs[0], golden[f"sv{it}"]) < TOL
    check_image(x, golden, it)
    ref_log = [str(l) for l in golden["log"]]
    assert len(ref_log) >= it, "c2_ref50.npz log is incomplete"
    assert [l.split()[2] for l in log] == [l.split()[2] for l in ref_log[:it]]  # cg_iters


@pytest.mark.gpu
def test_c2_resident_plan_drift_trace(gpu, golden, inputs):
    """The bench path (resident plan, CUDA graph, warm-started subspace SVT)
    downloaded after iterations 1, 2, 5, 10 and 50 of one run: every point of
    the trace within 1e-4 of the reference's image at that iteration."""
    y, mask, g, hcfg = inputs
    A = gpu
    plan = A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True))
    done, worst = 0, {}
    for it in ITERS:
        if f"x{it}_coils" not in golden:
            continue
        plan.run(it - done)
        plan.sync()
        done = it
        x, st = plan.download()
        assert st.outer_iters == it
        coils = [int(c) for c in golden["coils"]]
        worst[it] = max(rel(x[:, :, coils], golden[f"x{it}_coils"]),
                        rel(np.sqrt((np.abs(x) ** 2).sum(axis=2)), golden[f"rss{it}"]))
    print("drift trace", {k: f"{v:.2e}" for k, v in worst.items()})
    assert max(worst.values()) < TOL, worst


@pytest.mark.gpu
def test_c2_device_calibration_end_to_end(gpu, golden, inputs):
    """The user flow on the GPU alone: device calibration from the ACS block,
    then 50 iterations -- against the reference's run (its own calibration)."""
    if "x50" not in golden:
        pytest.fail("c2_ref50.npz has no iteration 50")
    y, mask, _, hcfg = inputs
    A = gpu
    a0, a1 = A.acs_range(256, 24)
    g = A.spirit_calibrate(y[:, a0:a1, :], 5, 1e-4, device=True)
    x = A.shlr_pi_reconstruct(y, mask, g, hcfg, A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True))
    assert rel(x, golden["x50"]) < TOL


@pytest.mark.gpu
def test_c2_runs_are_bitwise_repeatable(gpu, inputs):
    """Two independent plans at the headline size give bitwise-equal images
    (test_solvers.cpp's determinism contract at full size): the co-located
    SVT CTAs, the read-modify-written adjoints, the bulk-copy SPIRiT stage and
    the last-CTA reductions leave no ordering to chance."""
    A = gpu
    y, mask, g, hcfg = inputs
    out = []
    for _ in range(2):
        plan = A.PiPlan(y, mask, g, hcfg, A.AdmmConfig(max_outer=12, tol=1e-300, enable_spirit=True))
        plan.run(12)
        plan.sync()
        x, _ = plan.download()
        plan.close()
        out.append(x)
    assert np.array_equal(out[0], out[1])
