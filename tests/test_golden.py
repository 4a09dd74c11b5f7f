"""Golden fixtures produced by the reference itself (tests/golden/make_golden.py
runs oracle/_ref/ref_driver = proj/src/*.cpp unmodified).

CPU: the numpy oracle reproduces every fixture (pins the restatement).
GPU: the B200 path reproduces every fixture: image and singular values
within 1e-4 relative L2 (BASELINE north_star), log lines and stats equal,
masks bit-exact, lift index maps bit-exact."""
import glob
import os

import numpy as np
import pytest

import shlr_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PI_CASES = sorted(glob.glob(os.path.join(GOLDEN, "pi_*.npz")))
SVT_CASES = sorted(glob.glob(os.path.join(GOLDEN, "svt_*.npz")))
PARAM_CASES = sorted(glob.glob(os.path.join(GOLDEN, "param_*.npz")))
TOL = 1e-4  # BASELINE north_star: relative L2 for images and singular values


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def load(path):
    return dict(np.load(path, allow_pickle=True))


def log_values(lines):
    out = []
    for ln in lines:
        kv = dict(t.split("=") for t in str(ln).split())
        out.append((int(kv["iter"]), float(kv["relchange"]), int(kv["cg_iters"]), float(kv["cg_res"])))
    return out


def oracle_pi(g):
    m, n, j = g["y"].shape
    mask = O.SamplingMask(1, n, g["mask"])
    kern = O.SpiritKernels(int(g["kernel"]), j, g["kernels"]) if bool(g["spirit"]) else None
    acfg = O.AdmmConfig(max_outer=int(g["max_outer"]), tol=1e-300, enable_vc=bool(g["vc"]),
                        enable_spirit=bool(g["spirit"]))
    return O.shlr_pi_reconstruct(g["y"], mask, kern, O.HankelConfig(pencil=int(g["pencil"])), acfg,
                                 sv_iters=tuple(int(i) for i in g["sv_iters"]))


@pytest.mark.parametrize("path", PI_CASES, ids=os.path.basename)
def test_oracle_matches_reference_pi(path):
    g = load(path)
    x, st = oracle_pi(g)
    assert rel(x, g["x"]) < 1e-9
    assert st.log == [str(s) for s in g["log"]]
    for it in g["sv_iters"]:
        sr, sc = st.singular_values[int(it)]
        ref = g[f"sv{int(it)}"]
        assert rel(np.concatenate([sr, sc]), ref) < 1e-10


@pytest.mark.parametrize("path", SVT_CASES, ids=os.path.basename)
def test_oracle_matches_reference_svt(path):
    g = load(path)
    adj, sv = O.hankel_svt_unit(g["vecs"], int(g["p"]), float(g["tau"]))
    assert rel(adj, g["adj"]) < 1e-10
    assert rel(sv, g["sv"]) < 1e-12


def param_configs(g, M):
    """AdmmConfig / HankelConfig of a param fixture (defaults + the fixture's extra keys)."""
    extra = dict(str(e).split("=", 1) for e in g["extra"])
    acfg = M.AdmmConfig(max_outer=int(g["max_outer"]), tol=float(g["tol"]), enable_vc=bool(g["vc"]),
                        lam2=float(extra.get("lambda2", 2.0)))
    hcfg = M.HankelConfig(pencil=int(g["pencil"]), pencil_param=int(g["pencil_param"]))
    return acfg, hcfg


@pytest.mark.parametrize("path", PARAM_CASES, ids=os.path.basename)
def test_oracle_matches_reference_param(path):
    """Parameter imaging: shlr_param_reconstruct_slice (solvers.cpp:193-298) and
    recon_param_dataset (parammap.cpp:21-54) against the reference's own run."""
    g = load(path)
    acfg, hcfg = param_configs(g, O)
    n, l = g["mask"].shape
    mask = O.SamplingMask(n, l, g["mask"])
    if g["y"].ndim == 3:
        x, st = O.shlr_param_reconstruct_slice(g["y"], mask, hcfg, acfg)
        total, log = st.outer_iters, st.log
    else:
        x, total = O.recon_param_dataset(g["y"], mask, hcfg, acfg)
        log = None
    assert rel(x, g["x"]) < 1e-9
    assert total == int(g["outer_iters"])
    if log is not None:
        assert log == [str(s) for s in g["log"]]


def test_oracle_masks_bit_exact():
    g = load(os.path.join(GOLDEN, "masks.npz"))
    for i in range(len([k for k in g if k.startswith("bits")])):
        kind, n, rate, acs, seed = g[f"spec{i}"]
        if kind == "gauss":
            m = O.mask_gauss_cartesian(int(n), float(rate), int(acs), int(seed))
        else:
            m = O.mask_random2d(int(n), int(n), float(rate), int(acs), int(seed))
        assert np.array_equal(m.bits.reshape(g[f"bits{i}"].shape), g[f"bits{i}"])


def test_product_masks_bit_exact(api):
    """Host-side mask generators of the C-ABI (no GPU needed)."""
    g = load(os.path.join(GOLDEN, "masks.npz"))
    for i in range(len([k for k in g if k.startswith("bits")])):
        kind, n, rate, acs, seed = g[f"spec{i}"]
        if kind == "gauss":
            m = api.mask_gauss_cartesian(int(n), float(rate), int(acs), int(seed))
        else:
            m = api.mask_random2d(int(n), int(n), float(rate), int(acs), int(seed))
        assert np.array_equal(m.bits.reshape(g[f"bits{i}"].shape), g[f"bits{i}"])


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("path", PI_CASES, ids=os.path.basename)
def test_gpu_pi_matches_reference(gpu, path):
    A = gpu
    g = load(path)
    m, n, j = g["y"].shape
    kern = A.SpiritKernels(int(g["kernel"]), j, g["kernels"]) if bool(g["spirit"]) else None
    acfg = A.AdmmConfig(max_outer=int(g["max_outer"]), tol=1e-300, enable_vc=bool(g["vc"]),
                        enable_spirit=bool(g["spirit"]))
    last = int(g["sv_iters"][-1])
    log, st, svs = [], A.SolveStats(), []
    x = A.shlr_pi_reconstruct(g["y"], A.SamplingMask(1, n, g["mask"]), kern,
                              A.HankelConfig(pencil=int(g["pencil"])), acfg, log=log, stats=st,
                              debug_sv_iter=last, sv_out=svs)
    assert rel(x, g["x"]) < TOL
    assert st.outer_iters == int(g["max_outer"])
    got, want = log_values(log), log_values(g["log"])
    assert [(a[0], a[2]) for a in got] == [(b[0], b[2]) for b in want]  # iter, cg_iters exact
    for a, b in zip(got, want):
        assert abs(a[1] - b[1]) <= 1e-3 * abs(b[1]) + 1e-12    # relchange (3 sig. digits)
    assert rel(svs[0], g[f"sv{last}"]) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("path", SVT_CASES, ids=os.path.basename)
def test_gpu_svt_matches_reference(gpu, path):
    A = gpu
    g = load(path)
    adj, sv = A.hankel_svt_batched(g["vecs"], int(g["p"]), float(g["tau"]))
    assert rel(adj, g["adj"]) < TOL
    assert rel(sv, g["sv"]) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("path", [0, 1, 2])
@pytest.mark.parametrize("n,p,coils,vc", [(20, 7, 3, False), (20, 7, 3, True), (21, 8, 2, True),
                                          (256, 242, 8, False), (256, 23, 4, True), (256, 242, 8, True),
                                          (180, 162, 4, True), (15, 5, 2, True)])
def test_gpu_lift_index_map_bit_exact(gpu, n, p, coils, vc, path):
    """The kernels' own lift stage -- run on index-encoded spectra and decoded
    (shlr_cuda_lift_index_map_path): path 0 the full solver's lift_elem, 1 the
    subspace solver's lift_tab, 2 the large-d lift_global -- gives the
    reference lift_weighted order (operators.cpp:36-56) bit for bit: regular
    blocks, then vc blocks reading the dagger index (hankel.cpp:99-113),
    conjugated.  Tall and wide, odd and even lengths."""
    A = gpu
    got = A.lift_index_map(n, p, coils, vc, path)
    q = n - p + 1
    blocks = coils * (2 if vc else 1)
    want = np.zeros((p, blocks * q, 3), np.int32)
    dag = O.dagger_index(n)
    for i in range(p):
        for c in range(blocks * q):
            b, t = divmod(c, q)
            if b < coils:
                want[i, c] = (b, i + t, 0)
            else:
                want[i, c] = (b - coils, dag[i + t], 1)
    assert np.array_equal(got, want)
    # and the map reproduces the oracle's lift of identity-weighted spectra
    rng = np.random.default_rng(n)
    s = rng.normal(size=(coils, n)) + 1j * rng.normal(size=(coils, n))
    lifted = np.where(got[..., 2] == 1, np.conj(s[got[..., 0], got[..., 1]]), s[got[..., 0], got[..., 1]])
    blocks_o = [s] + ([O.virtual_coil_dagger(s)] if vc else [])
    wb = np.concatenate(blocks_o, axis=0)
    ref = np.moveaxis(O.hankel_lift(wb, p), 0, 1).reshape(p, blocks * q)
    assert np.array_equal(lifted, ref)
