"""The reference-side harness (oracle/_ref/ref_driver) is itself pinned to the
reference library's stock entry points.

`ref_driver pi ... replay=1` (and `sv_iters=` / `x_iters=`) runs `pi_replay`,
a builder-written copy of the `shlr_pi_reconstruct` loop
(proj/src/solvers.cpp:151-188) over the reference's public primitives, used to
dump the singular values / intermediate images of the golden fixtures.  These
tests prove that copy is bitwise equal to the stock library call on the same
inputs, with and without SPIRiT and virtual coils, and that the stock call
timed through its own log lines (`time=1`, the bench's reference arm) writes
the same log and image.  CPU only (test infrastructure)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

pytestmark = pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (make -C oracle)")


def run(cwd, *args):
    r = subprocess.run([REF, *args], cwd=cwd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return r.stdout


@pytest.fixture(scope="module")
def inputs(tmp_path_factory):
    from paper_2107_11650_b200 import cplx_io as io
    from paper_2107_11650_b200 import synth
    d = tmp_path_factory.mktemp("refdrv")
    io.write_cplx(synth.pi_phantom(32, 32, 4).kspace, str(d / "y.cplx"))
    run(d, "mask", "kind=gauss", "n=32", "rate=0.5", "acs=8", "seed=11650", "out=m.cplx")
    return d


@pytest.mark.parametrize("spirit,vc", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_replay_bitwise_equals_stock_shlr_pi_reconstruct(inputs, spirit, vc):
    common = ["y=y.cplx", "mask=m.cplx", f"spirit={spirit}", f"vc={vc}", "acs=8", "kernel=3",
              "pencil=20", "max_outer=4", "tol=1e-300"]
    tag = f"s{spirit}v{vc}"
    run(inputs, "pi", *common, f"out=stock_{tag}")
    run(inputs, "pi", *common, f"out=replay_{tag}", "replay=1", "x_iters=4")
    stock = (inputs / f"stock_{tag}.x.cplx").read_bytes()
    assert stock == (inputs / f"replay_{tag}.x.cplx").read_bytes()
    assert stock == (inputs / f"replay_{tag}.x4.cplx").read_bytes()  # x_iters dump = the result
    assert (inputs / f"stock_{tag}.log").read_text() == (inputs / f"replay_{tag}.log").read_text()


def test_stock_call_timed_through_its_log(inputs):
    common = ["y=y.cplx", "mask=m.cplx", "spirit=1", "acs=8", "kernel=3", "pencil=20", "max_outer=3",
              "tol=1e-300"]
    out = run(inputs, "pi", *common, "out=timed", "time=1")
    run(inputs, "pi", *common, "out=plain")
    lines = out.splitlines()
    assert lines[0].startswith("first_iter_seconds=")
    assert sum(ln.startswith("iter_seconds=") for ln in lines) == 2
    assert (inputs / "timed.x.cplx").read_bytes() == (inputs / "plain.x.cplx").read_bytes()
    assert (inputs / "timed.log").read_text() == (inputs / "plain.log").read_text()


def test_reference_mask_generator_matches_product(inputs, api):
    """The reference arm builds its mask with the reference's own generator
    (`ref_driver mask`); it is the product's mask bit for bit."""
    from paper_2107_11650_b200 import cplx_io as io
    bits = io.read_cplx(str(inputs / "m.cplx")).real.astype(np.uint8).reshape(-1)
    assert np.array_equal(bits, api.mask_gauss_cartesian(32, 0.5, 8, 11650).bits.reshape(-1))
