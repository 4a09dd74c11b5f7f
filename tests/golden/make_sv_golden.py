"""Pack the reference's own SHLR-SV run at the headline geometry into
tests/golden/sv_ref12.npz.

SHLR-SV = SPIRiT + virtual coils (the paper's most accurate variant,
PAPER.md:168,175) on the config-2 inputs: 256 x 256 x 8 coils, R = 5
Gaussian Cartesian mask with 24 ACS lines, K = 15 -> pencil 242, so the
lifted matrices are 242 x 240 (8 coils + 8 virtual coils x 15): tall
weighted lifts with d = 240, the large-d subspace levels.  Inputs are made
without the product (harness generator, reference mask generator, the
reference's own spirit_calibrate inside ref_driver):

    (DIR/y.cplx, DIR/m.cplx as in make_c2_golden.py)
    oracle/_ref/ref_driver pi y=DIR/y.cplx mask=DIR/m.cplx out=DIR/sv12 spirit=1 vc=1 acs=24 \\
        pencil=242 max_outer=12 tol=1e-300 x_iters=1,2,5,12 time=1

(about 57 min on one host core: 280 s per iteration).  Keeps the reference's
kernels, coils 0 and 5 plus the root-sum-of-squares image after iterations
1, 2, 5 and 12, and the log.

    python tests/golden/make_sv_golden.py DIR
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2107_11650_b200 import cplx_io as io  # noqa: E402

ITERS = (1, 2, 5, 12)
COILS_KEPT = (0, 5)


def main(d: str) -> None:
    out = {"kernels": io.read_cplx(os.path.join(d, "sv12.kernels.cplx")), "coils": np.array(COILS_KEPT)}
    for it in ITERS:
        x = io.read_cplx(os.path.join(d, f"sv12.x{it}.cplx"))
        out[f"x{it}_coils"] = x[:, :, list(COILS_KEPT)].astype(np.complex64)
        out[f"rss{it}"] = np.sqrt((np.abs(x) ** 2).sum(axis=2)).astype(np.float32)
    out["log"] = np.array([ln.strip() for ln in open(os.path.join(d, "sv12.log")) if ln.strip()])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sv_ref12.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), sorted(out))


if __name__ == "__main__":
    main(sys.argv[1])
