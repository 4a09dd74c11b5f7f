"""Pack the reference's own BASELINE config-2 run into tests/golden/c2_ref50.npz.

The reference run is the unmodified reference library (oracle/_ref, built by
oracle/Makefile from /root/reference/proj/src) driven by oracle/ref_driver.
Every input is made without the product: the image by the harness generator
(numpy), the mask by the reference's own generator, the SPIRiT kernels by the
reference's own spirit_calibrate (spirit.cpp:22-94) inside `ref_driver pi`
(no kernels= argument: it calibrates from the ACS block and writes them out):

    python -c 'import sys; sys.path.insert(0, "."); from paper_2107_11650_b200 import cplx_io as io, synth; \
        io.write_cplx(synth.pi_phantom(256, 256, 8).kspace, "DIR/y.cplx")'
    oracle/_ref/ref_driver mask kind=gauss n=256 rate=0.2 acs=24 seed=11650 out=DIR/m.cplx
    oracle/_ref/ref_driver pi y=DIR/y.cplx mask=DIR/m.cplx out=DIR/ref50 spirit=1 acs=24 pencil=242 \
        max_outer=50 tol=1e-300 sv_iters=1,2,5,10,50 x_iters=1,2,5,10,50 time=1

(config 2: 256 x 256 x 8 coils, R = 5 Gaussian Cartesian mask with 24 ACS
lines, K = 15 -> pencil 242, SPIRiT 5 x 5, defaults for lambda / lambda1 /
beta / tau; about 35 min on one host core).  `x_iters` / `sv_iters` use the
instrumented replay, which tests/test_ref_driver.py pins bitwise to the stock
shlr_pi_reconstruct.

The fixture keeps the reference's kernels, the image after 50 iterations
(complex64), coils 0 and 5 plus the root-sum-of-squares image after
iterations 1, 2, 5 and 10, the singular values of L + D/beta at those
iterations, and the relchange trace.

    python tests/golden/make_c2_golden.py DIR
"""
import os
import re
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2107_11650_b200 import cplx_io as io  # noqa: E402

ITERS = (1, 2, 5, 10, 50)
COILS_KEPT = (0, 5)


def main(d: str) -> None:
    out = {"kernels": io.read_cplx(os.path.join(d, "ref50.kernels.cplx")),
           "mask": io.read_cplx(os.path.join(d, "m.cplx")).real.astype(np.uint8).reshape(-1),
           "coils": np.array(COILS_KEPT)}
    for it in ITERS:
        px, ps = os.path.join(d, f"ref50.x{it}.cplx"), os.path.join(d, f"ref50.sv{it}.cplx")
        if not os.path.exists(px):
            continue
        x = io.read_cplx(px)
        if it == 50:
            out["x50"] = x.astype(np.complex64)
        out[f"x{it}_coils"] = x[:, :, list(COILS_KEPT)].astype(np.complex64)
        out[f"rss{it}"] = np.sqrt((np.abs(x) ** 2).sum(axis=2)).astype(np.float32)
        out[f"sv{it}"] = io.read_cplx(ps).real.astype(np.float32)
    rel = []
    for line in open(os.path.join(d, "ref50.log")):
        m = re.match(r"iter=(\d+) relchange=(\S+)", line)
        if m:
            rel.append(float(m.group(2)))
    out["relchange"] = np.array(rel)
    out["log"] = np.array([ln.strip() for ln in open(os.path.join(d, "ref50.log")) if ln.strip()])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_ref50.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), sorted(out))


if __name__ == "__main__":
    main(sys.argv[1])
