"""Pack the reference's own BASELINE config-2 run into tests/golden/c2_ref50.npz.

The reference run is the unmodified reference library (oracle/_ref, built by
oracle/Makefile from /root/reference/proj/src) driven by oracle/ref_driver on
the config-2 inputs that bench.make_inputs() generates (256 x 256 x 8 coils,
R = 5 Gaussian Cartesian mask with 24 ACS lines, K = 15 -> pencil 242, SPIRiT
5 x 5 kernels, defaults for lambda / lambda1 / beta / tau):

    python -c 'import bench, numpy as np; from paper_2107_11650_b200 import cplx_io as io; \
        y, m, g, h = bench.make_inputs(); io.write_cplx(y, "DIR/y.cplx"); \
        io.write_cplx(np.asarray(m.bits, float), "DIR/m.cplx"); io.write_cplx(g.weights, "DIR/k.cplx")'
    oracle/_ref/ref_driver pi y=y.cplx mask=m.cplx kernels=k.cplx out=DIR/ref50 spirit=1 \
        pencil=242 max_outer=50 tol=1e-300 sv_iters=1,2,5,10,50 time=1

(about 45 min on one host core).  Usage: python tests/golden/make_c2_golden.py DIR
"""
import os
import re
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2107_11650_b200 import cplx_io as io  # noqa: E402


def main(d: str) -> None:
    x = io.read_cplx(os.path.join(d, "ref50.x.cplx"))
    k = io.read_cplx(os.path.join(d, "k.cplx"))
    sv = {it: io.read_cplx(os.path.join(d, f"ref50.sv{it}.cplx")).real for it in (1, 50)}
    rel = []
    for line in open(os.path.join(d, "ref50.log")):
        m = re.match(r"iter=(\d+) relchange=(\S+)", line)
        if m:
            rel.append(float(m.group(2)))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_ref50.npz")
    np.savez_compressed(out, x50=x.astype(np.complex64), kernels=k,
                        sv1=sv[1].astype(np.float32), sv50=sv[50].astype(np.float32),
                        relchange=np.array(rel))
    print(out, os.path.getsize(out))


if __name__ == "__main__":
    main(sys.argv[1])
