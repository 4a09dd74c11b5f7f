"""Pack the reference's own BASELINE config-4 slice solves into tests/golden/c4_ref50.npz.

Config 4 (BASELINE.json configs[3], bench.make_param_inputs): 256 FE x 256 PE x
12 echoes x 4 coils T2 phantom, per-echo R=6 masks, K=13 (pencil 244), vc,
lambda2 = 2, 50 outer iterations.  The FE slices of recon_param_dataset are
independent ADMM problems (parammap.cpp:37-51), so the reference is run on
eight of them at full slice size (the centre, the edges and between) with
shlr_param_reconstruct_slice (solvers.cpp:193-298) through oracle/_ref/ref_driver:

    python tests/golden/make_c4_golden.py inputs DIR   # DIR/s128.cplx, DIR/s16.cplx, DIR/m.cplx
    for s in 128 16 0 64 100 160 200 255; do oracle/_ref/ref_driver param y=DIR/s$s.cplx mask=DIR/m.cplx \\
        out=DIR/r$s vc=1 pencil=244 max_outer=50 tol=1e-300; done
    python tests/golden/make_c4_golden.py pack DIR

The slice inputs are the FE-iFFT (hybrid) planes of the dataset, computed by the
oracle's centred FFT (pinned to the reference's fft.cpp).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2107_11650_b200 import cplx_io as io  # noqa: E402

SLICES = (128, 16, 0, 64, 100, 160, 200, 255)


def main(cmd: str, d: str) -> None:
    if cmd == "inputs":
        import bench
        import shlr_oracle as O
        os.makedirs(d, exist_ok=True)
        ds, mask, _, _ = bench.make_param_inputs()
        hybrid = O.fft_along_axis(ds.data, 0, True)
        for s in SLICES:
            io.write_cplx(hybrid[s], os.path.join(d, f"s{s}.cplx"))
        io.write_mask(mask.bits, os.path.join(d, "m.cplx"))
        return
    out = {"slices": np.array(SLICES)}
    for s in SLICES:
        out[f"x{s}"] = io.read_cplx(os.path.join(d, f"r{s}.x.cplx")).astype(np.complex64)
        out[f"log{s}"] = np.array(open(os.path.join(d, f"r{s}.log")).read().splitlines())
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c4_ref50.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
