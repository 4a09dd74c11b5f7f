"""Golden vectors for the metrics row from the reference
itself: oracle/_ref/ref_driver metrics (proj/src/io.cpp:105-117 ssos,
proj/src/metrics.cpp:9-75 rlne / mssim, unmodified) on seeded inputs.

    python tests/golden/make_metrics_golden.py      # -> tests/golden/metrics_ref.npz
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_11650_b200 import cplx_io as io  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def main():
    rng = np.random.default_rng(7)
    cases = {}
    x = rng.standard_normal((40, 36, 3)) + 1j * rng.standard_normal((40, 36, 3))
    pairs = []
    for rows, cols in [(64, 48), (11, 11), (23, 37)]:
        ref = np.abs(rng.standard_normal((rows, cols))) + 0.5
        rec = ref + 0.05 * rng.standard_normal((rows, cols))
        pairs.append((ref, rec))
    with tempfile.TemporaryDirectory() as d:
        io.write_cplx(x, os.path.join(d, "x.cplx"))
        subprocess.run([REF, "metrics", "x=x.cplx", "out=m"], cwd=d, check=True)
        cases["x"] = x
        cases["ssos"] = io.read_cplx(os.path.join(d, "m.ssos.cplx")).real
        for i, (ref, rec) in enumerate(pairs):
            io.write_cplx(ref.astype(np.complex128), os.path.join(d, "a.cplx"))
            io.write_cplx(rec.astype(np.complex128), os.path.join(d, "b.cplx"))
            out = subprocess.run([REF, "metrics", "ref=a.cplx", "rec=b.cplx"], cwd=d, check=True,
                                 capture_output=True, text=True).stdout
            kv = dict(line.split("=") for line in out.split())
            cases[f"ref{i}"], cases[f"rec{i}"] = ref, rec
            cases[f"rlne{i}"], cases[f"mssim{i}"] = float(kv["rlne"]), float(kv["mssim"])
    path = os.path.join(ROOT, "tests", "golden", "metrics_ref.npz")
    np.savez_compressed(path, npairs=len(pairs), **cases)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
