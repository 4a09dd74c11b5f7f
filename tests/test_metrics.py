"""Metrics row: ssos (proj/src/io.cpp:105-117), rlne and
mssim (proj/src/metrics.cpp:9-75) on the device against golden vectors the
reference itself produced (tests/golden/make_metrics_golden.py).  ssos is
bitwise the reference's (same FP64 operation order); rlne and mssim differ
only by the summation order of the final reduction (bar 1e-12 relative)."""
import os

import numpy as np
import pytest

import shlr_oracle as O

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "metrics_ref.npz")


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(G))


def test_oracle_metrics_match_reference(golden):
    assert np.array_equal(O.ssos(golden["x"]), golden["ssos"])
    for i in range(int(golden["npairs"])):
        a, b = golden[f"ref{i}"], golden[f"rec{i}"]
        assert abs(O.rlne(a, b) - golden[f"rlne{i}"]) <= 1e-13 * golden[f"rlne{i}"]
        assert abs(O.mssim(a, b) - golden[f"mssim{i}"]) <= 1e-13


@pytest.mark.gpu
def test_device_metrics_match_reference(gpu, golden):
    A = gpu
    assert np.array_equal(A.ssos(golden["x"]), golden["ssos"])  # bitwise
    for i in range(int(golden["npairs"])):
        a, b = golden[f"ref{i}"], golden[f"rec{i}"]
        assert abs(A.rlne(a, b) - golden[f"rlne{i}"]) <= 1e-12 * golden[f"rlne{i}"]
        assert abs(A.mssim(a, b) - golden[f"mssim{i}"]) <= 1e-12


@pytest.mark.gpu
def test_device_metrics_edge_cases(gpu):
    """The reference's error cases (metrics.cpp:10-11,19-20,24-29): zero
    reference, image smaller than the window; identical images give
    rlne 0 and mssim 1."""
    A = gpu
    a = np.abs(np.random.default_rng(1).standard_normal((16, 16))) + 0.1
    assert A.rlne(a, a) == 0.0
    assert abs(A.mssim(a, a) - 1.0) < 1e-12
    with pytest.raises(ValueError):
        A.rlne(np.zeros((4, 4)), a[:4, :4])
    with pytest.raises(ValueError):
        A.mssim(a[:10, :16], a[:10, :16])
    with pytest.raises(ValueError):
        A.ssos(np.zeros((3, 4)))
