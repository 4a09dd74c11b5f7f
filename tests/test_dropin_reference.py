"""The reference's own behavioural suite on the B200 path (SURVEY.md 8(b),
8(f) row 3).

dropin/Makefile builds the reference library from its unmodified sources
(read in place from /root/reference/proj in the build container) with the
entry points the drop-in replaces made weak -- shlr_pi_reconstruct,
shlr_param_reconstruct_slice (solvers.cpp), recon_param_dataset
(parammap.cpp), ssos (io.cpp), rlne / mssim (metrics.cpp) -- and supplies
them from dropin/shlr_dropin.cpp over the C-ABI (libshlr_b200.so).  Linked
into the reference's own unit tests, acceptance suite and CLI, unmodified.
The prebuilt binaries travel to the GPU box (dropin/_build/)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "dropin", "_build")
CLI = os.path.join(BUILD, "shlr_cli")
CLI_TESTS = os.path.join(BUILD, "cli_tests.sh")  # staged from proj/tests by dropin/Makefile

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="dropin/_build not built (make -C dropin)")


def run(args, cwd, **kw):
    return subprocess.run(args, cwd=cwd, capture_output=True, text=True, timeout=kw.pop("timeout", 600), **kw)


def test_cli_host_subcommands_and_parser(tmp_path):
    """The reference CLI (tools/shlr_cli.cpp) built on the CLI11 subset: the
    host-only subcommands run, parse errors keep CLI11's exit codes."""
    r = run([CLI, "phantom", "--kind", "pi", "--rows", "32", "--cols", "32", "--coils", "2", "--seed", "5",
             "--out", "ph"], tmp_path)
    assert r.returncode == 0, r.stderr
    r = run([CLI, "mask", "--type", "gauss", "--n", "32", "--rate", "0.5", "--acs", "8", "--seed", "3",
             "--out", "mask.cplx"], tmp_path)
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "ph_kspace.cplx").stat().st_size > 0 and (tmp_path / "mask.cplx").exists()
    assert run([CLI, "recon-pi", "--bogus", "1"], tmp_path).returncode == 109      # ExtrasError
    assert run([CLI], tmp_path).returncode == 106                                   # RequiredError
    assert run([CLI, "mask", "--n", "x"], tmp_path).returncode == 104               # ConversionError


def test_cli_reconstruction_has_no_cpu_fallback(tmp_path):
    """recon-pi goes through the drop-in: without a device it fails loudly
    (it never falls back to the reference's CPU solver it replaced)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    run([CLI, "phantom", "--kind", "pi", "--rows", "16", "--cols", "16", "--coils", "2", "--out", "ph"], tmp_path)
    run([CLI, "mask", "--type", "gauss", "--n", "16", "--rate", "0.5", "--acs", "4", "--out", "m.cplx"], tmp_path)
    r = run([CLI, "recon-pi", "--input", "ph_kspace.cplx", "--mask", "m.cplx", "--method", "shlr", "--max-outer", "1",
             "--out", "r"],
            tmp_path)
    assert r.returncode == 1 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_reference_unit_suite_on_b200(tmp_path):
    """All of the reference's unit tests (proj/tests/test_*.cpp), including
    test_solvers.cpp:184-302 (full sampling, determinism + log format,
    variant nesting bitwise, stopping rules) and test_parammap.cpp /
    test_metrics.cpp, with the solvers, the dataset driver and the metrics on
    the device."""
    r = run([os.path.join(BUILD, "unit_tests")], tmp_path, timeout=1200)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_reference_acceptance_suite_on_b200(tmp_path):
    """proj/tests/acceptance.cpp on the B200 path (criteria 5, 6, 7, 10, 11
    exercise the solvers: convergence, variants, stopping, determinism)."""
    r = run([os.path.join(BUILD, "acceptance")], tmp_path, timeout=1800)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_reference_cli_suite_on_b200(tmp_path):
    """proj/tests/cli_tests.sh (artifact plumbing, exit codes, manifest rerun
    bitwise, paired-run equivalence, bench shape) against the GPU-backed CLI."""
    r = run(["bash", CLI_TESTS, CLI], tmp_path, timeout=1200)
    print(r.stdout[-2000:])
    assert r.returncode == 0 and "all CLI checks passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
