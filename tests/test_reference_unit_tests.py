"""The reference's own unit tests for the path and the widened rows
(proj/tests/test_{ensf,rng,ensemble,parallel,snapshot,forecast,osse,budget}.cpp,
72 cases), compiled unmodified against
include/turbda/*.hpp and linked to libturbda_b200.so (oracle/reftests) -
the drop-in check for the C++ API.

Against its own implementation the reference passes 35 of the 38 hot-path
cases (the 4 snapshot cases pass everywhere); the 3
failures are defects of the tests: a Philox KAT typo
(test_rng.cpp:23), a sign error in the shrinkage test (test_ensf.cpp:189-199)
and the bimodal crossing test, which the reference's Euler-Maruyama misses at
the default 100 steps (test_ensf.cpp:312-329).  The B200 build must fail
exactly those three."""
import re
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "oracle" / "_ref" / "reftests_b200"
REF_BIN = ROOT / "oracle" / "_ref" / "reftests_ref"  # the same files against the reference
EXPECTED_FAILURES = {
    "philox4x32 known-answer vectors",
    "reverse SDE step: zero scores and zero noise shrink toward origin",
    "analyze pulls a collapsed prior toward a bimodal-side observation",
    # the reference throws DimensionError where its test expects ConfigError
    "climatological amplitude is the RMS over the trajectory",
    # the reference's own EnSF misses this property on the tiny test config
    # (measured: reftests_ref fails it at the same checks)
    "assimilation beats the free run on its own forecasts",
}


def _run(filt=None, binary=BIN):
    if not binary.exists():
        pytest.skip(f"{binary} not built (needs /root/reference at build time)")
    cmd = [str(binary)] + ([filt] if filt else [])
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600).stdout
    failed = set(re.findall(r"^\[FAIL\] (.*) \(", out, re.M))
    passed = set(re.findall(r"^\[PASS\] (.*) \(", out, re.M))
    return passed, failed, out


def test_host_only_reference_cases():
    """RNG, parallel_for and the operator/ensemble cases need no GPU."""
    for filt in ("philox", "splitmix", "stream", "uniform", "normal moments", "distinct entities",
                 "parallel_for", "TURBDA_WORKERS", "grid operators", "adjoint",
                 "operator locations", "observation validation", "ensemble validation",
                 "snapshot round", "snapshot header", "corrupt", "snapshot file", "config json",
                 "partial configs", "config hash", "experiment config", "model error config",
                 "parameter count", "published", "tokens per image", "training", "budget",
                 "significant",
                 "metrics serialization"):
        passed, failed, out = _run(filt)
        assert passed | failed, filt
        assert failed <= EXPECTED_FAILURES, out


@pytest.mark.gpu
def test_reference_suite_on_b200():
    passed, failed, out = _run()
    print(out[-3000:])
    assert len(passed) + len(failed) == 72
    assert failed == EXPECTED_FAILURES, out


@pytest.mark.gpu
def test_reference_suite_same_verdicts_as_reference():
    """The same 72 cases linked against the reference implementation (the
    cycle oracle, cuFFTW build) fail exactly where the B200 build fails."""
    passed_r, failed_r, out_r = _run(binary=REF_BIN)
    passed, failed, _ = _run()
    assert failed_r == failed, out_r
    assert passed_r == passed


CPP_LETKF = ROOT / "tests" / "cpp" / "_build" / "test_cpp_letkf"


def _run_cpp_letkf(filt=None):
    if not CPP_LETKF.exists():
        pytest.skip("tests/cpp/_build/test_cpp_letkf not built (make -C tests/cpp)")
    cmd = [str(CPP_LETKF)] + ([filt] if filt else [])
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600)


def test_cpp_letkf_api_host_cases():
    """gaspari_cohn and the argument checks of the C++ LETKF API need no GPU."""
    for filt in ("gaspari_cohn", "input validation"):
        r = _run_cpp_letkf(filt)
        assert r.returncode == 0, r.stdout


@pytest.mark.gpu
def test_cpp_letkf_api_on_b200():
    """The Eigen-free cases of proj/tests/test_letkf.cpp against the C++ API
    (include/turbda/letkf.hpp) on the GPU."""
    r = _run_cpp_letkf()
    print(r.stdout[-3000:])
    assert r.returncode == 0 and "failed=0" in r.stdout, r.stdout


REF_LETKF_BIN = ROOT / "oracle" / "_ref" / "reftests_ref_letkf"


def test_reference_letkf_tests_pin_the_eigen_subset():
    """proj/tests/test_letkf.cpp against the reference's own letkf.cpp, both
    compiled over oracle/ref_shadow/Eigen/Dense (Eigen is absent here): every
    host-only case passes, which pins the Eigen subset - and with it the LETKF
    oracle the GPU arm is compared with - on the reference's closed forms
    (scalar Kalman update, ETKF identities, global-ETKF limit, RTPS)."""
    passed, failed, out = _run(binary=REF_LETKF_BIN)
    host_only = failed - {"letkf pulls a climatological ensemble toward the truth"}
    assert len(passed) >= 13 and not host_only, out


@pytest.mark.gpu
def test_reference_letkf_tests_all_pass_on_gpu_box():
    """The one case that needs the SQG nature run (cuFFTW) passes too."""
    passed, failed, out = _run(binary=REF_LETKF_BIN)
    assert len(passed) == 14 and not failed, out
