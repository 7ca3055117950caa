"""CPU: the drop-in boundary loads, exports what include/turbda_b200.h
declares, and validates arguments before touching a device (no compute
calls here)."""
import ctypes as C
import re

import numpy as np
import pytest

from conftest import ROOT


def test_library_exports_every_declared_symbol():
    from paper_2407_12168_b200 import capi
    lib = capi.lib()
    declared = capi.exported_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name


def test_header_symbols_match_nm():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2407_12168_b200" / "lib" /
                          "libturbda_b200.so")], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (turbda_[a-z0-9_]+)", out))
    hdr = set(re.findall(r"\b(turbda_[a-z0-9_]+)\s*\(", (ROOT / "include" / "turbda_b200.h").read_text()))
    assert hdr <= exported
    # nothing but the C-ABI and the turbda:: C++ API leaks out of the library
    assert all(s.startswith("turbda_") for s in exported)


def test_cpp_api_symbols_exported():
    import subprocess
    out = subprocess.run(["nm", "-DC", "--defined-only", str(ROOT / "paper_2407_12168_b200" / "lib" /
                          "libturbda_b200.so")], capture_output=True, text=True, check=True).stdout
    for sym in ("turbda::analyze(", "turbda::relax_spread(", "turbda::prior_score(",
                "turbda::posterior_score(", "turbda::likelihood_score(", "turbda::reverse_sde_step(",
                "turbda::RngStream::normal()", "turbda::philox4x32(", "turbda::make_grid_operator(",
                "turbda::synthesize_observations(", "turbda::ensemble_mean(", "turbda::spread("):
        assert sym in out, sym


def test_params_init_defaults():
    from paper_2407_12168_b200 import capi
    p = capi.params()
    # reference defaults, proj/include/turbda/ensf.hpp:22-27
    assert (p.n_steps, p.eps, p.minibatch_j, p.damping_t, p.relax_factor) == (100, 0.01, 0, 1.0, 1.0)
    assert p.precision == capi.FP32 and p.device == -1 and p.device_count == 1


@pytest.mark.parametrize("field,value,code", [
    ("eps", 0.0, 1), ("eps", 1.0, 1), ("n_steps", 9, 1), ("minibatch_j", -1, 1),
    ("relax_factor", 1.5, 1), ("n_members", 0, 2), ("obs_dim", 7, 2), ("precision", 3, 1),
])
def test_validation_before_device(field, value, code):
    """Config/dimension errors are reported without a GPU (validation runs first)."""
    from paper_2407_12168_b200 import capi
    x = np.zeros((4, 8))
    y = np.zeros(8)
    r = np.ones(8)
    p = capi.params(d_total=8, d_local=8, obs_dim=8, n_members=4)
    setattr(p, field, value)
    with pytest.raises(capi.TurbdaError) as ei:
        capi.analyze(p, x, y, r, None, np.zeros_like(x))
    assert ei.value.code == code


def test_r_must_be_positive_host_mode():
    from paper_2407_12168_b200 import capi
    x = np.zeros((4, 8))
    r = np.ones(8)
    r[3] = 0.0
    p = capi.params(d_total=8, d_local=8, obs_dim=8, n_members=4)
    with pytest.raises(capi.TurbdaError) as ei:
        capi.analyze(p, x, np.zeros(8), r, None, np.zeros_like(x))
    assert ei.value.code == capi.CONFIG and b"r_diag" in bytes(ei.value.args[0], "utf8")


def test_uniform_r_validated_before_device():
    """TURBDA_R_UNIFORM: the one r value is checked (r > 0) before any device
    work; the other obs_dim - 1 entries are never read."""
    from paper_2407_12168_b200 import capi
    x = np.zeros((4, 8))
    p = capi.params(d_total=8, d_local=8, obs_dim=8, n_members=4, flags=capi.R_UNIFORM)
    with pytest.raises(capi.TurbdaError) as ei:
        capi.analyze(p, x, np.zeros(8), np.array([-1.0]), None, np.zeros_like(x))
    assert ei.value.code == capi.CONFIG


def test_python_module_mirrors_reference_binding():
    import paper_2407_12168_b200 as tb
    assert issubclass(tb.ConfigError, ValueError) and issubclass(tb.DimensionError, ValueError)
    g = tb.GridSpec()
    assert (g.nx, g.ny, g.nz) == (64, 64, 2) and g.grid_size() == 8192
    g.nx = g.ny = 8
    with pytest.raises(tb.DimensionError):  # d != grid size, proj/src/ensf.cpp:142-143
        tb.ensf_analyze(np.zeros((4, 100)), g, np.zeros(128))
    with pytest.raises(tb.DimensionError):  # members must be (M, d)
        tb.ensf_analyze(np.zeros(128), g, np.zeros(128))
    with pytest.raises(tb.ConfigError):
        tb.ensf_analyze(np.zeros((4, 128)), g, np.zeros(128), n_steps=5)
    with pytest.raises(tb.ConfigError):
        tb.ensf_analyze(np.zeros((4, 128)), g, np.zeros(128), r=0.0)


def test_no_cpu_fallback_without_device():
    """Without a GPU the compute path fails loudly instead of computing on the host."""
    from paper_2407_12168_b200 import capi
    if capi.device_count() > 0:
        pytest.skip("a GPU is visible")
    x = np.zeros((4, 8))
    p = capi.params(d_total=8, d_local=8, obs_dim=8, n_members=4)
    with pytest.raises(capi.TurbdaError) as ei:
        capi.analyze(p, x, np.zeros(8), np.ones(8), None, np.zeros_like(x))
    assert ei.value.code == capi.CUDA


@pytest.mark.parametrize("kw,code", [
    (dict(nx=8, ny=16), "CONFIG"),            # isotropic metric, proj/src/letkf.cpp:62-63
    (dict(rtps_alpha=1.5), "CONFIG"),         # LetkfConfig::validate
    (dict(cutoff_km=0.0), "CONFIG"),
    (dict(nx=6, ny=6), "CONFIG"),             # GridSpec::validate
    (dict(obs_dim=100), "DIMENSION"),         # identity operator of the wrong size
])
def test_letkf_validation_before_device(kw, code):
    """LETKF arm: argument checks precede any device work,
    as the reference's letkf input-validation test expects
    (proj/tests/test_letkf.cpp:310-337)."""
    from paper_2407_12168_b200 import capi
    base = dict(nx=8, ny=8, n_members=4, obs_kind=0, obs_dim=128)
    base.update(kw)
    p = capi.letkf_params(**base)
    x = np.zeros((4, 2 * p.nx * p.ny))
    with pytest.raises(capi.TurbdaError) as ei:
        capi.letkf_raw(p, x, np.zeros(p.obs_dim), np.ones(p.obs_dim), None, None,
                       np.zeros_like(x))
    assert ei.value.code == getattr(capi, code)


def test_gaspari_cohn_host_entry():
    from paper_2407_12168_b200 import capi
    assert capi.gaspari_cohn(0.0) == 1.0
    assert capi.gaspari_cohn(1.0) == pytest.approx(5.0 / 24.0, rel=1e-14)
    assert capi.gaspari_cohn(1.5) == pytest.approx(19.0 / 1152.0, rel=1e-13)
    assert capi.gaspari_cohn(2.0) == 0.0
    with pytest.raises(capi.TurbdaError):
        capi.gaspari_cohn(-0.1)
