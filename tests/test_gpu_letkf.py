"""GPU LETKF arm (csrc/letkf_kernels.cu) against the reference's own
letkf_analyze (proj/src/letkf.cpp compiled unmodified into
oracle/_ref/libturbda_ref_cycle.so over the Eigen subset in
oracle/ref_shadow/Eigen/Dense - Eigen itself is absent here), the numpy
restatement (oracle/letkf_oracle.py, which also covers the arctan extension
and explicit locations the reference's API does not take) and the
properties of the reference's own proj/tests/test_letkf.cpp.  fp64
agreement to rounding (1e-9)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import letkf_oracle as L

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.fixture(scope="module")
def capi():
    from paper_2407_12168_b200 import capi as c
    if c.device_count() < 1:
        pytest.skip("no CUDA device")
    return c


def ens(m, d, seed, mean=0.0, sd=1.0):
    return mean + sd * np.random.default_rng(seed).standard_normal((m, d))


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("n,m,stride,arctan,cutoff,alpha", [
    (8, 6, 0, False, 2000.0, 0.3),
    (16, 20, 3, False, 2000.0, 0.3),
    (16, 7, 0, True, 3000.0, 0.0),
    (32, 33, 4, False, 2000.0, 0.5),
    (64, 20, 4, False, 2000.0, 0.3),
    (16, 128, 2, False, 2500.0, 0.3),   # V in global scratch
])
def test_letkf_vs_restatement(capi, n, m, stride, arctan, cutoff, alpha):
    d = 2 * n * n
    x = ens(m, d, 100 + n + m)
    idx = None if stride == 0 else np.arange(0, d, stride, dtype=np.int64)
    nobs = d if idx is None else idx.size
    g = np.random.default_rng(7)
    y = 0.3 + g.standard_normal(nobs)
    r = 0.5 + g.random(nobs)
    got = capi.letkf_analyze(x, y, r, idx, nx=n, ny=n, cutoff_km=cutoff, rtps_alpha=alpha,
                             arctan=arctan)
    want = L.letkf_analyze(x, y, r, idx, n, n, cutoff_km=cutoff, rtps_alpha=alpha, arctan=arctan)
    assert rel_err(got, want) < TOL


@pytest.mark.parametrize("n,m,stride,cutoff,alpha", [
    (8, 6, 0, 2000.0, 0.3),
    (16, 20, 3, 2000.0, 0.3),
    (32, 33, 4, 2000.0, 0.5),
    (64, 20, 4, 2000.0, 0.3),
    (16, 128, 2, 2500.0, 0.3),
    (256, 64, 4, 2000.0, 0.3),          # BASELINE config 2's grid and ensemble
])
def test_letkf_vs_reference(capi, n, m, stride, cutoff, alpha):
    """The reference's letkf.cpp itself (proj/src/letkf.cpp:57-207)."""
    from conftest import ROOT
    from oracle.oracle import RefCycleOracle
    path = ROOT / "oracle" / "_ref" / "libturbda_ref_cycle.so"
    if not path.exists():
        pytest.skip("oracle/_ref/libturbda_ref_cycle.so not built")
    d = 2 * n * n
    x = ens(m, d, 100 + n + m)
    idx = None if stride == 0 else np.arange(0, d, stride, dtype=np.int64)
    nobs = d if idx is None else idx.size
    g = np.random.default_rng(7)
    y = 0.3 + g.standard_normal(nobs)
    r = 0.5 + g.random(nobs)
    got = capi.letkf_analyze(x, y, r, idx, nx=n, ny=n, cutoff_km=cutoff, rtps_alpha=alpha)
    want = RefCycleOracle(path).letkf_analyze(x, y, r, idx, n, n, cutoff_km=cutoff,
                                              rtps_alpha=alpha)
    assert rel_err(got, want) < TOL


def test_letkf_explicit_locations_and_sparse_obs(capi):
    """Arbitrary observation locations (cells with several observations,
    points with none inside the stencil keep the background)."""
    n, m = 16, 10
    d = 2 * n * n
    x = ens(m, d, 5)
    g = np.random.default_rng(3)
    idx = np.sort(g.choice(d, 40, replace=False)).astype(np.int64)
    locs = np.stack([g.uniform(0, 4, 40), g.uniform(0, 4, 40)], axis=1)  # one corner only
    y = g.standard_normal(40)
    got = capi.letkf_analyze(x, y, 0.7, idx, nx=n, ny=n, cutoff_km=1500.0, locations=locs)
    want = L.letkf_analyze(x, y, 0.7, idx, n, n, cutoff_km=1500.0, locations=locs)
    assert rel_err(got, want) < TOL
    # far from the observed corner the analysis is the (RTPS-inflated) background
    far = L.letkf_analyze(x, y, 0.7, idx, n, n, cutoff_km=1500.0, locations=locs, rtps_alpha=0.0)
    untouched = np.all(far == x, axis=0)
    assert untouched.sum() > 100
    got0 = capi.letkf_analyze(x, y, 0.7, idx, nx=n, ny=n, cutoff_km=1500.0, locations=locs,
                              rtps_alpha=0.0)
    assert np.array_equal(got0[:, untouched], x[:, untouched])


def test_letkf_reference_properties(capi):
    """proj/tests/test_letkf.cpp:121-237 on the GPU path."""
    n, d = 8, 128
    # zero innovation keeps the mean, members still move (:121-137)
    e = ens(6, d, 55, 0.2, 1.0)
    an = capi.letkf_analyze(e, e.mean(axis=0), 0.5, nx=n, ny=n)
    assert np.abs(an.mean(axis=0) - e.mean(axis=0)).max() < 1e-10
    assert np.abs(an - e).max() > 1e-6
    # near-perfect collocated obs pull the mean onto them (:139-151)
    e = ens(8, d, 66)
    y = 0.5 + np.random.default_rng(9).standard_normal(d)
    an = capi.letkf_analyze(e, y, 1e-8, nx=n, ny=n, cutoff_km=1000.0, rtps_alpha=0.0)
    assert np.abs(an.mean(axis=0) - y).max() < 1e-4
    # huge cutoff == global ETKF (:153-201)
    m = 6
    e = ens(m, d, 77, 0.5, 1.0)
    y = 0.4 + 1.2 * np.random.default_rng(31).standard_normal(d)
    local = capi.letkf_analyze(e, y, 0.8, nx=n, ny=n, cutoff_km=1e12, rtps_alpha=0.0)
    yb = e.T - e.mean(axis=0)[:, None]
    wbar, w = L.etkf_local_analysis(yb, y, e.mean(axis=0), np.full(d, 1 / 0.8), m)
    pert = e - e.mean(axis=0)
    want = e.mean(axis=0) + (pert.T @ wbar)[None, :] + w.T @ pert
    assert np.abs(local - want).max() < 1e-8
    tight = capi.letkf_analyze(e, y, 0.8, nx=n, ny=n, cutoff_km=2000.0, rtps_alpha=0.0)
    assert np.abs(tight - local).max() > 1e-6
    # member permutation equivariance (:203-223)
    e = ens(5, d, 88)
    y = np.random.default_rng(12).standard_normal(d)
    a = capi.letkf_analyze(e, y, 1.0, nx=n, ny=n)
    b = capi.letkf_analyze(e[::-1].copy(), y, 1.0, nx=n, ny=n)
    assert np.abs(a - b[::-1]).max() < 1e-9
    # bitwise reproducible (:225-237: identical at any worker count)
    assert np.array_equal(a, capi.letkf_analyze(e, y, 1.0, nx=n, ny=n))


def test_rtps_kernel(capi):
    """proj/tests/test_letkf.cpp:268-308."""
    bg = ens(20, 4, 50, 0.0, 2.0)
    an = ens(20, 4, 51, 0.1, 0.5)
    assert np.array_equal(capi.rtps_inflate(an, bg, 0.0), an)
    got = capi.rtps_inflate(an, bg, 0.3)
    assert rel_err(got, L.rtps_inflate(an, bg, 0.3)) < 1e-13
    sa, sb, si = (v.std(axis=0, ddof=1) for v in (an, bg, got))
    assert np.allclose(si, sa + 0.3 * (sb - sa), rtol=1e-10)
    out = capi.rtps_inflate(np.array([[0.5], [0.0]]), np.array([[1.0], [-1.0]]), 1.0)
    assert out[0, 0] == pytest.approx(1.25, rel=1e-13) and out[1, 0] == pytest.approx(-0.75, rel=1e-13)


def test_letkf_single_member_is_singular(capi):
    """M = 1: A = 0 -> SingularAnalysisError at the first observed point."""
    with pytest.raises(capi.TurbdaError) as ei:
        capi.letkf_analyze(ens(1, 128, 1), np.zeros(128), 1.0, nx=8, ny=8)
    assert ei.value.code == capi.SINGULAR and b"singular local analysis" in \
        str(ei.value).encode()


def test_letkf_device_pointers_and_uniform_r(capi):
    torch = pytest.importorskip("torch")
    n, m = 16, 12
    d = 2 * n * n
    x = ens(m, d, 9)
    idx = np.arange(0, d, 2, dtype=np.int64)
    y = np.random.default_rng(2).standard_normal(idx.size)
    host = capi.letkf_analyze(x, y, 0.9, idx, nx=n, ny=n)
    assert np.array_equal(capi.letkf_analyze(x, y, 0.9, idx, nx=n, ny=n, r_uniform=True), host)
    dev = torch.device("cuda:0")
    tx = torch.from_numpy(x).to(dev)
    out = torch.empty_like(tx)
    p = capi.letkf_params(nx=n, ny=n, n_members=m, obs_kind=1, obs_dim=idx.size, device=0,
                          flags=capi.INPUTS_ON_DEVICE | capi.R_UNIFORM)
    capi.letkf_raw(p, tx, torch.from_numpy(y).to(dev),
                   torch.tensor([0.9], dtype=torch.float64, device=dev),
                   torch.from_numpy(idx).to(dev), None, out,
                   stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), host)


@pytest.mark.parametrize("r,tol", [(1e-2, 1e-10), (1e-4, 1e-9), (1e-6, 1e-7)])
def test_letkf_ill_conditioned_local_problems(capi, r, tol):
    """Accurate observations make A = (M-1) I + Yb^T R^-1 Yb ill-conditioned
    (condition ~ 1/r): the tensor-core Newton-Schulz transform must still
    converge and agree with the eigendecomposition of the restatement (the
    tolerance follows the conditioning of W = sqrt(M-1) A^-1/2)."""
    n, m = 16, 20
    d = 2 * n * n
    x = ens(m, d, 31)
    y = np.random.default_rng(4).standard_normal(d)
    got = capi.letkf_analyze(x, y, r, nx=n, ny=n, cutoff_km=1500.0)
    want = L.letkf_analyze(x, y, r, None, n, n, cutoff_km=1500.0)
    assert rel_err(got, want) < tol


def test_unconverged_newton_schulz_points_redone_by_jacobi(tmp_path):
    """With the Newton-Schulz iteration capped at 3 (TURBDA_LETKF_NS_ITERS, a
    fresh process) no point converges: every one is listed and redone by the
    Jacobi eigensolver, and the analysis still matches the restatement."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    n, m = 16, 20
    d = 2 * n * n
    x = ens(m, d, 44)
    y = np.random.default_rng(9).standard_normal(d)
    np.save(tmp_path / "x.npy", x)
    np.save(tmp_path / "y.npy", y)
    code = ("import numpy as np, sys; from paper_2407_12168_b200 import capi; d = sys.argv[1]; "
            "x = np.load(d + '/x.npy'); y = np.load(d + '/y.npy'); "
            f"np.save(d + '/out.npy', capi.letkf_analyze(x, y, 0.5, None, nx={n}, ny={n}))")
    env = dict(os.environ, TURBDA_LETKF_NS_ITERS="3")
    subprocess.run([sys.executable, "-c", code, str(tmp_path)], check=True, env=env, cwd=str(ROOT))
    got = np.load(tmp_path / "out.npy")
    want = L.letkf_analyze(x, y, 0.5, None, n, n)
    assert rel_err(got, want) < TOL
