"""CPU: the numpy LETKF restatement (oracle/letkf_oracle.py) against the
closed forms and properties of the reference's own proj/tests/test_letkf.cpp
and against the reference's letkf.cpp itself (compiled unmodified over the
Eigen subset in oracle/ref_shadow/Eigen/Dense - Eigen is absent here).
Small grids: the restatement loops over grid points."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import letkf_oracle as L


def gaussian_ensemble(m, d, seed, mean=0.0, sd=1.0):
    return mean + sd * np.random.default_rng(seed).standard_normal((m, d))


def test_gaspari_cohn_closed_forms():
    # proj/tests/test_letkf.cpp:30-38
    assert L.gaspari_cohn(0.0) == 1.0
    assert L.gaspari_cohn(0.5) == pytest.approx(263.0 / 384.0, rel=1e-14)
    assert L.gaspari_cohn(1.0) == pytest.approx(5.0 / 24.0, rel=1e-14)
    assert L.gaspari_cohn(1.5) == pytest.approx(19.0 / 1152.0, rel=1e-13)
    assert L.gaspari_cohn(2.0) == 0.0 and L.gaspari_cohn(7.3) == 0.0
    with pytest.raises(ValueError):
        L.gaspari_cohn(-0.1)
    # :40-51 continuous and decreasing
    assert abs(L.gaspari_cohn(1 - 1e-9) - L.gaspari_cohn(1 + 1e-9)) < 1e-8
    prev = 1.0
    for i in range(201):
        v = L.gaspari_cohn(i * 0.01)
        assert v <= prev + 1e-15 and v >= 0.0
        prev = v


def test_etkf_no_obs_identity_and_scalar_kalman():
    wbar, w = L.etkf_local_analysis(np.zeros((0, 6)), np.zeros(0), np.zeros(0), np.zeros(0), 6)
    assert not wbar.any() and np.array_equal(w, np.eye(6))
    # :62-85 one scalar observation
    m = 7
    yb = np.array([[0.3, -0.5, 0.9, -0.1, 0.4, -0.7, -0.3]])
    yb -= yb.mean()
    bbar, y, r = 1.7, 2.9, 0.6
    s2 = (yb ** 2).sum() / (m - 1)
    wbar, w = L.etkf_local_analysis(yb, np.array([y]), np.array([bbar]), np.array([1 / r]), m)
    assert bbar + (yb @ wbar)[0] == pytest.approx(bbar + s2 / (s2 + r) * (y - bbar), rel=1e-12)
    pa = yb @ w
    assert (pa ** 2).sum() / (m - 1) == pytest.approx(r * s2 / (r + s2), rel=1e-12)


def test_etkf_defining_identities():
    # :87-119
    m, p = 8, 5
    g = np.random.default_rng(21)
    y, ybm = g.standard_normal(p), 0.3 * g.standard_normal(p)
    rinv = 0.5 + g.random(p)
    yb = g.standard_normal((p, m))
    yb -= yb.mean(axis=1, keepdims=True)
    wbar, w = L.etkf_local_analysis(yb, y, ybm, rinv, m)
    a = yb.T @ (rinv[:, None] * yb) + (m - 1) * np.eye(m)
    assert np.abs(a @ wbar - yb.T @ (rinv * (y - ybm))).max() < 1e-10
    assert np.abs(w - w.T).max() < 1e-12
    assert np.abs(a @ w @ w.T / (m - 1) - np.eye(m)).max() < 1e-10
    assert np.linalg.eigvalsh(w).min() > 0.0


def test_zero_innovation_keeps_mean():
    # :121-137
    ens = gaussian_ensemble(6, 128, 55, 0.2, 1.0)
    an = L.letkf_analyze(ens, ens.mean(axis=0), 0.5, None, 8, 8)
    assert np.abs(an.mean(axis=0) - ens.mean(axis=0)).max() < 1e-10
    assert np.abs(an - ens).max() > 1e-6


def test_near_perfect_obs_and_huge_cutoff_is_global_etkf():
    # :139-151
    ens = gaussian_ensemble(8, 128, 66)
    y = 0.5 + np.random.default_rng(9).standard_normal(128)
    an = L.letkf_analyze(ens, y, 1e-8, None, 8, 8, cutoff_km=1000.0, rtps_alpha=0.0)
    assert np.abs(an.mean(axis=0) - y).max() < 1e-4
    # :153-201
    m = 6
    ens = gaussian_ensemble(m, 128, 77, 0.5, 1.0)
    y = 0.4 + 1.2 * np.random.default_rng(31).standard_normal(128)
    local = L.letkf_analyze(ens, y, 0.8, None, 8, 8, cutoff_km=1e12, rtps_alpha=0.0)
    yb = ens.T.copy()
    ybm = yb.mean(axis=1)
    yb -= ybm[:, None]
    wbar, w = L.etkf_local_analysis(yb, y, ybm, np.full(128, 1 / 0.8), m)
    mean = ens.mean(axis=0)
    pert = ens - mean
    want = mean + (pert.T @ wbar)[None, :] + (w.T @ pert)
    assert np.abs(local - want).max() < 1e-8
    tight = L.letkf_analyze(ens, y, 0.8, None, 8, 8, cutoff_km=2000.0, rtps_alpha=0.0)
    assert np.abs(tight - local).max() > 1e-6


def test_member_permutation_equivariance():
    # :203-223
    ens = gaussian_ensemble(5, 128, 88)
    y = np.random.default_rng(12).standard_normal(128)
    a = L.letkf_analyze(ens, y, 1.0, None, 8, 8)
    b = L.letkf_analyze(ens[::-1].copy(), y, 1.0, None, 8, 8)
    assert np.abs(a - b[::-1]).max() < 1e-9


def test_rtps():
    # :268-295
    bg = gaussian_ensemble(20, 4, 50, 0.0, 2.0)
    an = gaussian_ensemble(20, 4, 51, 0.1, 0.5)
    assert np.array_equal(L.rtps_inflate(an, bg, 0.0), an)
    infl = L.rtps_inflate(an, bg, 0.3)
    assert np.abs(infl.mean(axis=0) - an.mean(axis=0)).max() < 1e-12
    sa, sb, si = (v.std(axis=0, ddof=1) for v in (an, bg, infl))
    assert np.allclose(si, sa + 0.3 * (sb - sa), rtol=1e-10)
    # :297-308 two-member hand case
    out = L.rtps_inflate(np.array([[0.5], [0.0]]), np.array([[1.0], [-1.0]]), 1.0)
    assert out[0, 0] == pytest.approx(0.25 + 4 * 0.25, rel=1e-13)
    assert out[1, 0] == pytest.approx(0.25 - 4 * 0.25, rel=1e-13)


def test_offsets_cover_each_cell_once():
    """The gather stencil is a periodic kernel: every residue at most once,
    weight gc(min-image distance / cutoff) (the GPU path convolves with it)."""
    for n, cutoff in ((8, 0.4), (8, 0.8), (8, 1e11), (16, 1.6), (64, 6.4)):
        offs = L.localization_offsets(n, n, cutoff)
        cells = [((ox % n), (oy % n)) for ox, oy, _ in offs]
        assert len(cells) == len(set(cells))
        for ox, oy, gc in offs:
            ax, ay = min(abs(ox), n - abs(ox)), min(abs(oy), n - abs(oy))
            assert gc == L.gaspari_cohn(math.hypot(ax, ay) / cutoff)


def _refcycle():
    from oracle.oracle import HERE, RefCycleOracle
    path = HERE / "_ref" / "libturbda_ref_cycle.so"
    if not path.exists():
        pytest.skip("oracle/_ref/libturbda_ref_cycle.so not built")
    return RefCycleOracle()


@pytest.mark.parametrize("n,m,stride,cutoff,alpha", [
    (8, 6, 0, 2000.0, 0.3), (16, 20, 3, 2000.0, 0.0), (16, 9, 0, 1e12, 0.5), (32, 12, 4, 3000.0, 0.3),
])
def test_two_restatements_agree(n, m, stride, cutoff, alpha):
    """numpy restatement (per point, reference gather order) vs the
    reference's own letkf_analyze (proj/src/letkf.cpp, unmodified; Eigen's
    SelfAdjointEigenSolver restated as cyclic Jacobi in the shadow header)."""
    rc = _refcycle()
    d = 2 * n * n
    x = gaussian_ensemble(m, d, 3 + n)
    idx = None if stride == 0 else np.arange(0, d, stride, dtype=np.int64)
    g = np.random.default_rng(4)
    nobs = d if idx is None else idx.size
    y = g.standard_normal(nobs)
    r = 0.4 + g.random(nobs)
    a = L.letkf_analyze(x, y, r, idx, n, n, cutoff_km=cutoff, rtps_alpha=alpha)
    b = rc.letkf_analyze(x, y, r, idx, n, n, cutoff_km=cutoff, rtps_alpha=alpha, workers=4)
    assert np.abs(a - b).max() <= 1e-10 * np.abs(a).max()
    # the reference is bitwise independent of the worker count
    assert np.array_equal(b, rc.letkf_analyze(x, y, r, idx, n, n, cutoff_km=cutoff,
                                              rtps_alpha=alpha, workers=1))
