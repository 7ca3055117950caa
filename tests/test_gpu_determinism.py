"""GPU: bitwise determinism of the reductions, the observation prep for any
index order, large Philox counters, long step tables and empty windows.

The reference promises byte-identical metrics across runs and worker counts
(proj/tests/test_osse.cpp:163-179, proj/tests/test_ensf.cpp:337-348): every
reduction here is fixed-order (no floating-point atomics), so repeated runs
must agree bit for bit.
"""
import numpy as np
import pytest

from oracle.oracle import conditioned_inputs, rel_l2

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-10
FP32_TOL = 1e-4


@pytest.fixture(scope="module")
def capi():
    from paper_2407_12168_b200 import capi as c
    if c.device_count() < 1:
        pytest.fail("no CUDA device visible to libturbda_b200.so")
    return c


def test_diag_bitwise_reproducible_at_scale(capi):
    """rmse/spread sums over 64 x 2M values (4096+ CTAs' worth of partials):
    three runs identical to the bit, and equal to numpy's to 1e-12."""
    g = np.random.default_rng(5)
    x = g.standard_normal((64, 1 << 21))
    truth = g.standard_normal(1 << 21)
    runs = [capi.diag(x, truth) for _ in range(3)]
    assert runs[0] == runs[1] == runs[2]
    mean = x.mean(axis=0)
    want = (float(((mean - truth) ** 2).sum()), float(((x - mean) ** 2).sum()))
    for a, b in zip(runs[0], want):
        assert abs(a - b) <= 1e-12 * abs(b)


def test_diag_sharded_flag_needs_a_communicator(capi):
    x = np.ones((4, 64))
    with pytest.raises(capi.TurbdaError) as ei:
        capi.diag(x, None, sharded=True)
    assert ei.value.code == capi.CONFIG


@pytest.mark.parametrize("precision", [0, 1])
def test_duplicate_and_unsorted_selection_deterministic(capi, port, precision):
    """Selection operators with repeated and unsorted indices (adjoint_scatter
    adds duplicates, proj/src/observation.cpp:18-27): the stable-sort prep is
    bitwise reproducible, the device path equals the host path, and both
    match the C restatement."""
    m, d = 20, 4096
    x, _, _, truth = conditioned_inputs(m, d)
    x = x.astype(np.float32).astype(np.float64)
    g = np.random.default_rng(3)
    idx = np.concatenate([g.integers(0, d, 3000), np.repeat(np.arange(100, 110), 7)])
    g.shuffle(idx)
    idx = idx.astype(np.int64)
    y = (truth[idx] + g.standard_normal(idx.size)).astype(np.float32).astype(np.float64)
    r = 0.5 + g.random(idx.size)
    runs = [capi.analyze_host(x, y, r, idx, n_steps=30, precision=precision) for _ in range(3)]
    assert np.array_equal(runs[0], runs[1]) and np.array_equal(runs[0], runs[2])
    want = port.analyze(x, y, r, idx, n_steps=30)
    assert rel_l2(runs[0], want) <= (FP64_TOL if precision else FP32_TOL)

    import torch
    dev = torch.device("cuda", 0)
    tx = torch.from_numpy(x).to(dev)
    ty = torch.from_numpy(y).to(dev)
    tr = torch.from_numpy(r).to(dev)
    ti = torch.from_numpy(idx).to(dev)
    out = torch.empty_like(tx)
    p = capi.params(d_total=d, d_local=d, obs_dim=idx.size, n_members=m, n_steps=30, obs_kind=1,
                    precision=precision, device=0, flags=capi.INPUTS_ON_DEVICE)
    capi.analyze(p, tx, ty, tr, ti, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), runs[0])


def test_sorted_selection_direct_path_equals_sort_path(capi):
    """Strictly increasing indices take the direct-write prep on the host
    path; the device path always sorts: the two agree bit for bit."""
    import torch
    m, d, stride = 16, 8192, 4
    x, y, idx, _ = conditioned_inputs(m, d, stride=stride)
    host = capi.analyze_host(x, y, 1.0, idx, n_steps=20)
    dev = torch.device("cuda", 0)
    out = torch.empty((m, d), dtype=torch.float64, device=dev)
    p = capi.params(d_total=d, d_local=d, obs_dim=idx.size, n_members=m, n_steps=20, obs_kind=1,
                    device=0, flags=capi.INPUTS_ON_DEVICE)
    capi.analyze(p, torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev),
                 torch.ones(idx.size, dtype=torch.float64, device=dev),
                 torch.from_numpy(idx).to(dev), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), host)


@pytest.mark.parametrize("precision,tol", [(1, FP64_TOL), (0, FP32_TOL)])
def test_philox_high_counter_word_window(capi, port, precision, tol):
    """A window at the end of a d_total = 1.34e8 state (config 3 weak-scaled
    to 8 GPUs): from pseudo-step 63 on, the noise blocks q = n >> 1 exceed
    2^32 and use the Philox counter's high word.  The port is pinned there
    against the reference's philox4x32 (tests/test_oracle_golden.py)."""
    d_total, w, m = 134_217_728, 2048, 20
    k0 = d_total - w
    g = np.random.default_rng(17)
    x = g.standard_normal((m, w), dtype=np.float32).astype(np.float64)
    y = g.standard_normal(w, dtype=np.float32).astype(np.float64)
    got = capi.analyze_host(x, y, 1.0, None, k0=k0, d_total=d_total, precision=precision)
    want = port.analyze(x, y, 1.0, None, k0=k0, d_total=d_total)
    assert rel_l2(got, want) <= tol


@pytest.mark.parametrize("precision,tol", [(1, FP64_TOL), (0, FP32_TOL)])
def test_long_step_table(capi, port, precision, tol):
    """n_steps far beyond what a shared-memory step table would hold (the
    reference only requires n_steps >= 10, proj/include/turbda/ensf.hpp:32):
    the kernels read the coefficients from global memory."""
    m, d, s = 8, 256, 12000
    x, y, _, _ = conditioned_inputs(m, d)
    x = x.astype(np.float32).astype(np.float64)
    y = y.astype(np.float32).astype(np.float64)
    got = capi.analyze_host(x, y, 1.0, None, n_steps=s, precision=precision)
    want = port.analyze(x, y, 1.0, None, n_steps=s)
    assert np.isfinite(got).all()
    assert rel_l2(got, want) <= tol


def test_empty_window_without_communicator_is_a_no_op(capi):
    p = capi.params(d_total=4096, k0=4096, d_local=0, obs_dim=0, n_members=8, device=0)
    capi.analyze(p, np.zeros((8, 0)), np.zeros(0), np.zeros(0), None, np.zeros((8, 0)))


def test_pageable_staging_ring_matches_pinned_and_rows(capi):
    """Pageable host arrays above 32 MB go through the pinned staging ring
    (pool-threaded gather / scatter, DMA from pinned slots); pinned arrays and
    per-member row pointers (turbda_ensf_analyze_rows, the C++ Ensemble
    layout) give the same bits."""
    import ctypes as C
    import torch
    m, d = 64, 80_000 + 37  # 41 MB of forecast, ragged chunks
    g = np.random.default_rng(23)
    x = g.standard_normal((m, d))
    y = g.standard_normal(d)
    page = capi.analyze_host(x, y, 1.0, None, n_steps=20)
    px = torch.from_numpy(x).pin_memory().numpy()
    pinned = capi.analyze_host(px, y, 1.0, None, n_steps=20)
    assert np.array_equal(page, pinned)
    rows = [np.array(x[j]) for j in range(m)]
    orows = [np.empty(d) for _ in range(m)]
    rp = (C.c_void_p * m)(*[r.ctypes.data for r in rows])
    op = (C.c_void_p * m)(*[o.ctypes.data for o in orows])
    p = capi.params(d_total=d, d_local=d, obs_dim=d, n_members=m, n_steps=20, device=0)
    capi.analyze_rows(p, rp, y, np.ones(d), None, op)
    assert np.array_equal(np.stack(orows), page)


def test_likelihood_score_and_sde_step_on_device(capi):
    """The C++ API's likelihood_score / reverse_sde_step run on the device
    (turbda_likelihood_score / turbda_reverse_sde_step, proj/src/ensf.cpp:
    84-94,108-130): duplicates add as adjoint_scatter does; a non-finite step
    reports SamplerDivergedError(t)."""
    import ctypes as C
    L = capi.lib()
    vp = C.c_void_p
    L.turbda_likelihood_score.argtypes = [vp, C.c_int64, vp, vp, vp, C.c_int64, C.c_int32, vp,
                                          C.c_int32, C.POINTER(capi.Status)]
    L.turbda_reverse_sde_step.argtypes = [vp, C.c_int32, C.c_int64, C.c_double, C.c_double, vp, vp,
                                          C.c_int32, C.POINTER(capi.Status)]
    g = np.random.default_rng(8)
    d = 1000
    z = g.standard_normal(d)
    idx = np.array([3, 7, 7, 999, 3, 0], np.int64)
    y = g.standard_normal(idx.size)
    r = 0.5 + g.random(idx.size)
    out = np.empty(d)
    st = capi.Status()
    assert L.turbda_likelihood_score(z.ctypes.data, d, y.ctypes.data, r.ctypes.data, idx.ctypes.data,
                                     idx.size, 1, out.ctypes.data, 0, C.byref(st)) == capi.OK
    want = np.zeros(d)
    np.add.at(want, idx, (y - z[idx]) / r)
    assert np.allclose(out, want, rtol=1e-13, atol=1e-15)
    n, t, dt = 3, 0.4, 0.01
    zz = g.standard_normal((n, d))
    sc = g.standard_normal((n, d))
    xi = g.standard_normal((n, d))
    b, s2 = -1.0 / (1.0 - t), 1.0 + 2.0 * t / (1.0 - t)
    want = zz + (-(b * zz - s2 * sc) * dt + np.sqrt(s2 * dt) * xi)
    got = zz.copy()
    assert L.turbda_reverse_sde_step(got.ctypes.data, n, d, t, dt, sc.ctypes.data, xi.ctypes.data, 0,
                                     C.byref(st)) == capi.OK
    assert np.allclose(got, want, rtol=1e-14, atol=1e-14)
    sc[1, 5] = np.inf
    assert L.turbda_reverse_sde_step(zz.ctypes.data, n, d, t, dt, sc.ctypes.data, xi.ctypes.data, 0,
                                     C.byref(st)) == capi.DIVERGED
    assert st.diverged_t == t


@pytest.mark.parametrize("precision,tol", [(1, FP64_TOL), (0, FP32_TOL)])
@pytest.mark.parametrize("m,d", [(20, 8192), (64, 3000)])
def test_selection_without_observations_in_the_window(capi, port, precision, tol, m, d):
    """A selection operator whose window holds no observation (obs_dim = 0,
    or every index outside [k0, k0 + d)): the prep leaves {A, B} = 0 through
    a memset alone, so the fused kernel (a programmatic dependent launch)
    follows a memset, not a kernel; the analysis is the prior-only sampler."""
    x, _, _, _ = conditioned_inputs(m, d)
    x = x.astype(np.float32).astype(np.float64)
    want = port.analyze(x, np.zeros(0), 1.0, np.zeros(0, np.int64), n_steps=20)
    got = capi.analyze_host(x, np.zeros(0), 1.0, np.zeros(0, np.int64), n_steps=20,
                            precision=precision)
    assert np.isfinite(got).all()
    assert rel_l2(got, want) <= tol
    # the same state as the window [d, 2d) of a 2d state whose observations all
    # sit in the other half
    idx = np.arange(0, d, 7, dtype=np.int64)
    y = np.ones(idx.size)
    got_w = capi.analyze_host(x, y, 1.0, idx, n_steps=20, k0=d, d_total=2 * d,
                              precision=precision)
    want_w = port.analyze(x, y[:0], 1.0, idx[:0], n_steps=20, k0=d, d_total=2 * d)
    assert rel_l2(got_w, want_w) <= tol


@pytest.mark.parametrize("m", [9, 21, 23, 41])
def test_fp64_padding_warps_exit(capi, port, m):
    """The fp64 kernel runs P = 2 particles per warp in 4-warp CTAs; warps
    past the last particle leave before integrating (N = 21: 11 groups, the
    third CTA has one padding warp; odd N: the last warp's second particle is
    padding).  Parity with the C restatement and the lowest-particle
    divergence verdict are unaffected."""
    x, y, _, _ = conditioned_inputs(m, 1000)
    got = capi.analyze_host(x, y, 1.0, None, n_steps=20, precision=capi.FP64)
    want = port.analyze(x, y, 1.0, None, n_steps=20)
    assert rel_l2(got, want) <= FP64_TOL
    r = np.ones(1000)
    r[3] = 1e-300  # diverges in every particle: the verdict names particle 0
    with pytest.raises(capi.TurbdaError) as ei:
        capi.analyze_host(x, y, r, None, n_steps=20, precision=capi.FP64)
    assert ei.value.code == capi.DIVERGED and ei.value.diverged_particle == 0
