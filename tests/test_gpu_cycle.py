"""GPU forecast model and GPU-resident cycle driver against the reference's
own SQG model and run_experiment (oracle/ref_cycle_shim.cpp: the unmodified
proj/src/{sqg,spectral,forecast,osse,config}.cpp built against cuFFTW, so the
reference arm needs the GPU box too).

Tolerances: the GPU SQG restates the reference's fp64 algorithm on the same
FFT library (cuFFT under cuFFTW), so short integrations agree to ~1e-12;
cycled runs with the fp64 faithful analysis agree to ~1e-9 over a few cycles
(chaos amplifies rounding over time); the LETKF variant runs the reference
driver with its own LETKF (proj/src/letkf.cpp over oracle/ref_shadow/Eigen); the fp32 analysis is compared through
the time-mean analysis RMSE (north_star: "analysis RMSE against truth over a
cycled SQG run must match within a stated tolerance"): 5 %.
"""
import json

import numpy as np
import pytest

from conftest import ROOT
from oracle.oracle import RefCycleOracle, rel_l2

pytestmark = pytest.mark.gpu

L16 = 2 * np.pi * 10 / 4  # keeps dx of the 64^2 default at 16^2 (proj/tests/helpers.hpp:15-20)


@pytest.fixture(scope="module")
def refc():
    p = ROOT / "oracle" / "_ref" / "libturbda_ref_cycle.so"
    if not p.exists():
        pytest.skip("oracle/_ref/libturbda_ref_cycle.so not built")
    return RefCycleOracle(p)


@pytest.fixture(scope="module")
def tb():
    import paper_2407_12168_b200 as m
    if m.device_count() < 1:
        pytest.fail("no CUDA device")
    return m


def small_config(**kw):
    cfg = {"grid": {"nx": 16, "ny": 16, "lx": L16, "ly": L16}, "cycles": 4, "ensemble_size": 6,
           "spinup_hours": 48.0, "clim_hours": 96.0, "variant": "ensf",
           "ensf": {"n_steps": 40}}
    for k, v in kw.items():
        if isinstance(v, dict) and isinstance(cfg.get(k), dict):
            cfg[k] = {**cfg[k], **v}
        else:
            cfg[k] = v
    return cfg


def test_sqg_advance_vs_reference(tb, refc):
    from paper_2407_12168_b200 import capi
    for n, lx in ((16, L16), (64, 2 * np.pi * 10)):
        state = refc.nature_run(n, n, lx, lx, 48.0, 0.0, 12.0, 5)[0]
        want, cfl_ref = refc.sqg_advance(state, 12.0, n, n, lx, lx)
        model = capi.SqgModel(batch=1, nx=n, ny=n, lx=lx, ly=lx)
        got = model.advance(state.reshape(1, 2, n, n).copy(), 12.0).ravel()
        assert rel_l2(got, want) <= 1e-11, (n, rel_l2(got, want))
        assert model.max_cfl == pytest.approx(cfl_ref, rel=1e-9)


def test_sqg_batch_members_independent(tb):
    from paper_2407_12168_b200 import capi
    snaps = capi.nature_run(24.0, 36.0, 12.0, 3, nx=16, ny=16, lx=L16, ly=L16)
    batch = snaps.reshape(-1, 2, 16, 16).copy()
    m3 = capi.SqgModel(batch=batch.shape[0], nx=16, ny=16, lx=L16, ly=L16)
    got = m3.advance(batch.copy(), 6.0)
    m1 = capi.SqgModel(batch=1, nx=16, ny=16, lx=L16, ly=L16)
    for b in range(batch.shape[0]):
        one = m1.advance(batch[b:b + 1].copy(), 6.0)
        assert rel_l2(one, got[b:b + 1]) <= 1e-14


def test_nature_run_vs_reference(tb, refc):
    from paper_2407_12168_b200 import capi
    want = refc.nature_run(32, 32, L16 * 2, L16 * 2, 48.0, 24.0, 12.0, 11)
    got = capi.nature_run(48.0, 24.0, 12.0, 11, nx=32, ny=32, lx=L16 * 2, ly=L16 * 2)
    assert got.shape == want.shape
    assert rel_l2(got, want) <= 1e-9, rel_l2(got, want)


def test_sqg_rejects_bad_duration_and_blows_up(tb):
    from paper_2407_12168_b200 import capi
    m = capi.SqgModel(batch=1, nx=16, ny=16, lx=L16, ly=L16)
    with pytest.raises(capi.TurbdaError) as ei:
        m.advance(np.zeros((1, 2, 16, 16)), 0.1)
    assert ei.value.code == capi.CONFIG
    x = np.zeros((1, 2, 16, 16))
    x[0, 0, 3, 3] = np.inf
    with pytest.raises(capi.TurbdaError) as ei:
        m.advance(x, 1.0)
    assert ei.value.code == capi.BLOWUP and ei.value.diverged_particle == 0


@pytest.mark.parametrize("extra", [{}, {"model_quality": "imperfect"},
                                   {"obs": {"thinning_stride": 4}}, {"variant": "free_run"},
                                   {"variant": "letkf"},
                                   {"variant": "letkf", "obs": {"thinning_stride": 3},
                                    "letkf": {"cutoff_km": 3000.0, "rtps_alpha": 0.5}}])
def test_run_experiment_fp64_vs_reference(tb, refc, extra):
    cfg = small_config(**extra)
    want = refc.run_experiment(cfg)
    cfg_gpu = json.loads(json.dumps(cfg))
    cfg_gpu.setdefault("ensf", {})["precision"] = "fp64"
    got = tb.run_experiment(json.dumps(cfg_gpu))
    assert [r["cycle"] for r in got] == [int(r["cycle"]) for r in want]
    keys = ("time", "forecast_rmse", "analysis_rmse", "forecast_spread", "analysis_spread")
    a = np.array([[r[k] for k in keys] for r in got])
    b = np.array([[r[k] for k in keys] for r in want])
    assert rel_l2(a, b) <= 1e-8, (extra, rel_l2(a, b))


def test_run_experiment_fp32_time_mean_rmse(tb, refc):
    cfg = small_config(cycles=8)
    want = refc.run_experiment(cfg)
    got = tb.run_experiment(json.dumps(cfg))
    m_ref = np.mean([r["analysis_rmse"] for r in want])
    m_gpu = np.mean([r["analysis_rmse"] for r in got])
    print(f"time-mean analysis RMSE: reference {m_ref:.5f}  B200 fp32 {m_gpu:.5f}")
    assert abs(m_gpu - m_ref) <= 0.05 * m_ref


def test_run_experiment_fault_injection_like_reference(tb, refc):
    """Fault injection after proj/tests/test_osse.cpp:207-226 (dt = 6 h, CFL far
    above stability): the GPU driver fails where the reference fails, with the
    same kind of error (blowup / diverged sampler) and, inside the cycle loop,
    the same cycle."""
    import re
    from paper_2407_12168_b200 import capi
    cfg = small_config(sqg={"dt": 6.0, "u0": 50.0}, cycles=40, spinup_hours=0.0, clim_hours=96.0)
    cfg["ensf"]["precision"] = "fp64"
    ref_err = None
    try:
        refc.run_experiment(cfg)
    except Exception as e:  # OracleError
        ref_err = str(e)
    ours = None
    try:
        tb.run_experiment(json.dumps(cfg))
    except (capi.TurbdaError, ValueError) as e:
        ours = str(e)
    print("reference:", ref_err, "| B200:", ours)
    assert (ref_err is None) == (ours is None)
    if ours is not None:
        assert ("blowup" in ours) == ("blowup" in ref_err)
        rt, ot = re.search(r"t=([0-9.]+)", ref_err), re.search(r"t=([0-9.]+)", ours)
        if rt and ot:
            assert float(rt.group(1)) == pytest.approx(float(ot.group(1)))
        rc, oc = re.search(r"cycle (\d+)", ref_err), re.search(r"cycle (\d+)", ours)
        assert (rc is None) == (oc is None)
        if rc:
            assert rc.group(1) == oc.group(1)


def test_letkf_cycle_beats_free_run(tb):
    """proj/tests/test_osse.cpp:181-205: assimilation (LETKF) beats the free
    run on its own forecasts."""
    base = small_config(cycles=6, ensemble_size=8, model_quality="imperfect")
    free = tb.run_experiment(json.dumps({**base, "variant": "free_run"}))
    lk = tb.run_experiment(json.dumps({**base, "variant": "letkf"}))
    mean = lambda rs: np.mean([r["analysis_rmse"] for r in rs])
    assert mean(lk) < mean(free)
    for r in lk:
        assert np.isfinite(r["analysis_rmse"]) and r["analysis_spread"] > 0


def test_snapshot_checkpoint_of_device_ensemble(tb, tmp_path):
    """A device-resident ensemble checkpoints straight from HBM (SQGSNAP v1,
    one header per member) and reads back bit-exactly."""
    import torch
    from paper_2407_12168_b200 import capi
    ens = torch.randn(4, 2, 16, 16, dtype=torch.float64, device="cuda:0")
    p = tmp_path / "ens.sqg"
    capi.snapshot_write(p, ens, 24.0, flags=capi.INPUTS_ON_DEVICE)
    back, t = capi.snapshot_read(p)
    assert t == 24.0 and np.array_equal(back, ens.cpu().numpy())


# --- BASELINE config 2 cycled, against the reference's own records ----------
# tests/golden/cycle_cfg2_reference.json is written on the GPU box by
# tests/golden/make_cycle_golden.py from the reference's run_experiment
# (proj/src/osse.cpp:182-253, unmodified, cuFFTW): 256 x 256 x 2, N = 64,
# S = 100, every-4th-point observations, 20 cycles.
CFG2_GOLDEN = ROOT / "tests" / "golden" / "cycle_cfg2_reference.json"
CFG2_SHORT = ROOT / "tests" / "golden" / "cycle_cfg2_short_reference.json"
REC_KEYS = ("time", "forecast_rmse", "analysis_rmse", "forecast_spread", "analysis_spread")


def _cfg2_golden(path=CFG2_GOLDEN):
    if not path.exists():
        pytest.skip(f"{path.name} not generated")
    return json.loads(path.read_text())


def _csv(records):
    """MetricsSeries::to_csv formatting (%.17g, proj/src/osse.cpp:71-99)."""
    return "\n".join(",".join("%.17g" % r[k] for k in ("cycle",) + REC_KEYS) for r in records)


@pytest.mark.slow
def test_cfg2_cycled_fp64_records_vs_reference(tb):
    """The faithful fp64 analysis inside the GPU-resident driver reproduces
    every per-cycle record of the reference's own 20-cycle run to 1e-8
    (short spin-up: 240 h + 800 h of climatology keep the chaotic nature
    run's amplification of the cuFFT rounding differences far below that;
    after the 2400 h spin-up of the long fixture the truths themselves differ
    at 1e-3, which is why that one is compared through its statistics)."""
    g = _cfg2_golden(CFG2_SHORT)
    cfg = json.loads(json.dumps(g["config"]))
    cfg["ensf"]["precision"] = "fp64"
    got = tb.run_experiment(json.dumps(cfg))
    want = g["records"]
    assert [int(r["cycle"]) for r in got] == [int(r["cycle"]) for r in want]
    a = np.array([[r[k] for k in REC_KEYS] for r in got])
    b = np.array([[r[k] for k in REC_KEYS] for r in want])
    err = rel_l2(a, b)
    per_cycle = [rel_l2(a[q], b[q]) for q in range(len(a))]
    print(f"config 2 cycled fp64 vs reference records: rel-L2 {err:.3e}; per cycle "
          + " ".join(f"{e:.1e}" for e in per_cycle))
    assert err <= 1e-8


@pytest.mark.slow
def test_cfg2_cycled_fp32_rmse_within_2pct_and_bitwise_reruns(tb):
    """north_star: analysis RMSE against truth over a cycled SQG run matches
    the reference within a stated tolerance - 2 % on the time-mean analysis
    RMSE for the fp32 fast path - and two runs give
    byte-identical metrics CSVs (proj/tests/test_osse.cpp:163-179)."""
    g = _cfg2_golden()
    cfg = g["config"]
    got = tb.run_experiment(json.dumps(cfg))
    again = tb.run_experiment(json.dumps(cfg))
    assert _csv(got) == _csv(again)
    m_ref = np.mean([r["analysis_rmse"] for r in g["records"]])
    m_gpu = np.mean([r["analysis_rmse"] for r in got])
    f_ref = np.mean([r["forecast_rmse"] for r in g["records"]])
    f_gpu = np.mean([r["forecast_rmse"] for r in got])
    print(f"config 2 time-mean analysis RMSE: reference {m_ref:.6f}  B200 fp32 {m_gpu:.6f} "
          f"(forecast {f_ref:.6f} / {f_gpu:.6f})")
    assert abs(m_gpu - m_ref) <= 0.02 * m_ref
    assert abs(f_gpu - f_ref) <= 0.02 * f_ref


@pytest.mark.slow
def test_cfg5_open_loop_cycles_vs_restatement(tb, port):
    """BASELINE config 5 cycled (1024 x 1024 x 2, N = 128, arctan obs on every
    4th point, 100 cycles) with the GPU-resident driver; at cycles 1, 10, 50
    and 100 the probe returns the forecast and analysis ensembles over a
    768-coordinate window and that cycle's observations, and the C
    restatement (oracle/ensf_oracle.c, arctan likelihood: the extension has
    no reference implementation) recomputes the window's analysis from the
    same forecast with the same (seed, cycle) noise: open-loop per-cycle
    parity at the fp32 tolerance."""
    from paper_2407_12168_b200 import capi
    from paper_2407_12168_b200.experiment import to_struct
    n, m, stride = 1024, 128, 4
    lx = 2 * np.pi * 10 * n / 64
    cfg = {"grid": {"nx": n, "ny": n, "lx": lx, "ly": lx}, "cycles": 100, "ensemble_size": m,
           "spinup_hours": 240.0, "clim_hours": 12.0 * (m + 4), "variant": "ensf",
           "obs": {"thinning_stride": stride, "operator": "arctan"}, "ensf": {"n_steps": 100},
           "seed": 7}
    d = 2 * n * n
    k0, w = 1_500_004, 768
    idx_all = np.arange(0, d, stride, dtype=np.int64)
    e = to_struct(cfg)
    rec, probes = capi.run_experiment_probe(e, [1, 10, 50, 100], k0, w, idx_all.size)
    assert len(rec) == 100 and np.isfinite(rec).all()
    sel = (idx_all >= k0) & (idx_all < k0 + w)
    for k, (fc, an, y) in sorted(probes.items()):
        want = port.analyze(fc, y[sel], e.obs_r, idx_all[sel], n_steps=100, seed=7, cycle=k,
                            k0=k0, d_total=d, arctan=True)
        err = rel_l2(an, want)
        print(f"config 5 cycle {k}: window analysis vs restatement rel-L2 {err:.2e}")
        assert err <= 1e-4, (k, err)
