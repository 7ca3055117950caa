"""The Python boundary (SURVEY 8(b) "Python _core"): the package against the
reference's own binding (proj/python/bindings.cpp, built unmodified into
oracle/_ref/refpy over the reference sources; every reference call runs in a
subprocess, see oracle.oracle.RefPython).  CPU: the configuration schema.
GPU: the model, both filters and the twin experiment."""
from __future__ import annotations

import json

import numpy as np
import pytest

from oracle.oracle import RefPython, rel_l2

L16 = 2 * np.pi * 10 / 4


@pytest.fixture(scope="module")
def ref():
    try:
        return RefPython()
    except FileNotFoundError as e:
        pytest.skip(str(e))


def test_default_config_and_hash_match_reference(ref):
    import paper_2407_12168_b200 as tb
    got = ref.run("out['json'] = ref.default_config_json()\n"
                  "out['hash'] = ref.config_hash(out['json'])\n"
                  "c = __import__('json').loads(out['json']); c['variant'] = 'letkf';"
                  " c['obs']['thinning_stride'] = 4; c['cycles'] = 7\n"
                  "out['hash2'] = ref.config_hash(__import__('json').dumps(c))")
    assert tb.default_config_json() == got["json"]  # byte-identical JSON
    assert tb.config_hash(got["json"]) == got["hash"]
    c = json.loads(tb.default_config_json())
    c["variant"], c["obs"]["thinning_stride"], c["cycles"] = "letkf", 4, 7
    assert tb.config_hash(json.dumps(c)) == got["hash2"]


def test_binding_surface():
    import paper_2407_12168_b200 as tb
    for name in ("GridSpec", "SqgParams", "nature_run", "advance", "ensf_analyze",
                 "letkf_analyze", "run_experiment", "default_config_json", "config_hash",
                 "ke_spectrum", "fit_loglog_slope", "vit_param_count", "estimate_training_flops",
                 "format_sig", "ConfigError", "DimensionError"):
        assert hasattr(tb, name), name
    p = tb.SqgParams()
    assert (p.f, p.n, p.u0, p.hyper_order, p.dt) == (1.0, 10.0, 0.1, 4, 0.25)
    with pytest.raises(tb.ConfigError):
        tb.config_hash(json.dumps({"variant": "kalman"}))


def _grid(tb, n=16):
    g = tb.GridSpec()
    g.nx = g.ny = n
    g.lx = g.ly = L16 * n / 16
    return g


def test_budget_helpers_match_reference(ref):
    import paper_2407_12168_b200 as tb
    got = ref.run("out['p'] = ref.vit_param_count(24, 2048, 4.0)\n"
                  "out['f'] = ref.estimate_training_flops([256, 256], [4, 4], 100.0, 2.5e9, 1e6)\n"
                  "out['s'] = [ref.format_sig(v, d) for v, d in ((1.208e9, 4), (6.144e21, 3),"
                  " (0.0, 4), (-3.25e-7, 2), (999.96, 4))]")
    assert tb.vit_param_count(24, 2048, 4.0) == got["p"]
    assert tb.estimate_training_flops([256, 256], [4, 4], 100.0, 2.5e9, 1e6) == got["f"]
    assert [tb.format_sig(v, d) for v, d in ((1.208e9, 4), (6.144e21, 3), (0.0, 4),
                                            (-3.25e-7, 2), (999.96, 4))] == got["s"]
    with pytest.raises(tb.ConfigError):
        tb.estimate_training_flops([256, 255], [4, 4], 1.0, 1.0, 1.0)


def test_fit_loglog_slope_matches_reference(ref):
    import paper_2407_12168_b200 as tb
    rng = np.random.default_rng(3)
    kappa = np.arange(12) * 0.3
    energy = np.abs(rng.standard_normal(12)) * np.concatenate([[0.0], kappa[1:] ** -3.0])
    energy[5] = 0.0  # empty bins (and kappa = 0) are skipped
    got = ref.run("out['s'] = ref.fit_loglog_slope(kappa, energy, 1, 10)\n"
                  "out['t'] = ref.fit_loglog_slope(kappa, energy, -3, 40)",
                  kappa=kappa, energy=energy)
    assert tb.fit_loglog_slope(kappa, energy, 1, 10) == pytest.approx(got["s"], rel=1e-14)
    assert tb.fit_loglog_slope(kappa, energy, -3, 40) == pytest.approx(got["t"], rel=1e-14)
    with pytest.raises(tb.ConfigError):
        tb.fit_loglog_slope(kappa, energy, 5, 6)


@pytest.mark.gpu
def test_model_calls_match_reference(ref):
    import paper_2407_12168_b200 as tb
    got = ref.run(
        "g = ref.GridSpec(); g.nx = g.ny = 16; g.lx = g.ly = L\n"
        "p = ref.SqgParams()\n"
        "snaps = ref.nature_run(g, p, 48.0, 24.0, 12.0, 3)\n"
        "out['snaps'] = np.stack(snaps)\n"
        "out['adv'] = ref.advance(g, p, snaps[-1], 6.0)\n"
        "out['k'], out['e'] = ref.ke_spectrum(g, p, snaps[-1])", L=L16)
    g, p = _grid(tb), tb.SqgParams()
    snaps = np.stack(tb.nature_run(g, p, 48.0, 24.0, 12.0, 3))
    assert snaps.shape == got["snaps"].shape == (3, 2, 16, 16)
    assert rel_l2(snaps, got["snaps"]) < 1e-9
    adv = tb.advance(g, p, got["snaps"][-1], 6.0)
    assert adv.shape == (2, 16, 16) and rel_l2(adv, got["adv"]) < 1e-11
    k, e = tb.ke_spectrum(g, p, got["snaps"][-1])
    assert np.array_equal(k, got["k"]) and rel_l2(e, got["e"]) < 1e-12


@pytest.mark.gpu
def test_filters_match_reference(ref):
    import paper_2407_12168_b200 as tb
    g = _grid(tb)
    rng = np.random.default_rng(0)
    truth = rng.standard_normal(512)
    members = (truth[None, :] + rng.standard_normal((8, 512))).astype(np.float32).astype(np.float64)
    y = (truth + rng.standard_normal(512)).astype(np.float32).astype(np.float64)
    got = ref.run(
        "g = ref.GridSpec(); g.nx = g.ny = 16; g.lx = g.ly = L\n"
        "out['ensf'] = ref.ensf_analyze(members, g, y, r=1.0, seed=9, cycle=1, n_steps=40)\n"
        "out['letkf'] = ref.letkf_analyze(members, g, y, r=0.7, cutoff_km=2500.0)",
        L=L16, members=members, y=y)
    fast = tb.ensf_analyze(members, g, y, r=1.0, seed=9, cycle=1, n_steps=40)
    faithful = tb.ensf_analyze(members, g, y, r=1.0, seed=9, cycle=1, n_steps=40,
                               precision="fp64")
    assert rel_l2(faithful, got["ensf"]) < 1e-10
    assert rel_l2(fast, got["ensf"]) < 1e-4
    lk = tb.letkf_analyze(members, g, y, r=0.7, cutoff_km=2500.0)
    assert rel_l2(lk, got["letkf"]) < 1e-9


@pytest.mark.gpu
def test_run_experiment_matches_reference(ref):
    import paper_2407_12168_b200 as tb
    cfg = json.loads(tb.default_config_json())
    cfg["grid"].update(nx=16, ny=16, lx=L16, ly=L16)
    cfg.update(cycles=3, ensemble_size=4, spinup_hours=24.0, clim_hours=48.0)
    cfg["ensf"]["n_steps"] = 20
    keys = ("forecast_rmse", "analysis_rmse", "forecast_spread", "analysis_spread")
    for variant in ("ensf", "letkf", "free_run"):
        cfg["variant"] = variant
        text = json.dumps(cfg)
        got = ref.run("out['rec'] = ref.run_experiment(text)", text=text)["rec"]
        mine_cfg = json.loads(text)
        mine_cfg["ensf"]["precision"] = "fp64"  # the faithful arithmetic of the reference
        mine = tb.run_experiment(json.dumps(mine_cfg))
        assert [r["cycle"] for r in mine] == [r["cycle"] for r in got] == [1, 2, 3]
        a = np.array([[r[k] for k in keys] for r in mine])
        b = np.array([[r[k] for k in keys] for r in got])
        assert rel_l2(a, b) < 1e-8, variant
