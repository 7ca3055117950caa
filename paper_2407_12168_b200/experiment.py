"""Python front-end of the GPU-resident twin experiment, mirroring the
reference binding's ``run_experiment(config_json)`` / ``default_config_json``
(proj/python/bindings.cpp:174-198) and the JSON schema of
``config_from_json`` (proj/src/config.cpp:64-131): absent keys keep the
reference defaults.  Extra keys of this build: ``ensf.precision``
("fp32" | "fp64"), ``ensf.score_mode`` ("componentwise" | "joint"),
``obs.operator`` ("linear" | "arctan").  The whole cycle runs on the GPU
(turbda_run_experiment), the LETKF variant included (turbda_letkf_analyze).
"""
from __future__ import annotations

import json

from . import capi
from ._core import ConfigError

_VARIANTS = {"free_run": capi.VARIANT_FREE_RUN, "letkf": capi.VARIANT_LETKF,
             "ensf": capi.VARIANT_ENSF}


def default_config() -> dict:
    e = capi.experiment()
    g = e.sqg
    return {
        "grid": {"nx": g.nx, "ny": g.ny, "nz": 2, "lx": g.lx, "ly": g.ly, "h": g.h},
        "sqg": {"f": g.f, "n": g.n, "u0": g.u0, "hyper_order": g.hyper_order,
                "hyper_efold": g.hyper_efold, "dt": g.dt, "drag_tau": g.drag_tau,
                "dealias_fraction": 2.0 / 3.0},
        "ensf": {"n_steps": e.n_steps, "eps": e.eps, "minibatch_j": e.minibatch_j,
                 "damping_t": e.damping_t, "relax_factor": e.relax_factor,
                 "precision": "fp32", "score_mode": "componentwise"},
        "model_error": {"enabled": bool(e.me_enabled), "base_amplitude": e.me_base_amplitude,
                        "mixture": [{"probability": e.me_prob[c], "amplitude_fraction": e.me_frac[c]}
                                    for c in range(e.me_ncomp)]},
        "obs": {"r": e.obs_r, "thinning_stride": e.obs_thinning, "operator": "linear"},
        "letkf": {"cutoff_km": e.letkf_cutoff_km, "domain_km": e.letkf_domain_km,
                  "rtps_alpha": e.letkf_rtps_alpha, "obs_thinning": e.letkf_obs_thinning},
        "variant": "ensf", "model_quality": "perfect", "cycles": e.cycles,
        "obs_interval": e.obs_interval, "ensemble_size": e.ensemble_size, "seed": e.seed,
        "spinup_hours": e.spinup_hours, "clim_hours": e.clim_hours,
    }


def default_config_json() -> str:
    return json.dumps(default_config(), indent=2)


def to_struct(cfg: dict) -> "capi.Experiment":
    e = capi.experiment()
    g = cfg.get("grid", {})
    if g.get("nz", 2) != 2:
        raise ConfigError("grid: nz must be 2")
    for k in ("nx", "ny", "lx", "ly", "h"):
        if k in g:
            setattr(e.sqg, k, g[k])
    q = cfg.get("sqg", {})
    for k in ("f", "n", "u0", "hyper_order", "hyper_efold", "dt", "drag_tau"):
        if k in q:
            setattr(e.sqg, k, q[k])
    if abs(q.get("dealias_fraction", 2.0 / 3.0) - 2.0 / 3.0) > 0:
        raise ConfigError("sqg: dealias_fraction is fixed at 2/3")
    f = cfg.get("ensf", {})
    for k in ("n_steps", "eps", "minibatch_j", "damping_t", "relax_factor"):
        if k in f:
            setattr(e, k, f[k])
    e.precision = {"fp32": capi.FP32, "fp64": capi.FP64}[f.get("precision", "fp32")]
    e.score_mode = {"componentwise": capi.SCORE_COMPONENTWISE,
                    "joint": capi.SCORE_JOINT}[f.get("score_mode", "componentwise")]
    me = cfg.get("model_error", {})
    if "enabled" in me:
        e.me_enabled = int(bool(me["enabled"]))
    if "base_amplitude" in me:
        e.me_base_amplitude = me["base_amplitude"]
    if "mixture" in me:
        comps = me["mixture"]
        if len(comps) > 8:
            raise ConfigError("model error: up to 8 mixture components")
        e.me_ncomp = len(comps)
        for c, comp in enumerate(comps):
            e.me_prob[c] = comp["probability"]
            e.me_frac[c] = comp["amplitude_fraction"]
    o = cfg.get("obs", {})
    if "r" in o:
        e.obs_r = o["r"]
    if "thinning_stride" in o:
        e.obs_thinning = o["thinning_stride"]
    e.obs_arctan = int(o.get("operator", "linear") == "arctan")
    lk = cfg.get("letkf", {})
    for k in ("cutoff_km", "domain_km", "rtps_alpha", "obs_thinning"):
        if k in lk:
            setattr(e, "letkf_" + k, lk[k])
    if "variant" in cfg:
        if cfg["variant"] not in _VARIANTS:
            raise ConfigError(f"unknown or unsupported variant '{cfg['variant']}'")
        e.variant = _VARIANTS[cfg["variant"]]
    if "model_quality" in cfg:
        e.model_quality = {"perfect": 0, "imperfect": 1}[cfg["model_quality"]]
    for k in ("cycles", "obs_interval", "ensemble_size", "seed", "spinup_hours", "clim_hours"):
        if k in cfg:
            setattr(e, k, cfg[k])
    return e


def run_experiment(config_json: str, device: int = -1, phases=None) -> list[dict]:
    """One twin experiment; per-cycle metrics as the reference binding returns them.
    ``phases``: optional numpy float64[4] receiving device seconds spent in the
    nature run, the forecasts, the analyses and the diagnostics."""
    e = to_struct(json.loads(config_json))
    try:
        rec, _ = capi.run_experiment_raw(e, device, phases)
    except capi.TurbdaError as err:
        if err.code == capi.CONFIG:
            raise ConfigError(str(err)) from err
        raise
    keys = ("cycle", "time", "forecast_rmse", "analysis_rmse", "forecast_spread",
            "analysis_spread")
    out = []
    for r in rec:
        d = dict(zip(keys, (float(v) for v in r)))
        d["cycle"] = int(d["cycle"])
        out.append(d)
    return out
