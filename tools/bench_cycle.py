#!/usr/bin/env python
"""Cycled twin experiment on one B200 (BASELINE configs 2 and 5, which the
headline bench.py measures one analysis of): nature run + climatology,
then per cycle the batched SQG forecast, observation synthesis, EnSF
analysis and rmse/spread, all GPU-resident (paper_2407_12168_b200.run_experiment).

    python tools/bench_cycle.py [--config cfg2|cfg5] [--cycles K] [--spinup H]

Prints one JSON line: wall time of the experiment, per-cycle time, the time
of the nature run alone (same call with cycles=1 minus one cycle is not
separable, so it is timed with variant free_run for reference), and the
time-mean analysis RMSE.
"""
import argparse
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

CONFIGS = {
    # 256 x 256 x 2 (d = 131072), N = 64, stride-4 obs, 20 cycles
    "cfg2": dict(n=256, members=64, stride=4, cycles=20),
    # 1024 x 1024 x 2 (d = 2.1M), N = 128, stride-4 obs (arctan), 100 cycles
    "cfg5": dict(n=1024, members=128, stride=4, cycles=100, arctan=True),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--cycles", type=int)
    ap.add_argument("--spinup", type=float, default=7200.0)
    ap.add_argument("--clim", type=float, default=2880.0)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--variant", choices=["ensf", "letkf", "free_run"], default="ensf")
    args = ap.parse_args()
    import paper_2407_12168_b200 as tb
    c = CONFIGS[args.config]
    lx = 2 * math.pi * 10 * c["n"] / 64  # keep the 64^2 grid spacing
    cycles = args.cycles or c["cycles"]
    cfg = {"grid": {"nx": c["n"], "ny": c["n"], "lx": lx, "ly": lx}, "cycles": cycles,
           "ensemble_size": c["members"], "spinup_hours": args.spinup, "clim_hours": args.clim,
           "variant": args.variant, "obs": {"thinning_stride": c["stride"],
                                       "operator": "arctan" if c.get("arctan") else "linear"},
           "ensf": {"precision": args.precision}}
    import numpy as np
    warm = dict(cfg, cycles=1, spinup_hours=0.0, clim_hours=12.0 * (c["members"] + 2))
    tb.run_experiment(json.dumps(warm))  # context, cuFFT plans, kernels loaded
    phases = np.zeros(4)
    t0 = time.perf_counter()
    rec = tb.run_experiment(json.dumps(cfg), phases=phases)
    t_ens = time.perf_counter() - t0
    d = 2 * c["n"] ** 2
    units = d * c["members"] * 100 * cycles
    print(json.dumps({
        "workload": f"{args.config} cycled ({args.variant}): {c['n']}x{c['n']}x2, "
                    f"N={c['members']}, stride-{c['stride']} obs, {cycles} cycles, "
                    f"spinup {args.spinup} h",
        "experiment_wall_s": t_ens,
        "device_s": {"nature_run_and_truth": phases[0], "ensemble_forecasts": phases[1],
                     "analyses_incl_obs": phases[2], "diagnostics": phases[3]},
        "forecast_s_per_cycle": phases[1] / cycles,
        "analysis_s_per_cycle": phases[2] / cycles,
        "analysis_units_per_s": units / phases[2] if args.variant == "ensf" else None,
        "time_mean_forecast_rmse": sum(r["forecast_rmse"] for r in rec) / len(rec),
        "time_mean_analysis_rmse": sum(r["analysis_rmse"] for r in rec) / len(rec),
        "cycles": len(rec)}))


if __name__ == "__main__":
    main()
