"""Golden records of BASELINE config 2 cycled, made by the REFERENCE itself.

    python tests/golden/make_cycle_golden.py [long|short] [OUT.json]   # GPU box (cuFFTW)

The reference's own cycle driver (proj/src/osse.cpp:182-253 run_experiment,
with proj/src/{sqg,spectral,forecast,config}.cpp and the EnSF hot path,
compiled unmodified against cuFFTW into oracle/_ref/libturbda_ref_cycle.so by
oracle/Makefile) runs the twin experiment of BASELINE config 2 - a
256 x 256 x 2 SQG grid (d = 131,072), N = 64 members, S = 100 pseudo-steps,
every-4th-point observations, 20 assimilation cycles - on the host cores
(the analysis) and cuFFT (the FFTs of its SQG model).  The per-cycle records
(cycle, time, forecast/analysis rmse and spread) go to
tests/golden/cycle_cfg2_reference.json ("long": 2400 h spin-up, the
climate the time-mean RMSE statistic is taken in) and
tests/golden/cycle_cfg2_short_reference.json ("short": 240 h spin-up, so the
chaotic SQG nature run has not amplified the rounding difference between
cuFFT-based models beyond ~1e-11 and whole trajectories can be compared),
which travel with the repo; tests/test_gpu_cycle.py compares the
GPU-resident driver against them.  The
reference needs a GPU only for cuFFTW, and /root/reference is not needed at
run time (the library is prebuilt into oracle/_ref).
"""
from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import RefCycleOracle, host_cores  # noqa: E402

HERE = Path(__file__).resolve().parent
OUT = {"long": HERE / "cycle_cfg2_reference.json", "short": HERE / "cycle_cfg2_short_reference.json"}


def cfg2_config(variant: str = "long") -> dict:
    """BASELINE config 2 in the reference's JSON schema (proj/src/config.cpp:
    64-131).  lx grows with nx so the grid spacing of the 64^2 default is kept
    (as proj/tests/helpers.hpp:15-20 does), so the default dt stays stable."""
    n = 256
    lx = 2 * math.pi * 10 * n / 64
    spin, clim = (2400.0, 1200.0) if variant == "long" else (240.0, 800.0)
    return {"grid": {"nx": n, "ny": n, "lx": lx, "ly": lx}, "cycles": 20, "ensemble_size": 64,
            "spinup_hours": spin, "clim_hours": clim, "variant": "ensf",
            "obs": {"thinning_stride": 4}, "ensf": {"n_steps": 100}, "seed": 7}


def main():
    variant = sys.argv[1] if len(sys.argv) > 1 else "long"
    out = Path(sys.argv[2]) if len(sys.argv) > 2 else OUT[variant]
    cfg = cfg2_config(variant)
    refc = RefCycleOracle(ROOT / "oracle" / "_ref" / "libturbda_ref_cycle.so")
    t0 = time.perf_counter()
    rec = refc.run_experiment(cfg)
    wall = time.perf_counter() - t0
    out.write_text(json.dumps({
        "config": cfg,
        "records": [{k: float(v) for k, v in r.items()} for r in rec],
        "generator": "tests/golden/make_cycle_golden.py: the reference's run_experiment "
                     "(oracle/_ref/libturbda_ref_cycle.so, proj/src/osse.cpp:182-253 unmodified, "
                     "cuFFTW for its SQG FFTs)",
        "host_threads": host_cores(), "wall_s": wall}, indent=1))
    print(f"wrote {out} ({len(rec)} cycles, {wall:.0f} s)")


if __name__ == "__main__":
    main()
