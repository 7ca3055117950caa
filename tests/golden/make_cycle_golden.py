"""Golden records of BASELINE config 2 cycled, made by the REFERENCE itself.

    python tests/golden/make_cycle_golden.py      # on the GPU box (cuFFTW)

The reference's own cycle driver (proj/src/osse.cpp:182-253 run_experiment,
with proj/src/{sqg,spectral,forecast,config}.cpp and the EnSF hot path,
compiled unmodified against cuFFTW into oracle/_ref/libturbda_ref_cycle.so by
oracle/Makefile) runs the twin experiment of BASELINE config 2 - a
256 x 256 x 2 SQG grid (d = 131,072), N = 64 members, S = 100 pseudo-steps,
every-4th-point observations, 20 assimilation cycles - on the host cores
(the analysis) and cuFFT (the FFTs of its SQG model).  The per-cycle records
(cycle, time, forecast/analysis rmse and spread) go to
tests/golden/cycle_cfg2_reference.json, which travels with the repo;
tests/test_gpu_cycle.py compares the GPU-resident driver against them.  The
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

OUT = Path(__file__).resolve().parent / "cycle_cfg2_reference.json"


def cfg2_config() -> dict:
    """BASELINE config 2 in the reference's JSON schema (proj/src/config.cpp:
    64-131).  lx grows with nx so the grid spacing of the 64^2 default is kept
    (as proj/tests/helpers.hpp:15-20 does), so the default dt stays stable."""
    n = 256
    lx = 2 * math.pi * 10 * n / 64
    return {"grid": {"nx": n, "ny": n, "lx": lx, "ly": lx}, "cycles": 20, "ensemble_size": 64,
            "spinup_hours": 2400.0, "clim_hours": 1200.0, "variant": "ensf",
            "obs": {"thinning_stride": 4}, "ensf": {"n_steps": 100}, "seed": 7}


def main():
    cfg = cfg2_config()
    refc = RefCycleOracle(ROOT / "oracle" / "_ref" / "libturbda_ref_cycle.so")
    t0 = time.perf_counter()
    rec = refc.run_experiment(cfg)
    wall = time.perf_counter() - t0
    OUT.write_text(json.dumps({
        "config": cfg,
        "records": [{k: float(v) for k, v in r.items()} for r in rec],
        "generator": "tests/golden/make_cycle_golden.py: the reference's run_experiment "
                     "(oracle/_ref/libturbda_ref_cycle.so, proj/src/osse.cpp:182-253 unmodified, "
                     "cuFFTW for its SQG FFTs)",
        "host_threads": host_cores(), "wall_s": wall}, indent=1))
    print(f"wrote {OUT} ({len(rec)} cycles, {wall:.0f} s)")


if __name__ == "__main__":
    main()
