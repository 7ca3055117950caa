"""Small analyses, one kernel family each, for the bounds-checked build (tools/checked_run.sh)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.oracle import conditioned_inputs  # noqa: E402


def main(case):
    from paper_2407_12168_b200 import capi
    if case == "letkf":
        n, m = 16, 20
        g = np.random.default_rng(1)
        x = g.standard_normal((m, 2 * n * n))
        y = g.standard_normal(2 * n * n)
        capi.letkf_analyze(x, y, 0.5, None, nx=n, ny=n)
        return
    m = {"f32_sorted_multi_cta": 64, "f32_unsorted": 20, "f32_unsorted_generic": 20,
         "f32_minibatch": 32, "f32_exact_tma": 64, "f64": 20, "joint": 16, "joint_big": 130}[case]
    d = 256 + 6  # ragged last tile
    x, y, idx, _ = conditioned_inputs(m, d, stride=3)
    kw = dict(n_steps=12)
    if case == "f32_minibatch":
        kw["minibatch_j"] = 7
    if case == "f64":
        kw["precision"] = capi.FP64
    if case in ("joint", "joint_big"):
        kw["joint"] = True
    out = capi.analyze_host(x, y, 0.8, idx, **kw)
    assert np.isfinite(out).all()


if __name__ == "__main__":
    if sys.argv[1] == "f32_exact_tma":
        os.environ["TURBDA_F32_EXACT_SHIFT"] = "1"
    if sys.argv[1] == "f32_unsorted_generic":
        os.environ["TURBDA_F32_J20"] = "0"
    main(sys.argv[1])
