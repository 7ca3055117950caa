#!/usr/bin/env python
"""LETKF arm timing: GPU turbda_letkf_analyze on
device-resident inputs (CUDA events, median of K runs) next to the CPU C++
restatement of proj/src/letkf.cpp (oracle/letkf_restated.cpp inside the
reference's own types and parallel_for, all host threads).

    python tools/bench_letkf.py [--cpu-max-points N] > profiles/rNN_bench_letkf.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CONFIGS = [
    # (label, nx, members, obs stride)
    ("64x64x2 N=20 identity (config 1 grid)", 64, 20, 1),
    ("128x128x2 N=40 stride 4", 128, 40, 4),
    ("256x256x2 N=64 stride 4 (config 2 grid)", 256, 64, 4),
    ("1024x1024x2 N=64 stride 4 (config 5 grid)", 1024, 64, 4),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--only", type=int, default=-1, help="run CONFIGS[only] alone")
    ap.add_argument("--cpu-max-points", type=int, default=16384,
                    help="run the CPU restatement only up to this many grid points")
    args = ap.parse_args()
    import torch

    from paper_2407_12168_b200 import capi
    from oracle.oracle import RefCycleOracle

    rc = RefCycleOracle()
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream()
    out = []
    for label, n, m, stride in (CONFIGS if args.only < 0 else [CONFIGS[args.only]]):
        d = 2 * n * n
        g = np.random.default_rng(n)
        x = g.standard_normal((m, d))
        idx = None if stride <= 1 else np.arange(0, d, stride, dtype=np.int64)
        nobs = d if idx is None else idx.size
        y = g.standard_normal(nobs)
        tx = torch.from_numpy(x).to(dev)
        ty = torch.from_numpy(y).to(dev)
        tr = torch.tensor([1.0], dtype=torch.float64, device=dev)
        ti = None if idx is None else torch.from_numpy(idx).to(dev)
        tout = torch.empty_like(tx)
        p = capi.letkf_params(nx=n, ny=n, n_members=m, obs_kind=0 if idx is None else 1,
                              obs_dim=nobs, device=0,
                              flags=capi.INPUTS_ON_DEVICE | capi.R_UNIFORM)
        with torch.cuda.stream(stream):
            for _ in range(2):
                capi.letkf_raw(p, tx, ty, tr, ti, None, tout, stream=stream.cuda_stream)
            times = []
            for _ in range(args.steps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                capi.letkf_raw(p, tx, ty, tr, ti, None, tout, stream=stream.cuda_stream)
                b.record(stream)
                b.synchronize()
                times.append(a.elapsed_time(b))
        gpu_ms = float(np.median(times))
        rec = {"workload": label, "points": n * n, "members": m, "obs": int(nobs),
               "gpu_ms": gpu_ms}
        if n * n <= args.cpu_max_points:
            workers = os.cpu_count() or 1
            t0 = time.perf_counter()
            want = rc.letkf_analyze(x, y, 1.0, idx, n, n, workers=workers)
            rec["cpu_restatement_s"] = time.perf_counter() - t0
            rec["cpu_threads"] = workers
            rec["speedup"] = rec["cpu_restatement_s"] * 1e3 / gpu_ms
            got = tout.cpu().numpy()
            rec["max_rel_diff_vs_cpu"] = float(np.abs(got - want).max() / np.abs(want).max())
        print(json.dumps(rec), flush=True)
        out.append(rec)


if __name__ == "__main__":
    main()
