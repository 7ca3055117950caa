#!/usr/bin/env python
"""Time the batched GPU SQG forecast (config-2 cycle shape: 64 members of
256 x 256 x 2, one 12 h forecast = 48 RK4 steps) with CUDA events; run
under ncu for the per-kernel split of one step."""
import argparse
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--members", type=int, default=64)
    ap.add_argument("--hours", type=float, default=12.0)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from paper_2407_12168_b200 import capi
    lx = 2 * math.pi * 10 * args.n / 64
    m = capi.SqgModel(batch=args.members, nx=args.n, ny=args.n, lx=lx, ly=lx)
    x = 0.1 * np.random.default_rng(0).standard_normal((args.members, 2, args.n, args.n))
    m.advance(x, 1.0)  # warm-up: plans, graph capture
    ts = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        m.advance(x, args.hours)
        ts.append(time.perf_counter() - t0)
    steps = args.hours / 0.25
    print(f"n={args.n} members={args.members}: {min(ts)*1e3:.1f} ms per {args.hours} h "
          f"({min(ts)/steps*1e3:.3f} ms per RK4 step, host buffers incl. H2D/D2H)")


if __name__ == "__main__":
    main()
