#!/usr/bin/env python
"""EnSF analysis throughput on B200 (BASELINE.json metric: d x N x steps / s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config cfg3|cfg1|cfg2|cfg4|cfg5] [--precision fp32|fp64]
                    [--score componentwise|joint] [--obs linear|arctan]

One "step" is one full EnSF analysis (turbda::analyze: every pseudo-time
step of the reverse SDE + relax_spread) of one synthetic forecast ensemble.

Default workload: BASELINE config 3, the configuration the metric is quoted
on ("at 1/2/4/8 B200"): d = 16,777,216 coordinates (2048x2048x4) per GPU,
N = 20 members, S = 100 pseudo-time steps, identity observations.  With
--gpus N every rank analyses its own 16.8M-coordinate shard of a 16.8M x N
state (weak scaling).  The componentwise score never couples coordinates,
so there is no data-path collective: the barrier and the max-over-ranks of
the device time are the only collectives.  Without an external launcher,
``--gpus N`` (N > 1) re-launches itself under torch.distributed.run with N
ranks (127.0.0.1 rendezvous); a line is printed only when the world size
equals --gpus.

Rank 0 prints ONE JSON line (keys per the driver contract).  The
``cpu_baseline`` leg and ``--impl reference`` time the reference's own CPU
implementation (oracle/_ref: proj/src/ensf.cpp compiled unmodified) on this
host's cores over the same bounded coordinate sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "EnSF analysis steps/sec (d×N×steps/s) at 1/2/4/8 B200; % HBM roofline"
UNIT = "units/s"  # one unit = one (particle, coordinate, pseudo-time step) update

CONFIGS = {
    # name: (d per GPU, N, S, obs stride, description)
    "cfg1": (8192, 20, 50, 1, "BASELINE cfg1 shape: d=8192, N=20, S=50, identity obs"),
    "cfg2": (131072, 64, 100, 4, "BASELINE cfg2: d=131072 (256x256x2), N=64, S=100, every-4th-point obs"),
    "cfg3": (16777216, 20, 100, 1, "BASELINE cfg3: d=16.8M (2048x2048x4) per GPU, N=20, S=100, identity obs"),
    "cfg4": (1048576, 512, 100, 1, "BASELINE cfg4: d=1M, N=512, S=100"),
    "cfg5": (2097152, 128, 100, 4, "BASELINE cfg5 analysis: d=2.1M (1024x1024x2), N=128, S=100, "
                                   "every-4th-point arctan obs"),
}
DEFAULT_CONFIG = "cfg3"
# algorithmic bytes per unit for a per-step-streaming fp32
# design (read z, read x, write z) - the HBM roofline the north star names.
BYTES_PER_UNIT = 12
MUFU_PER_CLK_PER_SM = 16  # ex2 throughput, measured (tools/pipe_microbench.cu)
L2_BYTES = 126 * 2**20


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.nvml_rows = []

    def sample_now(self):
        """One NVML sample, taken while queued timed work is still running
        (covers timed regions shorter than nvidia-smi's start-up)."""
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            flags = ["Active" if rs & b else "Not Active" for b in bits]
            self.nvml_rows.append([str(self.gpu), str(sm), str(mx), "", ""] + flags)
        except Exception:  # noqa: BLE001 - sampling is best effort
            pass

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.gpu)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        rows = []
        try:
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            rows += self.nvml_rows
            if self.path:
                try:
                    os.unlink(self.path)
                except OSError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        loaded = [v for v in sm if mx and v > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def obs_layout(d, stride, k0):
    """Observation indices of a shard: the global flat indices 0, s, 2s, ...
    (make_grid_operator, proj/src/observation.cpp:29-41) inside [k0, k0+d)."""
    if stride <= 1:
        return None, d
    first = (-k0) % stride
    n = len(range(k0 + first, k0 + d, stride))
    return (k0 + first, stride, n), n


def make_inputs_host(d, m, stride, k0, seed=1234):
    """Synthetic forecast for the CPU sample: N(0,1) members and observations
    (the throughput generator of SURVEY.md 8(d); the timing is insensitive
    to the values)."""
    rng = np.random.default_rng(seed + k0)
    x = rng.standard_normal((m, d))
    lay, nobs = obs_layout(d, stride, k0)
    idx = None if lay is None else np.arange(lay[0], lay[0] + lay[1] * lay[2], lay[1],
                                             dtype=np.int64)
    y = rng.standard_normal(nobs)
    return x, y, idx


def make_inputs_device(torch, dev, d, m, stride, k0, seed):
    """The same synthetic shapes generated on the device (a 16.8M x 20
    forecast is 2.7 GB: numpy would spend tens of seconds on it)."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed * 1000003 + k0)
    x = torch.randn((m, d), generator=g, device=dev, dtype=torch.float64)
    lay, nobs = obs_layout(d, stride, k0)
    y = torch.randn((nobs,), generator=g, device=dev, dtype=torch.float64)
    idx = None if lay is None else torch.arange(lay[0], lay[0] + lay[1] * lay[2], lay[1],
                                                dtype=torch.int64, device=dev)
    return x, y, torch.ones_like(y), idx


def reference_rate(x, y, idx, n_steps, steps, warmup, arctan=False):
    """The reference's CPU analyze (oracle/_ref) on the given sample; arctan
    observations (an extension the reference lacks) use the C restatement."""
    from oracle.oracle import RefOracle, host_cores, ref_available
    if arctan or not ref_available():
        from oracle.oracle import PortOracle
        impl, kind = PortOracle(), "port"
    else:
        impl, kind = RefOracle(), "reference"
    cores = host_cores()
    m, d = x.shape
    kw = dict(n_steps=n_steps, seed=7, cycle=1, workers=cores)
    if arctan:
        kw["arctan"] = True
    for _ in range(warmup):
        impl.analyze(x, y, 1.0, idx, **kw)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        impl.analyze(x, y, 1.0, idx, **kw)
        times.append(time.perf_counter() - t0)
    units = float(d) * m * n_steps
    total = sum(times)
    fp_mb = x.nbytes / 1e6
    return {"value": units * steps / total, "unit": UNIT, "cores": min(cores, m),
            "threads_requested": cores, "kind": kind,
            "sample": f"{m} members x {d} coordinates x {n_steps} pseudo-steps (a {d}-coordinate "
                      f"slice of the workload; its {fp_mb:.0f} MB forecast is far more cache-"
                      f"resident than the full state, which flatters the CPU), {warmup} warm-up + "
                      f"{steps} timed run(s), median {statistics.median(times):.3f} s; the "
                      f"reference parallelises over particles only, so at most N={m} threads",
            "ms_per_step": 1e3 * total / steps}


def _cpu_sample(d, m, base):
    """CPU sample width: `base` coordinates at N = 64, scaled by (64/N)^2 (the
    CPU cost grows with N^2 per coordinate) so every config's CPU leg takes
    seconds, a multiple of 64 coordinates."""
    return max(64, min(d, int(base * (64.0 / m) ** 2) // 64 * 64))


def run_reference_arm(args, json_out):
    """--impl reference: rank 0 times the reference's CPU implementation on
    the same config; other ranks exit without work."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    d_full, m, s, stride, desc = CONFIGS[args.config]
    d_sample = _cpu_sample(d_full, m, args.ref_sample_d)
    x, y, idx = make_inputs_host(d_sample, m, stride, 0)
    r = reference_rate(x, y, idx, s, args.steps, args.warmup, arctan=_arctan(args))
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "d_per_gpu": d_full, "members": m, "pseudo_steps": s,
                   "obs_stride": stride, "obs_operator": "arctan" if _arctan(args) else "linear",
                   "sample_d": d_sample},
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"],
                         "kind": r["kind"], "sample": r["sample"]},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=json_out, flush=True)


def _arctan(args):
    """h(x) = atan(x) observations: --obs, defaulting to the config's own
    (BASELINE config 5 observes through arctan)."""
    return (args.obs or ("arctan" if args.config == "cfg5" else "linear")) == "arctan"


def _json_stdout():
    """The one JSON line goes to the original stdout; everything else written
    to fd 1 afterwards (NCCL's version banner, library prints) goes to stderr."""
    out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n, json_out):
    """--gpus N without a launcher: one process per GPU under
    torch.distributed.run (the driver's own launch line); the ranks write to
    the original stdout (rank 0's JSON line), everything else to stderr."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(Path(__file__).resolve())] + sys.argv[1:]
    print(f"bench: spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    json_out.flush()
    return subprocess.call(cmd, stdout=json_out)


def timed_analyses(torch, fn, n, stream):
    """Device time of n back-to-back calls on `stream` (CUDA events)."""
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for q in range(n):
        fn(q)
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / n


def main():
    json_out = _json_stdout()
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=DEFAULT_CONFIG)
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--score", choices=["componentwise", "joint"], default="componentwise",
                    help="joint: the north-star joint-norm extension (fp64, one NCCL allreduce "
                         "of the N x N distances per pseudo-step across ranks)")
    ap.add_argument("--obs", choices=["linear", "arctan"], default=None,
                    help="observation operator (default: arctan for cfg5, linear otherwise)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 faithful-path leg")
    ap.add_argument("--no-e2e-variants", action="store_true",
                    help="skip the pageable / C++ row-pointer end-to-end legs")
    ap.add_argument("--ref-sample-d", type=int, default=8192,
                    help="CPU sample width at N=64 (scaled by (64/N)^2); used by both the "
                         "cpu_baseline leg and --impl reference")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    if args.impl == "reference":
        run_reference_arm(args, json_out)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus, json_out))

    import torch
    import torch.distributed as dist

    from paper_2407_12168_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}: refusing to report",
              file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        if rank == 0:
            print(f"bench: NCCL process group up, nranks={dist.get_world_size()}",
                  file=sys.stderr, flush=True)

    d, m, s, stride, desc = CONFIGS[args.config]
    d_total = d * world
    k0 = rank * d
    joint = args.score == "joint"
    arctan = _arctan(args)
    obs_kind = (0 if stride <= 1 else 1) + (2 if arctan else 0)
    # joint mode: distances/update in fp64 always; --precision picks the noise
    prec = capi.FP32 if args.precision == "fp32" else capi.FP64
    if joint and world > 1:
        uid = [capi.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        capi.comm_init(local, rank, world, uid[0])

    # --- resident inputs -------------------------------------------------------
    # working set > L2: one forecast of m*d*8 bytes per set; small workloads
    # rotate 3 sets and flush L2 before every timed step
    set_bytes = m * d * 8
    n_sets = 1 if set_bytes > 4 * L2_BYTES else 3
    dsets = [make_inputs_device(torch, dev, d, m, stride, k0, seed=1234 + 7 * q)
             for q in range(n_sets)]
    out = torch.empty((m, d), dtype=torch.float64, device=dev)
    obs_dim = dsets[0][1].numel()

    def mkparams(precision, flags, cycle=1):
        # the joint mode's windows share their per-step distances over the
        # library communicator: TURBDA_SHARDED on every rank
        flags |= capi.SHARDED if (joint and world > 1) else 0
        return capi.params(d_total=d_total, k0=k0, d_local=d, obs_dim=obs_dim, n_members=m,
                           n_steps=s, obs_kind=obs_kind, precision=precision, device=local,
                           flags=flags, cycle=cycle,
                           score_mode=capi.SCORE_JOINT if joint else capi.SCORE_COMPONENTWISE)

    p = mkparams(prec, capi.INPUTS_ON_DEVICE | capi.ASYNC)
    stream = torch.cuda.Stream(dev)  # a real stream: the events and kernels share it
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream

    def one(q, pp=p):
        tx, ty, tr, ti = dsets[q % n_sets]
        capi.analyze(pp, tx, ty, tr, ti, out, stream=sh)

    for q in range(args.warmup):
        one(q)
    torch.cuda.synchronize(dev)
    capi.check(local, p)  # divergence verdict of the warm-up runs

    # --- timed region: K device-resident analyses --------------------------------
    flush = set_bytes * (n_sets - 1) <= L2_BYTES if n_sets > 1 else False
    scratch = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev) if flush else None
    capi.profile_enable(True)
    capi.profile_read()
    launches0 = capi.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps if flush else 1)]
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        if flush:
            for q in range(args.steps):
                scratch.zero_()
                evs[q][0].record(stream)
                one(q)
                evs[q][1].record(stream)
                if q == args.steps - 1:
                    clocks.sample_now()
        else:
            evs[0][0].record(stream)
            for q in range(args.steps):
                one(q)
            evs[0][1].record(stream)
            clocks.sample_now()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    launches = capi.launch_count() - launches0
    kernel_ms, kernel_n = capi.profile_read()
    capi.profile_enable(False)
    capi.check(local, p)
    ms = sum(a_.elapsed_time(b_) for a_, b_ in evs) / args.steps
    ms_t = torch.tensor([ms, kernel_ms / max(kernel_n, 1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms, kern_ms = float(ms_t[0]), float(ms_t[1])
    clk = clocks.summary()

    units_per_gpu = float(d) * m * s
    value = units_per_gpu * world / (ms / 1e3)

    # --- fp64 faithful path, same config (device-resident, 1 warm-up + 2) -----
    fp64 = None
    if not args.no_fp64 and not joint and prec == capi.FP32:
        p64 = mkparams(capi.FP64, capi.INPUTS_ON_DEVICE | capi.ASYNC)
        one(0, p64)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        ms64 = timed_analyses(torch, lambda q: one(q, p64), 2, stream)
        capi.check(local, p64)
        t64 = torch.tensor([ms64], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t64, op=dist.ReduceOp.MAX)
        fp64 = {"value": units_per_gpu * world / (float(t64[0]) / 1e3), "unit": UNIT,
                "ms_per_step": float(t64[0]), "steps": 2, "warmup": 1,
                "kernel": "ensf_f64_kernel (the reference's own fp64 arithmetic: "
                          "fast_exp_nonpos, two-pass shift, num/den score)"}

    # --- end to end through the public API with host buffers -------------------
    import paper_2407_12168_b200 as tb
    grid = tb.GridSpec()
    # any (nx, ny, nz=2) whose size is d: the API only checks the size
    grid.nz = 2
    grid.nx = 256 if d % 512 == 0 else d // 2
    grid.ny = d // (2 * grid.nx)
    tx0, ty0, _, ti0 = dsets[0]
    hx = torch.empty((m, d), dtype=torch.float64, pin_memory=True)
    hx.copy_(tx0)
    hy = torch.empty((obs_dim,), dtype=torch.float64, pin_memory=True)
    hy.copy_(ty0)
    hx, hy = hx.numpy(), hy.numpy()
    hidx = None if ti0 is None else ti0.cpu().numpy()
    hout = torch.empty((m, d), dtype=torch.float64, pin_memory=True).numpy()
    del dsets, out
    torch.cuda.empty_cache()

    def e2e_call(q, out_arr=hout, x_arr=hx, y_arr=hy):
        if joint and world > 1:
            # a window of the sharded state: the C-ABI with host buffers
            pe = mkparams(prec, 0, cycle=1 + q)
            capi.analyze(pe, x_arr, y_arr, np.ones_like(y_arr), hidx, out_arr)
            return out_arr
        return tb.ensf_analyze(x_arr, grid, y_arr, r=1.0, seed=7, cycle=1 + q, n_steps=s,
                               thinning=stride if stride > 1 else 0,
                               precision=args.precision, device=local,
                               obs_operator="arctan" if arctan else "linear",
                               score_mode=args.score, out=out_arr)

    def wall(fn, n_warm, n_timed):
        for q in range(n_warm):
            fn(q)
        if world > 1:
            dist.barrier()
        ts = []
        for q in range(n_timed):
            t0 = time.perf_counter()
            fn(n_warm + q)
            ts.append(time.perf_counter() - t0)
        t = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    e2e_s = wall(e2e_call, args.warmup, args.steps)
    res_bytes = hout.nbytes
    e2e_value = units_per_gpu * world / e2e_s
    if joint and world > 1:
        h2d = hx.nbytes + hy.nbytes * (3 if stride > 1 else 2)  # x, y, r (+ idx)
    else:
        # x, y (+ the thinning operator's idx, built from `thinning`), one r
        h2d = hx.nbytes + hy.nbytes * (2 if stride > 1 else 1) + 8
    d2h = res_bytes + 8  # the analysis + the divergence word

    # the reference's own call shapes: pageable numpy in, fresh array out
    # (proj/python/bindings.cpp:140-155) and the C++ Ensemble's member rows
    # (turbda::analyze, proj/src/ensf.cpp:132 -> turbda_ensf_analyze_rows)
    variants = {}
    if not args.no_e2e_variants and world == 1 and not joint:
        px = np.array(hx)  # pageable copy
        py_ = np.array(hy)
        t_page = wall(lambda q: e2e_call(q, out_arr=None, x_arr=px, y_arr=py_), 1, 2)
        variants["pageable_fresh_out"] = {
            "value": units_per_gpu / t_page, "unit": UNIT, "s_per_step": t_page,
            "path": "paper_2407_12168_b200.ensf_analyze(members, grid, y) - the reference "
                    "binding's signature: pageable float64 numpy in, freshly allocated array out"}
        rows = [np.array(px[j]) for j in range(m)]  # separately allocated member vectors
        orows = [np.empty(d) for _ in range(m)]
        rp = (capi.C.c_void_p * m)(*[r_.ctypes.data for r_ in rows])
        op = (capi.C.c_void_p * m)(*[o_.ctypes.data for o_ in orows])
        ridx = None if hidx is None else np.ascontiguousarray(hidx)
        ones = np.ones(1)

        def rows_call(q):
            pr = mkparams(prec, capi.R_UNIFORM, cycle=1 + q)
            capi.analyze_rows(pr, rp, py_, ones, ridx, op)

        t_rows = wall(rows_call, 1, 2)
        variants["cpp_member_rows"] = {
            "value": units_per_gpu / t_rows, "unit": UNIT, "s_per_step": t_rows,
            "path": "turbda_ensf_analyze_rows (what turbda::analyze(const Ensemble&, ...) calls): "
                    "one pageable std::vector<double> per member in and out"}
        del px, rows, orows

    # --- roofline of the fused analysis kernel -------------------------------
    pk, pk_kind = peaks()
    units_per_launch = units_per_gpu
    # joint mode streams Z and X every pseudo-step in fp64: z read twice and
    # written once (24 B) + two passes over X amortised over N particles
    bytes_per_unit = (24 + 16 * m / m) if joint else BYTES_PER_UNIT
    achieved_gbs = bytes_per_unit * units_per_launch / (kern_ms / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"{args.config}_{args.precision}_{args.score}")
        except ValueError:
            traffic = None
    pair_evals = units_per_launch * m
    # sorted member tiles take 1/8 of the exponentials on the FMA pipe when
    # four tiles fit an SM (24 < N <~ 200) or one 32-warp CTA holds one
    # (440 <~ N <~ 800); ensf_kernels.cu launch_f32_p
    poly_share = 0.125 if (not joint and (24 < m <= 200 or 440 <= m <= 800)) else 0.0
    xu_ops_per_unit = m * (1.0 - poly_share) + 2.0
    mufu_peak = MUFU_PER_CLK_PER_SM * 148 * pk.get("sm_max_mhz", 1965.0) * 1e6
    fp64_peak = 64 * 2 * 148 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    roofline = {
        "bound": "hbm", "achieved": achieved_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
        "frac": achieved_gbs / pk["hbm_gbs"], "traffic": traffic,
        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})",
        "algorithmic_bytes_per_unit": bytes_per_unit, "units_per_launch": units_per_launch,
        "kernel": ("joint: gram_partial + reduce + allreduce + softmax + apply, all steps" if joint
                   else "ensf_f32_kernel" if prec == capi.FP32 else "ensf_f64_kernel"),
        "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms,
        "binding_roofline": ({
            "bound": "sfu (MUFU.EX2, one exp per pair-eval)",
            "achieved": pair_evals / (kern_ms / 1e3), "unit": "pair-evals/s",
            "peak": mufu_peak, "frac": pair_evals / (kern_ms / 1e3) / mufu_peak,
            "peak_source": "16 ex2/clk/SM measured x 148 SMs x sm_max_mhz",
            "note": "MUFU-only ceiling; a share of the exponentials comes from an FMA-pipe "
                    "polynomial (DESIGN.md section 3), so the kernel can pass 1.0",
            # every op the kernel issues to the XU (MUFU) pipe: the exponentials
            # left on MUFU plus lg2, sqrt, sin, cos of the Box-Muller noise (2 per
            # unit), each 8 cycles per warp-instruction per SM partition
            # (tools/mufu_ops_microbench.cu)
            "xu_ops_per_unit": xu_ops_per_unit,
            "xu_pipe_frac": units_per_launch * xu_ops_per_unit / (kern_ms / 1e3) / mufu_peak}
            if not joint and prec == capi.FP32 else {
            "bound": "fp64 pipe (the reference's fast_exp_nonpos + the weight sums, ~25 fp64 "
                     "ops per pair-eval; ncu: profiles/r02_ncu_full_cfg3_f64.md)",
            "achieved": pair_evals / (kern_ms / 1e3), "unit": "pair-evals/s",
            "peak": fp64_peak * 1e12 / 2.0 / 25.0,
            "frac": pair_evals / (kern_ms / 1e3) / (fp64_peak * 1e12 / 2.0 / 25.0),
            "peak_source": "64 fp64 ops/clk/SM x 148 x sm_max_mhz / 25 ops per pair-eval"}
            if not joint else {
            "bound": "fp64 pipe (Gram + weighted sum: 2 DFMA per pair-eval)",
            "achieved": 4.0 * pair_evals / (kern_ms / 1e3) / 1e12, "unit": "TFLOP/s",
            "peak": fp64_peak, "frac": 4.0 * pair_evals / (kern_ms / 1e3) / 1e12 / fp64_peak,
            "peak_source": "64 DFMA/clk/SM (tools/pipe_microbench: 59 measured) x 2 x 148 x sm_max_mhz"}),
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if (joint or prec == capi.FP64) else "f32",
        "data": "synthetic (N(0,1) forecast members and observations generated on the device)",
        "config": {"workload": desc + (" [joint-norm score extension]" if joint else ""),
                   "score": args.score, "d_per_gpu": d, "d_total": d_total, "members": m,
                   "pseudo_steps": s, "obs_stride": stride,
                   "obs_operator": "arctan" if arctan else "linear",
                   "l2": (f"L2 flushed (512 MB write) before each step, outside its timing; "
                          f"{n_sets} input sets of {set_bytes / 1e6:.0f} MB" if flush else
                          f"inputs larger than L2 ({n_sets} set(s) of {set_bytes / 1e6:.0f} MB "
                          f"forecast > 126 MB L2), steps timed back to back"),
                   "parallelism": f"state-dim shards x{world}"},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "path": "paper_2407_12168_b200.ensf_analyze(members, grid, y, out=...) "
                        "with pinned numpy in/out; chunked H2D/compute/D2H pipeline",
                "variants": variants},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if fp64 is not None:
        line["fp64_value"] = fp64["value"]
        line["fp64"] = fp64
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        xs, ys, idxs = make_inputs_host(_cpu_sample(d, m, args.ref_sample_d), m, stride, 0)
        cb = reference_rate(xs, ys, idxs, s, 3, 1, arctan=arctan)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), file=json_out, flush=True)
    if joint and world > 1:
        capi.comm_destroy(local)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
