#!/usr/bin/env python
"""EnSF analysis throughput on B200 (BASELINE.json metric: d x N x steps / s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config cfg2|cfg1|cfg3|cfg4|cfg5] [--precision fp32|fp64]
                    [--obs linear|arctan]

One "step" is one full EnSF analysis (turbda::analyze: every pseudo-time
step of the reverse SDE + relax_spread) of one synthetic forecast ensemble.
Default workload: BASELINE config 2 (d = 131,072 coordinates per GPU, N = 64
members, S = 100 pseudo-time steps, every-4th-point observations).  With
--gpus N (torchrun, one rank per GPU) every rank analyses its own
131,072-coordinate shard of a d = 131,072 N state: weak scaling, no
data-path collective (the componentwise score never couples coordinates);
the barrier and the max-over-ranks of the device time are the only
collectives.

Rank 0 prints ONE JSON line (keys per the driver contract).  The
``cpu_baseline`` leg and ``--impl reference`` time the reference's own CPU
implementation (oracle/_ref: proj/src/ensf.cpp compiled unmodified) on this
host's cores over a bounded coordinate sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
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
    "cfg3": (16777216, 20, 100, 1, "BASELINE cfg3: d=16.8M (2048x2048x4), N=20, S=100"),
    "cfg4": (1048576, 512, 100, 1, "BASELINE cfg4: d=1M, N=512, S=100"),
    "cfg5": (2097152, 128, 100, 4, "BASELINE cfg5 analysis: d=2.1M (1024x1024x2), N=128, S=100, "
                                   "every-4th-point arctan obs"),
}
# algorithmic bytes per unit for a per-step-streaming fp32
# design (read z, read x, write z) - the HBM roofline the north star names.
BYTES_PER_UNIT = 12
MUFU_PER_CLK_PER_SM = 16  # ex2 throughput, measured (tools/pipe_microbench.cu)


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


def make_inputs(d, m, stride, k0, seed=1234):
    """Synthetic SQG-shaped forecast: N(0,1) members and observations (the
    throughput generator of SURVEY.md 8(d), drawn with numpy here)."""
    rng = np.random.default_rng(seed + k0)
    x = rng.standard_normal((m, d))
    if stride <= 1:
        idx = None
        y = rng.standard_normal(d)
    else:
        first = (-k0) % stride  # global indices 0, s, 2s, ... that fall in this shard
        idx = np.arange(k0 + first, k0 + d, stride, dtype=np.int64)
        y = rng.standard_normal(idx.size)
    return x, y, idx


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
    return {"value": units * steps / total, "unit": UNIT, "cores": min(cores, m),
            "threads_requested": cores, "kind": kind,
            "sample": f"{m} members x {d} coordinates x {n_steps} pseudo-steps "
                      f"(a {d}-coordinate slice of the workload), {steps} run(s), "
                      f"median {statistics.median(times):.3f} s",
            "ms_per_step": 1e3 * total / steps}


def run_reference_arm(args, cfg, json_out=None):
    """--impl reference: rank 0 times the reference's CPU implementation."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    d_full, m, s, stride, desc = CONFIGS[cfg]
    d_sample = _cpu_sample(d_full, m, args.ref_sample_d)
    x, y, idx = make_inputs(d_sample, m, stride, 0)
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
    print(json.dumps(line), file=json_out or sys.stdout, flush=True)


def _cpu_sample(d, m, base):
    """CPU sample width: `base` coordinates at N = 64, scaled by (64/N)^2 (the
    CPU cost grows with N^2 per coordinate) so every config's CPU leg takes
    seconds, a multiple of 64 coordinates."""
    return max(64, min(d, int(base * (64.0 / m) ** 2) // 64 * 64))


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


def main():
    json_out = _json_stdout()
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--score", choices=["componentwise", "joint"], default="componentwise",
                    help="joint: the north-star joint-norm extension (fp64, one NCCL allreduce "
                         "of the N x N distances per pseudo-step across ranks)")
    ap.add_argument("--obs", choices=["linear", "arctan"], default=None,
                    help="observation operator (default: arctan for cfg5, linear otherwise)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-d", type=int, default=32768)
    ap.add_argument("--ref-sample-d", type=int, default=8192)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    if args.impl == "reference":
        run_reference_arm(args, args.config, json_out)
        return

    import torch
    import torch.distributed as dist

    from paper_2407_12168_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    d, m, s, stride, desc = CONFIGS[args.config]
    d_total = d * world
    k0 = rank * d
    joint = args.score == "joint"
    arctan = _arctan(args)
    # joint mode: distances/update in fp64 always; --precision picks the noise
    prec = capi.FP32 if args.precision == "fp32" else capi.FP64
    if joint and world > 1:
        uid = [capi.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        capi.comm_init(local, rank, world, uid[0])

    # --- resident inputs: 3 rotating sets so the working set exceeds L2 ----
    n_sets = 3
    host_sets = [make_inputs(d, m, stride, k0, seed=1234 + 7 * q) for q in range(n_sets)]
    dsets = []
    for x, y, idx in host_sets:
        tx = torch.from_numpy(x).to(dev)
        ty = torch.from_numpy(y).to(dev)
        tr = torch.ones_like(ty)
        ti = None if idx is None else torch.from_numpy(idx).to(dev)
        dsets.append((tx, ty, tr, ti))
    out = torch.empty((m, d), dtype=torch.float64, device=dev)
    obs_dim = host_sets[0][1].size
    p = capi.params(d_total=d_total, k0=k0, d_local=d, obs_dim=obs_dim, n_members=m, n_steps=s,
                    obs_kind=(0 if stride <= 1 else 1) + (2 if arctan else 0),
                    precision=prec, device=local,
                    flags=capi.INPUTS_ON_DEVICE | capi.ASYNC,
                    score_mode=capi.SCORE_JOINT if joint else capi.SCORE_COMPONENTWISE)
    stream = torch.cuda.Stream(dev)  # a real stream: the events and kernels share it
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream

    def one(q):
        tx, ty, tr, ti = dsets[q % n_sets]
        capi.analyze(p, tx, ty, tr, ti, out, stream=sh)

    for q in range(args.warmup):
        one(q)
    torch.cuda.synchronize(dev)
    capi.check(local, p)  # divergence verdict of the warm-up runs

    # --- timed region: K device-resident analyses ---------------------------
    # Inputs larger than L2 (3 rotating sets): the K steps are timed back to
    # back.  Smaller workloads: L2 is flushed (a 512 MB write) before every
    # step, outside that step's event pair, and the per-step times are summed.
    l2_bytes = 126 * 2**20
    set_bytes = n_sets * m * d * 8
    # between two uses of one input set the other sets stream through L2
    flush = (n_sets - 1) * m * d * 8 <= l2_bytes
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

    # --- end to end through the public API with pinned host buffers ---------
    import paper_2407_12168_b200 as tb
    grid = tb.GridSpec()
    # any (nx, ny, nz=2) whose size is d: the API only checks the size
    grid.nz = 2
    grid.nx = 256 if d % 512 == 0 else d // 2
    grid.ny = d // (2 * grid.nx)
    x0, y0, _ = host_sets[0]
    hx = torch.from_numpy(x0).pin_memory().numpy()
    hy_full = torch.from_numpy(np.ascontiguousarray(y0)).pin_memory().numpy()
    hout = torch.empty((m, d), dtype=torch.float64).pin_memory().numpy()
    e2e_times = []
    if world > 1:
        dist.barrier()
    for q in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if joint and world > 1:
            # a window of the sharded state: the C-ABI with host buffers
            pe = capi.params(d_total=d_total, k0=k0, d_local=d, obs_dim=obs_dim, n_members=m,
                             n_steps=s, obs_kind=(0 if stride <= 1 else 1) + (2 if arctan else 0),
                             precision=prec, device=local, cycle=1 + q,
                             score_mode=capi.SCORE_JOINT)
            capi.analyze(pe, hx, hy_full, np.ones_like(hy_full), host_sets[0][2], hout)
            res = hout
        else:
            res = tb.ensf_analyze(hx, grid, hy_full, r=1.0, seed=7, cycle=1 + q, n_steps=s,
                                  thinning=stride if stride > 1 else 0,
                                  precision=args.precision, device=local,
                                  obs_operator="arctan" if arctan else "linear",
                                  score_mode=args.score, out=hout)
        if q >= args.warmup:
            e2e_times.append(time.perf_counter() - t0)
    e2e_s = torch.tensor([sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = units_per_gpu * world / float(e2e_s[0])
    if stride > 1 and k0 != 0:
        pass  # the e2e leg analyses each rank's shard as its own state (same cost)
    if joint and world > 1:
        h2d = x0.nbytes + y0.nbytes * (3 if stride > 1 else 2)  # x, y, r (+ idx)
    else:
        h2d = x0.nbytes + y0.nbytes * (2 if stride > 1 else 1) + 8  # x, y (+ idx), one r
    d2h = res.nbytes + 8

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
            traffic = json.loads(tf.read_text()).get(f"{args.config}_{args.precision}")
        except ValueError:
            traffic = None
    pair_evals = units_per_launch * m
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
            "note": "MUFU-only ceiling; for N > 24 (sorted member tiles, up to ~200 members) one "
                    "pair-eval slot in eight takes its exponential from an FMA-pipe polynomial, "
                    "so that kernel's own MUFU-bound ceiling is 8/7 of this peak"} if not joint else {
            "bound": "fp64 pipe (Gram + weighted sum: 2 DFMA per pair-eval)",
            "achieved": 4.0 * pair_evals / (kern_ms / 1e3) / 1e12, "unit": "TFLOP/s",
            "peak": fp64_peak, "frac": 4.0 * pair_evals / (kern_ms / 1e3) / 1e12 / fp64_peak,
            "peak_source": "64 DFMA/clk/SM (tools/pipe_microbench: 59 measured) x 2 x 148 x sm_max_mhz"}),
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if (joint or prec == capi.FP64) else "f32",
        "data": "synthetic",
        "config": {"workload": desc + (" [joint-norm score extension]" if joint else ""),
                   "score": args.score, "d_per_gpu": d, "d_total": d_total, "members": m,
                   "pseudo_steps": s, "obs_stride": stride,
                   "obs_operator": "arctan" if arctan else "linear",
                   "l2": (f"L2 flushed (512 MB write) before each step, outside its timing; "
                          f"inputs {set_bytes / 1e6:.0f} MB" if flush else
                          f"{n_sets} rotating resident input sets ({set_bytes / 1e6:.0f} MB; "
                          f"{(n_sets - 1) * m * d * 8 / 1e6:.0f} MB > 126 MB L2 pass between "
                          f"reuses), steps timed back to back"),
                   "parallelism": f"state-dim shards x{world}"},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "path": "paper_2407_12168_b200.ensf_analyze(members, grid, y, out=...) "
                        "with pinned numpy in/out; chunked H2D/compute/D2H pipeline"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        xs, ys, idxs = make_inputs(_cpu_sample(d, m, args.cpu_sample_d), m, stride, 0)
        cb = reference_rate(xs, ys, idxs, s, 1, 0, arctan=arctan)
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
