"""Multi-process sharding check (run under torchrun, one rank per GPU).

Each rank analyses its contiguous shard of a d-coordinate state with the joint
score; the library's NCCL communicator (turbda_comm_init) sums the per-step
N x N (+2N) distance partials - the one collective of the path.  Rank 0
gathers the shards and compares with the C oracle on the whole state, and
checks the componentwise mode reassembles bit-exactly with no collective.
With the communicator the componentwise shards also min-reduce their
divergence verdict (every rank raises the unsharded run's error) and
turbda_diag sums the rmse/spread partials over the shards.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/joint_multiproc_check.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import PortOracle, conditioned_inputs, rel_l2  # noqa: E402
from paper_2407_12168_b200 import capi  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    uid = [capi.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    capi.comm_init(local, rank, world, uid[0])

    m, d = 20, 6000
    x, y, _, _ = conditioned_inputs(m, d)
    x = 0.05 * x
    lo, hi = d * rank // world, d * (rank + 1) // world
    part_j = capi.analyze_host(x[:, lo:hi], y[lo:hi], 4.0, None, n_steps=20, joint=True,
                               device=local, k0=lo, d_total=d, precision=capi.FP64, sharded=True)
    part_c = capi.analyze_host(x[:, lo:hi], y[lo:hi], 4.0, None, n_steps=20, device=local,
                               k0=lo, d_total=d)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, part_j, part_c))
    if rank == 0:
        parts.sort(key=lambda t: t[0])
        got_j = np.concatenate([p[1] for p in parts], axis=1)
        got_c = np.concatenate([p[2] for p in parts], axis=1)
        port = PortOracle()
        want_j = port.analyze(x, y, 4.0, None, n_steps=20, joint=True)
        whole_c = capi.analyze_host(x, y, 4.0, None, n_steps=20, device=local)
        ej = rel_l2(got_j, want_j)
        print(f"joint sharded x{world} vs oracle rel-L2 {ej:.3e}; componentwise shards bitwise "
              f"{np.array_equal(got_c, whole_c)}", flush=True)
        ok = ej <= 1e-9 and np.array_equal(got_c, whole_c)
        print("JOINT_MULTIPROC_OK" if ok else "JOINT_MULTIPROC_FAIL", flush=True)
    # N > 64 (the W X GEMM + elementwise update path), sharded
    m2, d2 = 80, 3000
    x2, y2, _, _ = conditioned_inputs(m2, d2)
    x2 = 0.05 * x2
    lo2, hi2 = d2 * rank // world, d2 * (rank + 1) // world
    part_b = capi.analyze_host(x2[:, lo2:hi2], y2[lo2:hi2], 4.0, None, n_steps=20, joint=True,
                               device=local, k0=lo2, d_total=d2, precision=capi.FP64, sharded=True)
    parts_b = [None] * world
    dist.all_gather_object(parts_b, (lo2, part_b))
    if rank == 0:
        parts_b.sort(key=lambda t: t[0])
        got_b = np.concatenate([p[1] for p in parts_b], axis=1)
        eb = rel_l2(got_b, PortOracle().analyze(x2, y2, 4.0, None, n_steps=20, joint=True))
        print(f"joint N={m2} sharded x{world} vs oracle rel-L2 {eb:.3e}", flush=True)
        print("JOINT_BIG_MULTIPROC_OK" if eb <= 1e-9 else "JOINT_BIG_MULTIPROC_FAIL", flush=True)
    # divergence only inside the last rank's window: every rank must report
    # the unsharded run's (particle, step)
    r = np.ones(d)
    r[d * (world - 1) // world + 7] = 1e-9
    verdict = None
    try:
        capi.analyze_host(x[:, lo:hi], y[lo:hi], r[lo:hi], None, n_steps=20, device=local,
                          k0=lo, d_total=d, precision=capi.FP64, sharded=True)
    except capi.TurbdaError as e:
        verdict = (e.code, e.diverged_particle, e.diverged_step)
    verdicts = [None] * world
    dist.all_gather_object(verdicts, verdict)
    # rmse / spread partial sums over the shards
    truth = y
    sums = capi.diag(x[:, lo:hi], truth[lo:hi], device=local, sharded=True)
    if rank == 0:
        whole = None
        try:
            capi.analyze_host(x, y, r, None, n_steps=20, device=local, precision=capi.FP64)
        except capi.TurbdaError as e:
            whole = (e.code, e.diverged_particle, e.diverged_step)
        mean = x.mean(axis=0)
        want = (float(((mean - truth) ** 2).sum()), float(((x - mean) ** 2).sum()))
        ok_v = whole is not None and whole[0] == capi.DIVERGED and all(v == whole for v in verdicts)
        ok_d = all(abs(a - b) <= 1e-10 * abs(b) for a, b in zip(sums, want))
        print(f"verdicts {verdicts} whole {whole}; diag {sums} want {want}", flush=True)
        print("SHARD_VERDICT_OK" if ok_v and ok_d else "SHARD_VERDICT_FAIL", flush=True)
    # an empty window (fewer tiles than ranks): rank 0 holds the whole state,
    # the others none; the empty ranks must join every collective (the joint
    # per-step allreduce and the verdict min-reduce) instead of returning
    lo_e, hi_e = (0, d) if rank == 0 else (d, d)
    part_e = capi.analyze_host(x[:, lo_e:hi_e], y[lo_e:hi_e], 4.0, None, n_steps=20, joint=True,
                               device=local, k0=lo_e, d_total=d, precision=capi.FP64, sharded=True)
    r_e = np.ones(d)
    r_e[7] = 1e-9
    verdict_e = None
    try:
        capi.analyze_host(x[:, lo_e:hi_e], y[lo_e:hi_e], r_e[lo_e:hi_e], None, n_steps=20,
                          device=local, k0=lo_e, d_total=d, precision=capi.FP64, sharded=True)
    except capi.TurbdaError as e:
        verdict_e = (e.code, e.diverged_particle, e.diverged_step)
    verdicts_e = [None] * world
    dist.all_gather_object(verdicts_e, verdict_e)
    if rank == 0:
        ee = rel_l2(part_e, PortOracle().analyze(x, y, 4.0, None, n_steps=20, joint=True))
        ok_e = ee <= 1e-9 and verdicts_e[0] is not None and verdicts_e[0][0] == capi.DIVERGED \
            and all(v == verdicts_e[0] for v in verdicts_e)
        print(f"empty windows: joint rel-L2 {ee:.3e}, verdicts {verdicts_e}", flush=True)
        print("EMPTY_WINDOW_OK" if ok_e else "EMPTY_WINDOW_FAIL", flush=True)
    capi.comm_destroy(local)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
