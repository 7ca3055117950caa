"""CPU, world size 2 over gloo: the state-dimension sharding used by
``bench.py --gpus N`` / ``device_count > 1``.  Each rank analyses its own
coordinate window with the C oracle (noise keyed by the global coordinate);
the gathered windows must equal the unsharded analysis bit for bit, and no
collective other than the gather is needed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_bounds(d, world, rank, align=64):
    tiles = (d + align - 1) // align
    lo = min(d, tiles * rank // world * align)
    hi = min(d, tiles * (rank + 1) // world * align)
    return lo, hi


def _worker(rank, world, port, result):
    import sys
    sys.path.insert(0, str(ROOT))
    from oracle.oracle import PortOracle, throughput_inputs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_o = PortOracle()
    d, m = 1000, 12
    x, y, idx = throughput_inputs(m, d, oracle=port_o, stride=3)
    lo, hi = _shard_bounds(d, world, rank)
    sel = (idx >= lo) & (idx < hi)
    part = port_o.analyze(x[:, lo:hi], y[sel], 0.8, idx[sel], n_steps=15, k0=lo, d_total=d,
                          workers=2)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, part))
    if rank == 0:
        whole = port_o.analyze(x, y, 0.8, idx, n_steps=15, workers=2)
        got = np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0])], axis=1)
        result.put(bool(np.array_equal(got, whole)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shards_reassemble_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_shard_bounds_cover_state():
    for d in (1, 63, 64, 1000, 131072):
        for world in (1, 2, 3, 8):
            b = [_shard_bounds(d, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == d
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


def test_bench_shard_observation_indices():
    """bench.py's per-rank observation indices are the global every-s-th
    points that fall into the rank's window."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import torch
    d, stride = 1000, 4
    for k0 in (0, 1000, 2000, 3000, 1001, 2003):
        want = np.arange(k0, k0 + d)[np.arange(k0, k0 + d) % stride == 0]
        _, y, idx = bench.make_inputs_host(d, 2, stride, k0)
        assert np.array_equal(idx, want) and y.size == want.size
        _, ty, _, tidx = bench.make_inputs_device(torch, torch.device("cpu"), d, 2, stride, k0, 1)
        assert np.array_equal(tidx.numpy(), want) and ty.numel() == want.size
    _, _, idx = bench.make_inputs_host(d, 2, 1, 0)
    assert idx is None


def test_bench_refuses_mismatched_world(tmp_path):
    """bench.py prints no line when WORLD_SIZE differs from --gpus."""
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2"], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 2 and out.stdout.strip() == ""
    assert "refusing" in out.stderr


def _joint_worker(rank, world, port, result):
    """Joint-norm score (north_star extension) sharded by coordinates: per
    pseudo-step each rank forms the N x N partial squared distances over its
    window, ONE all_reduce(sum) makes them global, and the softmax, weighted
    prior sum, likelihood and Euler-Maruyama update stay local - the data
    flow of csrc/joint_kernels.cu + the NCCL allreduce, restated in numpy
    after oracle/ensf_oracle.c (orc_analyze, joint = 1)."""
    import sys
    sys.path.insert(0, str(ROOT))
    from oracle.oracle import PortOracle, throughput_inputs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    po = PortOracle()
    d, m, n_steps, seed, cycle, eps, r = 1000, 12, 15, 7, 1, 0.01, 0.8
    x, y, idx = throughput_inputs(m, d, oracle=po, stride=3)
    lo, hi = _shard_bounds(d, world, rank)
    xl = x[:, lo:hi]
    sel = (idx >= lo) & (idx < hi)
    il, yl = idx[sel] - lo, y[sel]
    fexp = np.vectorize(po.fast_exp_nonpos)
    ent = [(cycle << 32) | i for i in range(m)]
    z = np.stack([po.stream_normals(seed, 6, ent[i], hi - lo, lo) for i in range(m)])
    dt = (1.0 - eps) / n_steps
    for s in range(n_steps):
        t = max(1.0 - s * dt - dt, eps)
        alpha, beta2 = 1.0 - t, t
        b, s2, damp = -1.0 / (1.0 - t), 1.0 + 2.0 * t / (1.0 - t), 1.0 - t
        diff = z[:, None, :] - alpha * xl[None, :, :]
        part = torch.from_numpy(np.einsum("ijk,ijk->ij", diff, diff))
        dist.all_reduce(part)  # the one collective of the step
        dd = part.numpy()
        w = fexp((dd.min(axis=1, keepdims=True) - dd) / (2.0 * beta2))
        num = w @ xl
        sc = -(z - alpha * num / w.sum(axis=1, keepdims=True)) / beta2
        np.add.at(sc, (slice(None), il), damp * (yl - z[:, il]) / r)
        xi = np.stack([po.stream_normals(seed, 6, ent[i], hi - lo, (s + 1) * d + lo)
                       for i in range(m)])
        z = z + (-(b * z - s2 * sc) * dt + np.sqrt(s2 * dt) * xi)
    part_out = po.relax_spread(z, xl, 1.0)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, part_out))
    if rank == 0:
        whole = po.analyze(x, y, r, idx, n_steps=n_steps, joint=True, workers=2)
        got = np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0])], axis=1)
        err = float(np.linalg.norm(got - whole) / np.linalg.norm(whole))
        result.put(err)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_joint_mode_one_allreduce_per_step():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_joint_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert err < 1e-9, err
