"""World-size-2 sharding on CPU (gloo): each rank takes its contiguous env
shard (no collective on the data path), computes its sensor frames, and only
validation crosses ranks (all_gather of per-shard digests), exactly as
bench.py does over NCCL.  The per-rank compute here is the CPU oracle -- this
test covers the sharding / gather host logic, not the kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import sdf_tuple
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import synthetic
from paper_2408_06506_b200.pipeline import shard_range

E, S = 5, 2


def _inputs():
    _, cam, bg, lut, pts = synthetic.sensor_setup((80, 60), (10, 14))
    sdf = synthetic.peg_grid((16, 16, 32))
    depth = synthetic.depth_batch(cam, bg, E * S, config_id=77).reshape(E, S, 60, 80)
    obj, sen = synthetic.peg_states(E, S, config_id=77)
    return lut, pts, sdf, depth, obj, sen


def _frames(lo, hi):
    lut, pts, sdf, depth, obj, sen = _inputs()
    d = depth[lo:hi].reshape(-1, 60, 80)
    objE = np.repeat(obj[lo:hi], S, axis=0)
    senE = sen[lo:hi].reshape(-1, 13)
    rgb, f_n, f_t, force, torque = O.sensor_frames(d, lut.coeffs, lut.degree, pts.points, sdf_tuple(sdf), objE,
                                                   senE, (1000.0, 100.0, 10.0, 2.0))
    return np.array([rgb.sum(dtype=np.float64), np.abs(f_n).sum(), np.abs(f_t).sum(), hi - lo], dtype=np.float64)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(E, rank, world)
    digest = torch.from_numpy(_frames(lo, hi))
    gathered = [torch.zeros(4, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, digest)
    if rank == 0:
        out.put(torch.stack(gathered).numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_two_rank_shards_cover_all_envs():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    full = _frames(0, E)
    assert parts[:, 3].sum() == E
    np.testing.assert_allclose(parts[:, :3].sum(axis=0), full[:3], rtol=1e-12)


# ---- bench.py's own shard / gather functions (the code the NCCL run uses)

def _bench_worker(rank, world, port, out):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    frames, S = 37, 1
    lo, hi = shard_range(frames, rank, world)
    # stand-in per-frame outputs: frame g's rows are a function of g only
    g = torch.arange(lo, hi, dtype=torch.float64)
    f_n = (g[:, None, None, None] * 1000 + torch.arange(24, dtype=torch.float64).view(1, 2, 4, 3)).float()
    rgb = (g[:, None, None, None].to(torch.int64) * 7 + torch.arange(30).view(1, 2, 5, 3)).remainder(256).to(
        torch.uint8)
    idx = bench.sample_indices(frames, 9)
    owned = [(r, int(x) - lo) for r, x in enumerate(idx) if lo <= x < hi]
    got = bench.gather_rows([("rgb", rgb), ("f_n", f_n)], owned, len(idx), world, torch.device("cpu"))
    dig = torch.stack([g.to(torch.int64) * 3 + 1, g.to(torch.int64) ** 2], dim=1)
    table = bench.gather_digests(dig, hi - lo, world, torch.device("cpu"))
    if rank == 0:
        out.put((idx, got["rgb"], got["f_n"], table))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_bench_gather_reassembles_global_frames():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    idx, rgb, f_n, table = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    g = idx.astype(np.float64)
    np.testing.assert_array_equal(
        f_n, (g[:, None, None, None] * 1000 + np.arange(24).reshape(1, 2, 4, 3)).astype(np.float32))
    np.testing.assert_array_equal(
        rgb, ((idx[:, None, None, None] * 7 + np.arange(30).reshape(1, 2, 5, 3)) % 256).astype(np.uint8))
    a = np.arange(37)
    np.testing.assert_array_equal(table, np.stack([a * 3 + 1, a ** 2], axis=1))


def test_sample_indices_cover_shard_boundaries():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench
    idx = bench.sample_indices(8192, 16)
    assert len(idx) >= 16 and idx[0] == 0 and idx[-1] == 8191
    for n in (2, 4, 8):
        for r in range(1, n):
            b = r * 8192 // n
            assert b in idx and b - 1 in idx
    assert list(bench.sample_indices(1, 16)) == [0]
