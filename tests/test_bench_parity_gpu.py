"""The benchmark's own configuration, exactly as bench.py builds and times
it (fp32 force outputs, uint8 RGB, the captured step graph), checked against
the oracle on sampled frames -- the same check bench.py prints in its
``parity`` block -- and the per-frame digest table, which must not depend on
how the envs are sharded over ranks."""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2408_06506_b200 import synthetic  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(cfg, rank=0, world=1, envs=None):
    import dataclasses
    wl = synthetic.CONFIGS[cfg]
    if envs:
        wl = dataclasses.replace(wl, n_envs=envs)
    dev = torch.device("cuda", 0)
    c = bench.setup_workload(wl, rank, world, dev)
    c.arr.capture(c.depth, c.obj, c.sen)
    for _ in range(2):
        c.arr.replay()
    torch.cuda.synchronize()
    return c


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_bench_config_parity_as_measured(cfg):
    c = _run(cfg)
    if cfg == 3:
        assert c.arr.f_n.dtype == torch.float32 and c.arr.rgb_u8 is not None and c.E * c.S == 8192
    v = bench.validate(c, 1, 0, torch.device("cuda", 0), n_samples=24 if cfg != 5 else 12)
    p = v["parity"]
    assert p["ok"], p
    if c.wl.ff:
        assert p["contact_taxels"] > 0  # non-vacuous
    assert v["digest"]["frames"] == c.wl.frames


def test_digest_table_is_shard_invariant():
    """Two shards (world 2, built one after the other on this GPU) give the
    single-shard digest table when concatenated in env order."""
    from paper_2408_06506_b200.pipeline import frame_digests  # noqa: F401
    envs = 300  # 600 frames: > 2 x 148 per shard, the kernels' large-batch shape
    full = _run(3, envs=envs)
    names, d1 = full.arr.frame_digests()
    d1 = d1.cpu().numpy()
    del full
    parts = []
    for r in range(2):
        c = _run(3, rank=r, world=2, envs=envs)
        parts.append(c.arr.frame_digests()[1].cpu().numpy())
        del c
    np.testing.assert_array_equal(np.concatenate(parts), d1)
    # any changed byte changes its frame's digest and only that one
    c = _run(3, envs=4)
    base = c.arr.frame_digests()[1].clone()
    c.arr.rgb_u8[0, 1, 10, 10, 2] ^= 1
    after = c.arr.frame_digests()[1]
    assert after[1, 0] != base[1, 0]
    assert torch.equal(after[0], base[0]) and torch.equal(after[2:], base[2:])
