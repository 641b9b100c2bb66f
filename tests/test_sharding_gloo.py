"""N>1 host path on CPU (world_size 2, gloo): contiguous env shards with
global env ids in every RNG key reproduce the unsharded store bit-for-bit,
and the episode-statistics all-reduce (the only collective on the path)
equals the unsharded statistics. The oracle stands in for the device here;
the device side of the same contract is tests/test_parity_gpu.py::
test_env_offset_shard_equals_slice."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2108_13976_b200.sharding import shard_envs, weak_shard

CFG = dict(num_taggers=3, num_runners=17, obs_mode=O.PARTIAL, episode_length=20, seed=4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, steps, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        off, n = shard_envs(total, world, rank)
        cfg = O.make_config(**CFG)
        w = O.OracleWorld(cfg, n, env_offset=off)
        w.rollout(0, steps, cfg.seed)
        stats = torch.tensor(w.stats(), dtype=torch.float64)
        dist.all_reduce(stats)  # the episode-statistics all-reduce
        snap = w.snapshot()
        gathered = [None] * world
        dist.all_gather_object(gathered, (off, snap))
        if rank == 0:
            np.save(os.path.join(out_dir, "stats.npy"), stats.numpy())
            merged = {}
            for k in snap:
                parts = [g[1][k] for g in sorted(gathered, key=lambda g: g[0])]
                merged[k] = np.concatenate(parts, axis=0)
            np.savez(os.path.join(out_dir, "merged.npz"), **merged)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [24, 25])
def test_two_rank_shards_equal_unsharded(tmp_path, total):
    steps = 50
    mp.spawn(_worker, args=(2, _free_port(), total, steps, str(tmp_path)), nprocs=2, join=True)
    cfg = O.make_config(**CFG)
    whole = O.OracleWorld(cfg, total)
    whole.rollout(0, steps, cfg.seed)
    merged = dict(np.load(tmp_path / "merged.npz"))
    assert O.first_divergence(merged, whole.snapshot()) is None
    np.testing.assert_array_equal(np.load(tmp_path / "stats.npy")[:5], whole.stats()[:5])


def test_shard_arithmetic():
    assert shard_envs(10, 3, 0) == (0, 4)
    assert shard_envs(10, 3, 1) == (4, 3)
    assert shard_envs(10, 3, 2) == (7, 3)
    assert sum(shard_envs(16000, 8, r)[1] for r in range(8)) == 16000
    assert weak_shard(2000, 3) == (6000, 2000)
    with pytest.raises(ValueError):
        shard_envs(1, 2, 0)
