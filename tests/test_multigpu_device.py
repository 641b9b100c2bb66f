"""N>1 path with the PRODUCT library, on one B200:

- two processes (gloo for the host plumbing), each owning a contiguous env
  shard with global env ids, stepping the fused device path; the shards
  concatenate to a single-process store of all envs bit-for-bit, and the
  device-reduced statistics summed over the ranks equal the unsharded ones;
- the library's NCCL entry point (wdg_stats_allreduce) executes a real
  ncclAllReduce (a world-1 communicator: this pool's boxes have one GPU, and
  NCCL refuses two ranks on one device);
- bench.py under torchrun with 2 ranks (--same-device) times the all-reduce
  inside its window and reports it."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle as O  # noqa: E402
import paper_2108_13976_b200 as W  # noqa: E402
from paper_2108_13976_b200.sharding import shard_envs  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KW = dict(num_taggers=20, num_runners=80, obs_mode=O.PARTIAL, episode_length=14, seed=21)
STEPS = 60


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dc():
    oc = O.make_config(**KW)
    return W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_}), oc


def _worker(rank, world, port, total, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        off, n = shard_envs(total, world, rank)
        dc, oc = _dc()
        ws = W.Workspace(dc, n, env_offset=off)
        drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, KW["seed"])
        drv.run(STEPS // 2)
        for _ in range(STEPS - STEPS // 2):
            drv.step()
        st = torch.zeros(8, dtype=torch.float64, device="cuda")
        drv.reduce_stats_into(st)
        host = st.cpu()
        dist.all_reduce(host)  # the statistics all-reduce over the ranks
        snap = {name: ws.store.pull(name) for name in O.array_layout(oc, n)}
        gathered = [None] * world
        dist.all_gather_object(gathered, (off, snap))
        if rank == 0:
            np.save(os.path.join(out_dir, "stats.npy"), host.numpy())
            merged = {k: np.concatenate([g[1][k] for g in sorted(gathered, key=lambda g: g[0])], axis=0)
                      for k in snap}
            np.savez(os.path.join(out_dir, "merged.npz"), **merged)
        ws.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [40, 41])
def test_two_process_device_shards_equal_single_store(tmp_path, total):
    mp.spawn(_worker, args=(2, _free_port(), total, str(tmp_path)), nprocs=2, join=True)
    dc, oc = _dc()
    ws = W.Workspace(dc, total)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, KW["seed"])
    for _ in range(STEPS):
        drv.step()
    merged = dict(np.load(tmp_path / "merged.npz"))
    whole = {name: ws.store.pull(name) for name in merged}
    assert O.first_divergence(merged, whole) is None
    np.testing.assert_array_equal(np.load(tmp_path / "stats.npy"), drv.stats())
    ws.close()


def test_stats_allreduce_through_nccl_entry_point():
    assert W.nccl_version() >= 21800
    dc, _ = _dc()
    ws = W.Workspace(dc, 30)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, KW["seed"])
    drv.run(40)
    comm = W.Comm(1, 0, W.comm_unique_id())
    assert (comm.world, comm.rank) == (1, 0)
    out = torch.full((8,), -1.0, dtype=torch.float64, device="cuda")
    comm.stats_allreduce(drv, out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), drv.stats())
    assert out[0].item() > 0  # episodes ended inside the window
    comm.close()
    with pytest.raises(ValueError):
        W.Comm(1, 0, b"short")
    ws.close()


def test_torchrun_two_ranks_bench_times_the_allreduce():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--same-device", "--steps", "20", "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["envs_total"] == 4000
    assert line["collective"]["allreduces_timed"] >= 1
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    # all-reduced statistics cover both shards' env-steps
    assert line["episode_stats"]["env_steps"] >= 2 * 2000 * 23
