"""Oracle parity at every BASELINE.json config point, on the exact launch
paths bench.py and the sweeps time:

- C2 / C3: 2000 envs x A in {10, 100, 500, 1000} agents, T = llround(A/5)
  taggers (bench_agents, harness.cpp:823-832), partial K=5 — the benchmark
  config itself (episode 500) and a short-episode twin (resets inside the
  window). 20 back-to-back RolloutDriver::step calls (overlapped launches,
  no host sync: the bench path), then 10 steps checked one by one; sampled
  GLOBAL env ids are re-run by the oracle (keys use global ids).
- C3 secondary: full observations at A in {500, 1000} (the cooperative
  wide-row writer, 16 MB of obs per env-step), 2 envs, every step.
- C4: 1+4 agents, full obs, E in {1, 10000}, every step, single-step launches
  and run() windows (multi-step residency).
- The sweep's continuous partial points (A in {100, 200, 1000}, 2000 envs) on
  the same protocol as C3.
Discrete Tag: bit-exact on every array."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_2108_13976_b200 as W  # noqa: E402

pytestmark = pytest.mark.gpu


def cfg_pair(**kw):
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    return dc, oc


def envs_equal(ws, o, e0, n, where):
    layout = O.array_layout(o.cfg, n)
    dev = {name: ws.store.pull(name, e0, n) for name in layout}
    d = O.first_divergence(dev, o.snapshot())
    assert d is None, f"{where}: env {e0}: first divergence {d}"


@pytest.mark.parametrize("episode", [500, 6])
@pytest.mark.parametrize("A", [10, 100, 500, 600, 1000])  # 600: the 160-thread lattice CTA
def test_c3_partial_2000_envs_bench_path(A, episode):
    T = int(np.floor(A / 5 + 0.5))
    dc, oc = cfg_pair(num_taggers=T, num_runners=A - T, obs_mode=O.PARTIAL, k_nearest=5,
                      episode_length=episode, seed=0)
    E = 2000
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    picks = (0, 591, 592, 1337, 1999)  # wave borders of 148 x 4 CTAs included
    worlds = {e: O.OracleWorld(oc, 1, env_offset=e) for e in picks}
    for _ in range(20):
        drv.step()  # overlapped launches, no host sync in between
    for e, o in worlds.items():
        o.rollout(0, 20, oc.seed)
        envs_equal(ws, o, e, 1, "after 20 back-to-back steps")
    for t in range(20, 30):
        drv.step()
        for e, o in worlds.items():
            o.rollout(t, 1, oc.seed)
            envs_equal(ws, o, e, 1, f"step {t}")
    drv.check()
    st = drv.stats()
    assert st[W.STAT_ENV_STEPS] == 30 * E
    if episode == 6:
        assert st[W.STAT_EPISODES] >= E  # every env finished an episode
    for e, o in worlds.items():
        assert ws.resets.episodes_started(e) == o.episodes(0)
    ws.close()


@pytest.mark.parametrize("episode", [500, 6])
@pytest.mark.parametrize("A", [100, 200, 1000])
def test_continuous_partial_2000_envs_bench_path(A, episode):
    """The sweep's continuous partial points on their launch path: A = 100
    (brute force, 32-bit keys), 200 and 1000 (bucket grid, flattened 3 x 3
    block scan with paired keys; LEAN at 1000). Same protocol as the C3 test:
    20 back-to-back steps, then 10 checked one by one, sampled global env ids
    re-run by the oracle, bit-exact on every array."""
    T = int(np.floor(A / 5 + 0.5))
    dc, oc = cfg_pair(variant=O.CONTINUOUS, num_taggers=T, num_runners=A - T, obs_mode=O.PARTIAL,
                      k_nearest=5, episode_length=episode, seed=0)
    E = 2000
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    picks = (0, 443, 444, 1337, 1999)  # wave borders of 148 x 3 CTAs included
    worlds = {e: O.OracleWorld(oc, 1, env_offset=e) for e in picks}
    for _ in range(20):
        drv.step()
    for e, o in worlds.items():
        o.rollout(0, 20, oc.seed)
        envs_equal(ws, o, e, 1, "after 20 back-to-back steps")
    for t in range(20, 30):
        drv.step()
        for e, o in worlds.items():
            o.rollout(t, 1, oc.seed)
            envs_equal(ws, o, e, 1, f"step {t}")
    drv.check()
    assert drv.stats()[W.STAT_ENV_STEPS] == 30 * E
    for e, o in worlds.items():
        assert ws.resets.episodes_started(e) == o.episodes(0)
    ws.close()


@pytest.mark.parametrize("A", [500, 1000])
def test_c3_full_obs_large_agents(A):
    T = A // 5
    dc, oc = cfg_pair(num_taggers=T, num_runners=A - T, obs_mode=O.FULL, episode_length=7, seed=2)
    E = 2
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, E)
    for t in range(12):
        drv.step()
        o.rollout(t, 1, oc.seed)
        envs_equal(ws, o, 0, E, f"full obs A={A} step {t}")
    drv.run(8)
    o.rollout(12, 8, oc.seed)
    envs_equal(ws, o, 0, E, f"full obs A={A} after run(8)")
    drv.check()
    np.testing.assert_array_equal(drv.stats()[:5], o.stats()[:5])
    ws.close()


@pytest.mark.parametrize("E", [1, 10000])
def test_c4_env_sweep_end_points(E):
    dc, oc = cfg_pair(num_taggers=1, num_runners=4, obs_mode=O.FULL, episode_length=9, grid_size=5, seed=3)
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, E)
    for t in range(25):
        drv.step()
        o.rollout(t, 1, oc.seed)
        envs_equal(ws, o, 0, E, f"C4 E={E} step {t}")
    drv.run(70)  # multi-step residency windows (64 + 6) / graph replays
    o.rollout(25, 70, oc.seed)
    envs_equal(ws, o, 0, E, f"C4 E={E} after run(70)")
    drv.check()
    np.testing.assert_array_equal(drv.stats()[:5], o.stats()[:5])
    assert drv.stats()[W.STAT_EPISODES] > 0
    ws.close()
