"""GPU parity: the sm_100a Tag path (through the C ABI) against the CPU oracle
(oracle/tag_oracle.c, pinned to the reference by test_oracle_pinning.py) and
the reference-generated golden fixtures.

Bar (BASELINE.json north_star): discrete Tag is BIT-EXACT on every array at
every step (sampled actions, rewards, done, observations, positions, flags,
counters, reset timing, episode counters). Continuous Tag calls sin/cos whose
host (glibc sinf/cosf) and device results may differ by 1 ulp,
so it is checked teacher-forced with the tolerance CONT_ATOL below, integers
and flags exact."""
import json
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_2108_13976_b200 as W  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden as MG  # noqa: E402

CONT_ATOL = 1e-5  # |device - oracle| for f32 arrays, continuous teacher-forced step


def cfg_pair(**kw):
    """(device TagConfig, oracle config) with identical fields."""
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    return dc, oc


def dev_snapshot(ws, names):
    return {n: ws.store.pull(n) for n in names}


def to_dev(arr):
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).cuda()


def assert_same(dev, ora, where, cont=False):
    if not cont:
        d = O.first_divergence(dev, ora)
        assert d is None, f"{where}: first divergence {d}"
        return
    for n in ora:
        a, b = dev[n], ora[n]
        if a.dtype == np.float32:
            err = np.max(np.abs(a.astype(np.float64) - b.astype(np.float64))) if a.size else 0.0
            assert err <= CONT_ATOL, f"{where}: {n} max |err| {err}"
        else:
            np.testing.assert_array_equal(a, b, err_msg=f"{where}: {n}")


CONFIGS = {
    "disc_full_1x5": (dict(num_taggers=1, num_runners=4), 1),
    "disc_full_60x12": (dict(num_taggers=2, num_runners=10, episode_length=40, seed=3), 60),
    "disc_part_60x12": (dict(num_taggers=2, num_runners=10, obs_mode=O.PARTIAL, episode_length=40, seed=4), 60),
    "disc_part_7x100_k7": (dict(num_taggers=20, num_runners=80, obs_mode=O.PARTIAL, k_nearest=7,
                                grid_size=12, seed=5), 7),
    "disc_full_5x100": (dict(num_taggers=20, num_runners=80, grid_size=10, episode_length=30, seed=6), 5),
    "disc_part_3x1000": (dict(num_taggers=200, num_runners=800, obs_mode=O.PARTIAL, seed=42), 3),
    "disc_part_2x1100_g7": (dict(num_taggers=100, num_runners=1000, obs_mode=O.PARTIAL, k_nearest=12,
                                 grid_size=7, seed=8), 2),
    "disc_part_9x33_k20": (dict(num_taggers=3, num_runners=30, obs_mode=O.PARTIAL, k_nearest=20,
                                grid_size=50, seed=9), 9),
    # C3's A = 100 shape: brute-force K-NN (partial obs up to 128 agents)
    "disc_part_6x100": (dict(num_taggers=20, num_runners=80, obs_mode=O.PARTIAL, episode_length=50,
                             seed=10), 6),
    # brute-force K-NN at 150 agents (grid less than half occupied)
    "disc_part_4x150": (dict(num_taggers=30, num_runners=120, obs_mode=O.PARTIAL, episode_length=50,
                             seed=11), 4),
    # K=8 at 400 agents on lattice cells (generic MAXK=8 instantiation)
    "disc_part_2x400_k8": (dict(num_taggers=80, num_runners=320, obs_mode=O.PARTIAL, k_nearest=8,
                                episode_length=25, seed=15), 2),
    # K=1 on lattice cells (compile-time K=1)
    "disc_part_2x400_k1": (dict(num_taggers=80, num_runners=320, obs_mode=O.PARTIAL, k_nearest=1,
                                episode_length=25, seed=16), 2),
    # K=20 (obs rows of 83 floats, the cooperative wide-row writer) on lattice cells
    "disc_part_2x300_k20": (dict(num_taggers=60, num_runners=240, obs_mode=O.PARTIAL, k_nearest=20,
                                 episode_length=25, seed=14), 2),
    # 3000 agents on a 40 x 40 lattice (12 agent strides per thread, 1600 cells)
    "disc_part_2x3000_g40": (dict(num_taggers=600, num_runners=2400, obs_mode=O.PARTIAL, grid_size=40,
                                  episode_length=20, seed=13), 2),
    # 250 agents on a 30 x 30 grid: ring search over 15 x 15 bucket cells
    "disc_part_3x250_ring": (dict(num_taggers=50, num_runners=200, obs_mode=O.PARTIAL, grid_size=30,
                                  episode_length=50, seed=12), 3),
}
CONT_CONFIGS = {
    "cont_full_20x12": (dict(variant=O.CONTINUOUS, num_taggers=2, num_runners=10, episode_length=40,
                             world_length=8.0, seed=3), 20),
    "cont_part_20x12": (dict(variant=O.CONTINUOUS, num_taggers=2, num_runners=10, obs_mode=O.PARTIAL,
                             episode_length=40, world_length=8.0, seed=4), 20),
    "cont_part_3x300": (dict(variant=O.CONTINUOUS, num_taggers=60, num_runners=240, obs_mode=O.PARTIAL,
                             world_length=12.0, tag_radius=0.6, seed=5), 3),
    "cont_part_5x100": (dict(variant=O.CONTINUOUS, num_taggers=20, num_runners=80, obs_mode=O.PARTIAL,
                             world_length=10.0, tag_radius=0.5, seed=6), 5),
}


@pytest.mark.parametrize("name", list(CONFIGS) + list(CONT_CONFIGS))
def test_registration_matches_oracle(name):
    kw, envs = {**CONFIGS, **CONT_CONFIGS}[name]
    dc, oc = cfg_pair(**kw)
    ws = W.Workspace(dc, envs)
    o = O.OracleWorld(oc, envs)
    assert_same(dev_snapshot(ws, o.layout), o.snapshot(), "registration", cont=dc.variant == W.CONTINUOUS)
    ws.close()


@pytest.mark.parametrize("logits", [False, True])
@pytest.mark.parametrize("name", list(CONFIGS))
def test_unfused_lockstep_discrete(name, logits):
    """check_consistency_single (harness.cpp:563-633): sample -> run_step ->
    compare (before reset) -> reset, every step, bit-exact."""
    kw, envs = CONFIGS[name]
    dc, oc = cfg_pair(**kw)
    ws = W.Workspace(dc, envs)
    o = O.OracleWorld(oc, envs)
    A, C, V = dc.num_agents(), dc.action_categories(), dc.action_choices()
    rng = np.random.default_rng(7)
    steps = 60 if dc.num_agents() < 500 else 25
    for t in range(steps):
        lg = rng.normal(0, 2, (envs, A, C, V)) if logits else np.zeros((envs, A, C, V))
        W.sample_actions(ws.store, to_dev(lg), lg.size, C, V, t, oc.seed)
        o.sample(t, oc.seed, lg)
        ws.engine.run_step(ws.plan, ws.store, t)
        o.step(t)
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"step {t}")
        ids = ws.resets.detect_done()
        assert ids == [e for e in range(envs) if o.view("done")[e]]
        ws.resets.auto_reset(ids)
        o.reset_done()
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"reset {t}")
        for e in ids:
            assert ws.resets.episodes_started(e) == o.episodes(e)
    ws.close()


@pytest.mark.parametrize("name", list(CONFIGS))
def test_fused_rollout_matches_oracle(name):
    """RolloutDriver::step (harness.cpp:478-490) as ONE fused kernel per step
    (sample -> step -> stats -> reset-on-done): bit-exact every step, and the
    device EpisodeTracker stats equal the oracle's."""
    kw, envs = CONFIGS[name]
    dc, oc = cfg_pair(**kw)
    ws = W.Workspace(dc, envs)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, envs)
    steps = 80 if dc.num_agents() < 500 else 30
    for t in range(steps):
        drv.step()
        o.rollout(t, 1, oc.seed)
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"fused step {t}")
    drv.check()
    np.testing.assert_array_equal(drv.stats()[:5], o.stats()[:5])
    for e in range(envs):
        assert ws.resets.episodes_started(e) == o.episodes(e)
    ws.close()


def test_fused_equals_unfused_driver():
    dc, oc = cfg_pair(num_taggers=4, num_runners=20, obs_mode=O.PARTIAL, episode_length=25, seed=21)
    ws1, ws2 = W.Workspace(dc, 40), W.Workspace(dc, 40)
    d1 = W.RolloutDriver(ws1.store, ws1.plan, ws1.resets, 5)
    d2 = W.RolloutDriver(ws2.store, ws2.plan, ws2.resets, 5)
    d2.set_fused(False)
    names = O.array_layout(oc, 40).keys()
    for t in range(60):
        d1.step()
        d2.step()
        assert O.first_divergence(dev_snapshot(ws1, names), dev_snapshot(ws2, names)) is None, t
    ws1.close()
    ws2.close()


@pytest.mark.parametrize("name", list(CONT_CONFIGS))
def test_continuous_teacher_forced(name):
    """Continuous Tag: before every step the oracle's state is pushed to the
    device, then one sample+step (+reset) is compared: f32 within CONT_ATOL,
    actions/flags/counters/done exact."""
    kw, envs = CONT_CONFIGS[name]
    dc, oc = cfg_pair(**kw)
    ws = W.Workspace(dc, envs)
    o = O.OracleWorld(oc, envs)
    A = dc.num_agents()
    rng = np.random.default_rng(3)
    state = ["loc_x", "loc_y", "speed", "direction", "active", "step_count", "is_tagger"]
    for t in range(50):
        for n in state:
            ws.store.push(n, o.pull(n))
        lg = rng.normal(0, 1.5, (envs, A, 2, 3))
        W.sample_actions(ws.store, to_dev(lg), lg.size, 2, 3, t, oc.seed)
        o.sample(t, oc.seed, lg)
        ws.engine.run_step(ws.plan, ws.store, t)
        o.step(t)
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"cont step {t}", cont=True)
        ids = ws.resets.detect_done()
        ws.resets.auto_reset(ids)
        o.reset_done()
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"cont reset {t}", cont=True)
    ws.close()


GOLDEN = sorted(f for f in os.listdir(os.path.join(HERE, "golden")) if f.endswith(".npz"))


@pytest.mark.parametrize("fname", GOLDEN)
def test_golden_fixture_on_device(fname):
    """Replays a fixture generated by the reference itself (make_golden.py):
    the device must reproduce the reference's per-step digests (FNV-1a over
    every array, after the step and after the reset) exactly — discrete and
    continuous (the device replays the reference host's glibc sinf/cosf
    bit-for-bit, §8f row 4) — and its final arrays and episode counters."""
    g = np.load(os.path.join(HERE, "golden", fname))
    name = fname[:-4]
    spec = MG.CONFIGS[name]
    dc, oc = cfg_pair(**spec["cfg"])
    envs = spec["envs"]
    ws = W.Workspace(dc, envs)
    names = list(O.array_layout(oc, envs).keys())
    cont = dc.variant == W.CONTINUOUS
    init = {n: g["init_" + n] for n in names}
    assert_same(dev_snapshot(ws, names), init, "init")
    A, C, V = dc.num_agents(), dc.action_categories(), dc.action_choices()
    step_dig = json.loads(str(g["step_digest"]))
    reset_dig = json.loads(str(g["reset_digest"]))
    for t in range(spec["steps"]):
        lg = MG.logits_for(name, oc, envs, t) if spec.get("logits") else np.zeros((envs, A, C, V))
        W.sample_actions(ws.store, to_dev(lg), lg.size, C, V, t, oc.seed)
        ws.engine.run_step(ws.plan, ws.store, t)
        assert MG.digest(dev_snapshot(ws, names)) == step_dig[t], f"{'cont ' if cont else ''}step {t}"
        ws.resets.auto_reset(ws.resets.detect_done())
        assert MG.digest(dev_snapshot(ws, names)) == reset_dig[t], f"{'cont ' if cont else ''}reset {t}"
    final = {n: g["final_" + n] for n in names}
    assert_same(dev_snapshot(ws, names), final, "final")
    assert [ws.resets.episodes_started(e) for e in range(envs)] == list(g["episodes"])
    ws.close()


def test_headline_shape_sampled_envs_bit_exact():
    """C2 (2000 envs x 1000 agents, 200 taggers, partial K=5) at full size on
    the device; a sample of envs is re-run by the oracle with the same GLOBAL
    env ids (keys use global ids, so a 2-env oracle world at env_offset=e
    reproduces env e) and must match bit-for-bit after 20 fused steps."""
    dc, oc = cfg_pair(num_taggers=200, num_runners=800, obs_mode=O.PARTIAL, k_nearest=5, seed=0)
    E = 2000
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    drv.run(20)
    drv.check()
    layout = O.array_layout(oc, 2)
    for e0 in (0, 777, 1998):
        o = O.OracleWorld(oc, 2, env_offset=e0)
        o.rollout(0, 20, oc.seed)
        dev = {n: ws.store.pull(n, e0, 2) for n in layout}
        assert_same(dev, o.snapshot(), f"env {e0}")
    # size-independent invariants over all 2000 envs
    x, y = ws.store.pull("loc_x"), ws.store.pull("loc_y")
    assert x.min() >= 0 and x.max() <= 19 and np.all(x == np.round(x))
    assert y.min() >= 0 and y.max() <= 19 and np.all(y == np.round(y))
    assert np.all(ws.store.pull("active")[:, :200] == 1)  # taggers never deactivate
    st = drv.stats()
    assert st[W.STAT_ENV_STEPS] == 20 * E
    ws.close()


def test_env_offset_shard_equals_slice():
    """Sharding contract: a store at env_offset=k reproduces
    envs [k, k+n) of the unsharded store bit-for-bit."""
    dc, _ = cfg_pair(num_taggers=3, num_runners=17, obs_mode=O.PARTIAL, episode_length=15, seed=12)
    big = W.Workspace(dc, 30)
    part = W.Workspace(dc, 10, env_offset=10)
    d1 = W.RolloutDriver(big.store, big.plan, big.resets, 1)
    d2 = W.RolloutDriver(part.store, part.plan, part.resets, 1)
    d1.run(40)
    d2.run(40)
    for n in big.store.array_names():
        np.testing.assert_array_equal(big.store.pull(n, 10, 10), part.store.pull(n), err_msg=n)
    big.close()
    part.close()


# ---- DataStore semantics ------------------------------------
def test_datastore_registration_rules():
    s = W.DataStore(2, 3)
    s.register_array(W.ArraySpec("loc_x", [2, 3], W.REAL32, True), np.zeros(6))
    np.testing.assert_array_equal(s.pull("loc_x"), np.zeros((2, 3), np.float32))
    with pytest.raises(W.WarpError) as ei:
        s.register_array(W.ArraySpec("loc_x", [2, 3]))
    assert ei.value.code == W.DUPLICATE_NAME
    with pytest.raises(W.WarpError) as ei:
        s.register_array(W.ArraySpec("bad", [2, 3]), np.zeros(5))
    assert ei.value.code == W.SHAPE_MISMATCH
    with pytest.raises(W.WarpError) as ei:
        s.register_array(W.ArraySpec("bad", [3, 3]))
    assert ei.value.code == W.SHAPE_MISMATCH
    with pytest.raises(W.WarpError) as ei:
        s.lock()
    assert ei.value.code == W.MISSING_PLACEHOLDER
    for n, sh, k in [("observations", [2, 3, 4], W.REAL32), ("sampled_actions", [2, 3, 1], W.INT32),
                     ("rewards", [2, 3], W.REAL32), ("done", [2], W.BOOL8)]:
        s.register_array(W.ArraySpec(n, sh, k))
    s.lock()
    assert s.locked()
    with pytest.raises(W.WarpError) as ei:
        s.register_array(W.ArraySpec("late", [2, 3]))
    assert ei.value.code == W.STORE_LOCKED
    with pytest.raises(W.WarpError) as ei:
        s.handle("nope")
    assert ei.value.code == W.UNKNOWN_NAME
    inf = s.info("observations")
    assert (inf.env_stride, inf.agent_stride, inf.has_agent_axis) == (12, 4, True)
    # env-slice write visible, others unchanged
    s.push("loc_x", np.array([[7, 7, 7]], np.float32), env_begin=1)
    np.testing.assert_array_equal(s.pull("loc_x"), [[0, 0, 0], [7, 7, 7]])
    with pytest.raises(W.WarpError) as ei:
        s.pull("loc_x", 2, 1)
    assert ei.value.code == W.INDEX_OUT_OF_RANGE
    # restore_snapshot isolation + idempotence
    s.push("loc_x", np.array([[1, 2, 3]], np.float32), env_begin=0)
    s.restore_snapshot([1])
    np.testing.assert_array_equal(s.pull("loc_x"), [[1, 2, 3], [0, 0, 0]])
    s.restore_snapshot([])
    s.restore_snapshot([0, 1])
    s.restore_snapshot([0, 1])
    np.testing.assert_array_equal(s.pull("loc_x"), np.zeros((2, 3)))
    with pytest.raises(W.WarpError) as ei:
        s.restore_snapshot([2])
    assert ei.value.code == W.INDEX_OUT_OF_RANGE
    s.close()


# ---- sampler ---------------------------------------------
def _sampler_store(E, A, C=1):
    s = W.DataStore(E, A)
    s.register_array(W.ArraySpec("sampled_actions", [E, A, C], W.INT32))
    return s


def test_sampler_distribution_and_errors():
    E, A = 1000, 1000
    s = _sampler_store(E, A)
    p = np.array([0.5, 0.3, 0.2])
    lg = np.broadcast_to(np.log(p), (E, A, 1, 3)).copy()
    W.sample_actions(s, to_dev(lg), lg.size, 1, 3, 0, 123)
    a = s.pull("sampled_actions").ravel()
    f = np.bincount(a, minlength=3) / a.size
    chi2 = a.size * np.sum((f - p) ** 2 / p)
    assert chi2 < 9.21  # p > 0.01 at 2 dof
    # bit-exact vs the oracle sampler on a random subset
    o_cfg = O.make_config(num_taggers=1, num_runners=A - 1)
    lib = O.oracle_lib()
    stream = lib.oracle_substream(123, 0x616374696f6e7331)
    import ctypes as Cc
    for e, ag in [(0, 0), (5, 17), (999, 999), (512, 3)]:
        u = lib.oracle_uniform(stream, 0, e, ag, 0, 0)
        row = (Cc.c_double * 3)(*lg[e, ag, 0])
        assert lib.oracle_sample_from_logits(row, 3, u) == a[e * A + ag]
    # near-deterministic row
    lg2 = np.zeros((E, A, 1, 5))
    lg2[..., 0] = 1000.0
    s2 = _sampler_store(E, A)
    W.sample_actions(s2, to_dev(lg2), lg2.size, 1, 5, 3, 9)
    assert np.all(s2.pull("sampled_actions") == 0)
    # uniform-5 frequencies in [0.198, 0.202] at 1e6 draws
    W.sample_actions(s2, to_dev(np.zeros_like(lg2)), lg2.size, 1, 5, 4, 9)
    f5 = np.bincount(s2.pull("sampled_actions").ravel(), minlength=5) / (E * A)
    assert np.all((f5 > 0.198) & (f5 < 0.202))
    # non-finite -> WD_ERR_NON_FINITE, actions untouched (sampler.cpp:23-25)
    before = s2.pull("sampled_actions")
    bad = np.zeros_like(lg2)
    bad[10, 20, 0, 3] = np.nan
    with pytest.raises(W.WarpError) as ei:
        W.sample_actions(s2, to_dev(bad), bad.size, 1, 5, 5, 9)
    assert ei.value.code == W.NON_FINITE
    np.testing.assert_array_equal(s2.pull("sampled_actions"), before)
    with pytest.raises(W.WarpError) as ei:
        W.sample_actions(s2, to_dev(lg2), lg2.size - 1, 1, 5, 5, 9)
    assert ei.value.code == W.SHAPE_MISMATCH
    s.close()
    s2.close()


def test_fused_nonfinite_logits_sticky_error():
    dc, _ = cfg_pair(num_taggers=2, num_runners=10)
    ws = W.Workspace(dc, 8)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
    bad = np.zeros((8, 12, 1, 5))
    bad[3, 4, 0, 1] = np.inf
    t = to_dev(bad)
    drv.set_logits(t, bad.size)
    drv.step()
    with pytest.raises(W.WarpError) as ei:
        drv.check()
    assert ei.value.code == W.NON_FINITE
    ws.close()


# ---- resets ----------------------------------------------
def test_reset_isolation_and_rerandomization():
    dc, oc = cfg_pair(num_taggers=2, num_runners=10, obs_mode=O.PARTIAL, seed=5)
    ws = W.Workspace(dc, 2)
    names = list(O.array_layout(oc, 2).keys())
    drv = W.RolloutDriver(ws.store, ws.plan, None, 0)  # no auto reset
    drv.run(3)
    before = dev_snapshot(ws, names)
    ws.resets.auto_reset([0])
    after = dev_snapshot(ws, names)
    for n in names:  # env 1 untouched
        np.testing.assert_array_equal(after[n][1], before[n][1], err_msg=n)
    assert ws.resets.episodes_started(0) == 1 and ws.resets.episodes_started(1) == 0
    assert ws.resets.detect_done() == []
    x1 = ws.store.pull("loc_x")[0].copy()
    ws.resets.auto_reset([0])
    assert not np.array_equal(ws.store.pull("loc_x")[0], x1)  # episode 2 differs
    o = O.OracleWorld(oc, 2)
    o.rollout(0, 3, 0)
    # oracle with tracking only differs in stats; reset env 0 twice
    o.reset_ids([0])
    o.reset_ids([0])
    np.testing.assert_array_equal(ws.store.pull("observations")[0], o.pull("observations")[0])
    with pytest.raises(W.WarpError) as ei:
        ws.resets.auto_reset([5])
    assert ei.value.code == W.INDEX_OUT_OF_RANGE
    ws.close()


def test_reset_manager_policy_validation():
    dc, _ = cfg_pair()
    ws = W.Workspace(dc, 2)
    with pytest.raises(W.WarpError) as ei:
        W.ResetManager(ws.store, W.ResetPolicy(True, ["loc_x"], None))
    assert ei.value.code == W.INVALID_ARGUMENT
    with pytest.raises(W.WarpError) as ei:
        W.ResetManager(ws.store, W.ResetPolicy(True, ["nope"], None))
    assert ei.value.code == W.UNKNOWN_NAME
    ws.close()


@pytest.mark.parametrize("name", ["disc_full_60x12", "disc_part_60x12", "disc_part_7x100_k7",
                                  "disc_part_3x1000", "disc_part_9x33_k20", "disc_part_3x250_ring"]
                         + list(CONT_CONFIGS))
def test_device_tag_reference_twin_matches_oracle(name):
    """The device TagReference twin (twin_kernels.cu, the check's independent
    second implementation) against the oracle: unfused sample -> run_step ->
    auto_reset, bit-exact on every array (continuous too: same libm replica)."""
    kw, envs = {**CONFIGS, **CONT_CONFIGS}[name]
    if name in CONT_CONFIGS and not O.libm_matches_replica():
        pytest.skip("host libm is not the glibc FMA variant the device replicates")
    dc, oc = cfg_pair(**{**kw, "episode_length": min(kw.get("episode_length", 500), 20)})
    ws = W.Workspace(dc, envs, reference=True)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, envs)
    assert_same(dev_snapshot(ws, o.layout), o.snapshot(), "twin registration")
    rng = np.random.default_rng(2)
    A, C, V = dc.num_agents(), dc.action_categories(), dc.action_choices()
    steps = 30 if A < 500 else 8
    for t in range(steps):
        lg = rng.normal(0, 2, (envs, A, C, V))
        d_lg = to_dev(lg)
        drv.set_logits(d_lg, lg.size)
        drv.step()
        o.rollout(t, 1, oc.seed, lg)
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"twin step {t}")
    for e in range(envs):
        assert ws.resets.episodes_started(e) == o.episodes(e)
    ws.close()


def test_fault_injection_detected_in_rewards():
    """Mutation test of the parity harness: with the device
    fault hook set, the first divergence must be in rewards."""
    dc, oc = cfg_pair(num_taggers=2, num_runners=10, obs_mode=O.PARTIAL, seed=1)
    W.set_fault_tag_radius_bias(1.0)
    try:
        ws = W.Workspace(dc, 60)
        o = O.OracleWorld(oc, 60)
        first = None
        for t in range(100):
            W.sample_actions(ws.store, to_dev(np.zeros((60, 12, 1, 5))), 60 * 12 * 5, 1, 5, t, oc.seed)
            o.sample(t, oc.seed)
            ws.engine.run_step(ws.plan, ws.store, t)
            o.step(t)
            first = O.first_divergence(dev_snapshot(ws, o.layout), o.snapshot())
            if first:
                break
            ws.resets.auto_reset(ws.resets.detect_done())
            o.reset_done()
        assert first is not None and first[0] == "rewards"
        ws.close()
    finally:
        W.set_fault_tag_radius_bias(0.0)


@pytest.mark.parametrize("kw,envs,steps", [
    # k_nearest > 32 (the shared-memory kernels keep top-K lists in registers)
    (dict(num_taggers=10, num_runners=40, obs_mode=O.PARTIAL, k_nearest=40, episode_length=6, seed=3), 3, 10),
    (dict(variant=O.CONTINUOUS, num_taggers=8, num_runners=40, obs_mode=O.PARTIAL, k_nearest=33,
          episode_length=6, world_length=6.0, tag_radius=0.8, seed=4), 2, 8),
    # more than 227 KB of shared memory per env
    (dict(num_taggers=2400, num_runners=9600, obs_mode=O.PARTIAL, episode_length=3, seed=5), 1, 4),
])
def test_large_shapes_run_on_the_global_memory_path(kw, envs, steps):
    """Shapes the shared-memory kernels cannot take (k_nearest > 32, more
    than 65535 agents, more than 227 KB of shared memory per env) run on the
    global-memory kernels (the TagReference twin's code) instead of failing;
    the reference only requires k < agents (tag_env.cpp:36-39). Bit-exact
    against the oracle through the fused-looking driver (unfused underneath)."""
    if kw.get("variant") == O.CONTINUOUS and not O.libm_matches_replica():
        pytest.skip("host libm is not the glibc FMA variant the device replicates")
    dc, oc = cfg_pair(**kw)
    ws = W.Workspace(dc, envs)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, envs)
    assert_same(dev_snapshot(ws, o.layout), o.snapshot(), "registration")
    for t in range(steps):
        drv.step()
        o.rollout(t, 1, oc.seed)
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"step {t}")
    drv.check()
    for e in range(envs):
        assert ws.resets.episodes_started(e) == o.episodes(e)
    ws.close()


def test_cpp_facade_example(tmp_path):
    """The header-only C++ facade (include/warp_b200.hpp) drives the same
    fused rollout from C++ (reference-side integration path)."""
    import subprocess
    from test_abi import build_cpp_example
    exe = build_cpp_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "env_steps=640" in r.stdout


@pytest.mark.parametrize("multistep", [-1, 0])
@pytest.mark.parametrize("kw,envs", [(dict(num_taggers=1, num_runners=4), 300),
                                     (dict(num_taggers=1, num_runners=4), 6000),
                                     (dict(num_taggers=20, num_runners=80, obs_mode=O.PARTIAL,
                                           grid_size=10, episode_length=15), 37)])
def test_graph_replay_equals_direct_launches(kw, envs, multistep):
    """RolloutDriver::run replays a captured CUDA graph of fused launches whose
    step index is read on device; it must equal step-by-step launches and the
    oracle bit-for-bit, across window boundaries (53 = 3 x 16 + 5), then
    continue with direct steps. multistep=0 forces the graph path on the C4
    shapes (plain PDL edges between the nodes at 300 envs, none at 6000)."""
    dc, oc = cfg_pair(**kw)
    W.set_tuning("multistep", multistep)
    try:
        ws1, ws2 = W.Workspace(dc, envs), W.Workspace(dc, envs)
        d1 = W.RolloutDriver(ws1.store, ws1.plan, ws1.resets, 9)
        d2 = W.RolloutDriver(ws2.store, ws2.plan, ws2.resets, 9)
        d2.set_graphs(False)
        d1.run(53)
        d1.step()
        d1.run(32)
        for _ in range(86):
            d2.step()
        assert d1.next_step() == d2.next_step() == 86
        names = O.array_layout(oc, envs).keys()
        assert O.first_divergence(dev_snapshot(ws1, names), dev_snapshot(ws2, names)) is None
        if envs <= 300:
            o = O.OracleWorld(oc, envs)
            o.rollout(0, 86, 9)
            assert_same(dev_snapshot(ws1, names), o.snapshot(), "graph replay")
            np.testing.assert_array_equal(d1.stats()[:5], o.stats()[:5])
        d1.check()
        ws1.close()
        ws2.close()
    finally:
        W.set_tuning("multistep", -1)


@pytest.mark.parametrize("kw,envs", [
    (dict(num_taggers=3, num_runners=20, obs_mode=O.PARTIAL, seed=31), 9),    # packed brute K-NN
    (dict(num_taggers=20, num_runners=80, obs_mode=O.PARTIAL, seed=32), 4),   # one-env brute
    (dict(num_taggers=40, num_runners=160, obs_mode=O.PARTIAL, seed=33), 3),  # lattice cells
    (dict(num_taggers=20, num_runners=80, seed=34), 4),                        # full obs, grid resolve
    (dict(num_taggers=60, num_runners=240, obs_mode=O.PARTIAL, k_nearest=20, seed=35), 2),  # wide rows
])
def test_off_lattice_state_falls_back_exactly(kw, envs):
    """Pushed state outside what placement produces — half-integer positions
    in some envs, a tagger flag moved off the [0, T) prefix — must disable the
    integral fast paths (32-bit-key K-NN, lattice cells, prefix resolve) for
    exactly those steps and stay bit-exact with the oracle."""
    dc, oc = cfg_pair(**kw)
    ws = W.Workspace(dc, envs)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, envs)
    A = dc.num_agents()
    x = o.pull("loc_x").reshape(envs, A)
    x[0, ::3] += 0.5
    o.push("loc_x", x)
    ws.store.push("loc_x", x)
    tg = o.pull("is_tagger").reshape(envs, A)
    tg[envs - 1, A - 1] = 1  # a tagger outside the prefix
    o.push("is_tagger", tg)
    ws.store.push("is_tagger", tg)
    for t in range(12):
        drv.step()
        o.rollout(t, 1, oc.seed)
        assert_same(dev_snapshot(ws, o.layout), o.snapshot(), f"off-lattice step {t}")
    ws.close()


@pytest.mark.parametrize("kw,envs", [
    (dict(num_taggers=200, num_runners=800, obs_mode=O.PARTIAL, episode_length=30, seed=41), 1500),
    (dict(num_taggers=1, num_runners=4, episode_length=9, seed=42), 5000),
    (dict(num_taggers=40, num_runners=160, obs_mode=O.PARTIAL, episode_length=20, seed=44), 2000),
    (dict(num_taggers=20, num_runners=80, episode_length=15, seed=45), 1000),
    (dict(variant=O.CONTINUOUS, num_taggers=20, num_runners=80, obs_mode=O.PARTIAL, episode_length=12,
          seed=43), 1200),
])
@pytest.mark.parametrize("pdl_mode", ["1", "2", "3"])  # per-env waits, released at entry / exit; plain PDL
def test_overlapped_steps_equal_serial_steps(kw, envs, pdl_mode):
    """RolloutDriver::step launches consecutive fused steps with programmatic
    dependent launch: a CTA of step t+1 starts once its own envs finished step
    t, inside step t's tail. 100 back-to-back steps (no host sync, resets
    included, several waves of CTAs) must equal the same steps launched one
    after another without overlap (set_overlap(False))."""
    dc, oc = cfg_pair(**kw)
    W.set_tuning("pdl_mode", int(pdl_mode))  # overlap even where the plan would not choose it
    try:
        ws1 = W.Workspace(dc, envs)
        d1 = W.RolloutDriver(ws1.store, ws1.plan, ws1.resets, 5)
        ws2 = W.Workspace(dc, envs)
        d2 = W.RolloutDriver(ws2.store, ws2.plan, ws2.resets, 5)
        d2.set_overlap(False)
        for _ in range(100):
            d1.step()
        d1.run(100)  # graph replays / multi-step windows, overlapped
        for _ in range(100):
            d2.step()
        d2.run(100)
    finally:
        W.set_tuning("reset")
    names = list(O.array_layout(oc, envs).keys())
    d = O.first_divergence(dev_snapshot(ws1, names), dev_snapshot(ws2, names))
    assert d is None, f"overlapped vs serial steps: first divergence {d}"
    np.testing.assert_array_equal(d1.stats(), d2.stats())
    ws1.close()
    ws2.close()


def test_spec_tag_examples_device():
    """SPEC.md:245-267 known answers (lowest-index credit among same-cell
    taggers, +2 for two simultaneous credits, -1 for a tagged runner, zero
    observations once inactive) on the device step, and equal to the oracle."""
    from test_oracle_pinning import check_spec_tag_scene, spec_tag_scene
    oc, x, y = spec_tag_scene()
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    ws = W.Workspace(dc, 1)
    o = O.OracleWorld(oc, 1)
    for name, arr in (("loc_x", x), ("loc_y", y), ("sampled_actions", np.zeros((1, 5, 1), np.int32))):
        ws.store.push(name, arr)
        o.push(name, arr)
    ws.engine.run_step(ws.plan, ws.store, 0)
    o.step(0)
    check_spec_tag_scene(ws.store.pull)
    assert_same(dev_snapshot(ws, o.layout), o.snapshot(), "SPEC tag scene")
    ws.close()


def test_spec_continuous_tie_device():
    """Continuous equidistant taggers: the lower index is credited (min over
    (d^2, index)), on the device step, equal to the oracle."""
    from test_oracle_pinning import check_spec_continuous_tie, spec_continuous_tie_scene
    oc, state = spec_continuous_tie_scene()
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    ws = W.Workspace(dc, 1)
    o = O.OracleWorld(oc, 1)
    for n, v in state.items():
        ws.store.push(n, v)
        o.push(n, v)
    ws.engine.run_step(ws.plan, ws.store, 0)
    o.step(0)
    check_spec_continuous_tie(ws.store.pull)
    assert_same(dev_snapshot(ws, o.layout), o.snapshot(), "continuous tie scene", cont=True)
    ws.close()


@pytest.mark.parametrize("cont", [False, True])
def test_fused_sampler_near_boundary_rows_bit_exact(cont):
    """The fused sampler decides on f32 ex2.approx estimates and falls back to
    the reference f64 arithmetic when the target lies within 1e-5 x total of a
    cumulative sum (tag_kernels.cu sample_fast). Logits built from each row's
    own uniform u put the target at relative distances +-1e-9 .. +-1e-3 from
    the first boundary, so both paths run; the whole store after the step must
    equal the oracle's (sampler.cpp:5-40 on the same logits). (Targets within a
    few ulp of a boundary are the documented f64 exp deviation, DESIGN §4:
    CUDA's and glibc's exp may round differently there.)"""
    E = 40
    dc, oc = cfg_pair(num_taggers=10, num_runners=40, obs_mode=O.PARTIAL, k_nearest=5, seed=3,
                      variant=O.CONTINUOUS if cont else O.DISCRETE, episode_length=50)
    A = oc.num_taggers + oc.num_runners
    C, V = (2, 3) if cont else (1, 5)
    lib = O.oracle_lib()
    stream = lib.oracle_substream(oc.seed, 0x616374696f6e7331)
    deltas = [1e-9, -1e-9, 1e-7, -1e-7, 1e-6, -1e-6, 3e-5, -3e-5, 1e-3, -1e-3]
    lg = np.zeros((E, A, C, V))
    close = 0
    for e in range(E):
        for a in range(A):
            for c in range(C):
                u = lib.oracle_uniform(stream, 0, e, a, c, 0)
                d = deltas[(e * A + a + c) % len(deltas)]
                close += abs(d) < 1e-5
                p0 = min(max(u + d, 1e-12), 1.0 - 1e-12)
                lg[e, a, c, 0] = np.log(p0)
                lg[e, a, c, 1:] = np.log((1.0 - p0) / (V - 1))
    assert close > E * A * C // 2
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    drv.set_logits(to_dev(lg), lg.size)
    drv.step()
    o = O.OracleWorld(oc, E)
    o.rollout(0, 1, oc.seed, lg)
    d = O.first_divergence({n: ws.store.pull(n) for n in o.layout}, o.snapshot())
    assert d is None, f"first divergence {d}"
    drv.check()
    ws.close()


@pytest.mark.parametrize("keys", [0, 1])
@pytest.mark.parametrize("ties", [False, True])
@pytest.mark.parametrize("kw,envs,grid", [
    (dict(num_taggers=2, num_runners=10, world_length=8.0, seed=4), 20, False),
    # bucket grid forced on small envs: 1 x 1 and 3 x 3 cells, so the 3 x 3
    # block scan clamps at every border
    (dict(num_taggers=2, num_runners=10, world_length=8.0, seed=4), 20, True),
    (dict(num_taggers=8, num_runners=32, world_length=6.0, tag_radius=0.7, seed=8), 6, True),
    (dict(num_taggers=60, num_runners=240, world_length=12.0, tag_radius=0.6, seed=5), 3, False),
    (dict(num_taggers=120, num_runners=480, world_length=20.0, tag_radius=0.5, seed=7), 2, False),
])
def test_continuous_keyed_ring_search_bit_exact(kw, envs, grid, ties, keys):
    """Continuous partial K-NN with the keyed ring search forced on or off
    (tuning key cont_keys; the plan enables it on every grid plan): fused
    steps bit-exact vs the oracle. ties=True pushes integral positions first,
    so equal d2 abound and the keyed search must hand those agents to the
    exact one (neighbor_grid.hpp:62-111 order: (d2, index)). Both searches
    start with the flattened 3 x 3 block scan (scan_block3)."""
    dc, oc = cfg_pair(variant=O.CONTINUOUS, obs_mode=O.PARTIAL, k_nearest=5, episode_length=30, **kw)
    W.set_tuning("cont_keys", keys)
    if grid:
        W.set_tuning("brute_max", 1)
    try:
        ws = W.Workspace(dc, envs)
        o = O.OracleWorld(oc, envs)
        if ties:
            for n in ("loc_x", "loc_y"):
                v = np.floor(o.pull(n))
                o.push(n, v)
                ws.store.push(n, v)
        A = dc.num_agents()
        lg = np.random.default_rng(11).normal(0, 1.5, (envs, A, 2, 3))
        drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
        drv.set_logits(to_dev(lg), lg.size)
        for t in range(12):
            drv.step()
            o.rollout(t, 1, oc.seed, lg)
            d = O.first_divergence({n: ws.store.pull(n) for n in o.layout}, o.snapshot())
            assert d is None, f"step {t}: first divergence {d}"
        if grid:
            assert ws.plan.geometry()["uses_grid"] == 1
        drv.check()
        ws.close()
    finally:
        W.set_tuning("cont_keys", -1)
        W.set_tuning("brute_max", -1)
