"""Bit-exact continuous trig row.

The reference moves continuous agents with std::cos / std::sin on float
(move_continuous, proj/include/warp/tag_env.hpp:86-100) and caches them for the
observations (fill_sincos, proj/src/tag_env.cpp:214-221): glibc 2.39 sinf /
cosf, which on x86-64 dispatch to an FMA build. The device replicates that
build step for step (tag_kernels.cu sincosf_ref); the C replica in
oracle/tag_oracle.c follows the same steps and is checked here against the
host libm. With it, continuous Tag is bit-exact end to end (GPU test)."""
import numpy as np
import pytest

import oracle as O
import paper_2108_13976_b200 as W


def test_replica_matches_host_libm_dense():
    """Every 13th float bit pattern in [-2pi, 2pi] (167 M values x 2 functions)."""
    bad = O.oracle_lib().oracle_trig_mismatches(0.0, 6.2831855, 13)
    if bad and not O.libm_matches_replica():
        pytest.skip("host libm is not the glibc FMA variant the replica follows")
    assert bad == 0


def test_replica_small_and_boundary_values():
    lib = O.oracle_lib()
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.sinf.restype = libm.cosf.restype = ctypes.c_float
    libm.sinf.argtypes = libm.cosf.argtypes = [ctypes.c_float]
    if not O.libm_matches_replica():
        pytest.skip("host libm is not the glibc FMA variant the replica follows")
    vals = [0.0, -0.0, 1e-30, 2.4e-4, 0.78539815, 0.7853982, 1.5707964, 3.1415927, 4.712389,
            6.2831855, 119.99999, 120.0, 1e5, -3.0]
    for v in vals:
        assert np.float32(lib.oracle_sinf_replica(v)).tobytes() == np.float32(libm.sinf(v)).tobytes(), v
        assert np.float32(lib.oracle_cosf_replica(v)).tobytes() == np.float32(libm.cosf(v)).tobytes(), v


CONT = {
    "cont_full_20x12": (dict(variant=O.CONTINUOUS, num_taggers=2, num_runners=10, episode_length=40,
                             world_length=8.0, seed=3), 20),
    "cont_part_20x12": (dict(variant=O.CONTINUOUS, num_taggers=2, num_runners=10, obs_mode=O.PARTIAL,
                             episode_length=40, world_length=8.0, seed=4), 20),
    "cont_part_3x300": (dict(variant=O.CONTINUOUS, num_taggers=60, num_runners=240, obs_mode=O.PARTIAL,
                             world_length=12.0, tag_radius=0.6, seed=5), 3),
    # brute-force K-NN: two envs per CTA, and one env per CTA with idle lanes
    "cont_part_5x100": (dict(variant=O.CONTINUOUS, num_taggers=20, num_runners=80, obs_mode=O.PARTIAL,
                             episode_length=30, world_length=10.0, tag_radius=0.5, seed=6), 5),
    "cont_part_2x200": (dict(variant=O.CONTINUOUS, num_taggers=40, num_runners=160, obs_mode=O.PARTIAL,
                             episode_length=30, world_length=14.0, tag_radius=0.5, seed=7), 2),
    # runtime K (non-exact instantiations): K=3 brute-force, K=12 ring search (MAXK 32)
    "cont_part_9x30_k3": (dict(variant=O.CONTINUOUS, num_taggers=6, num_runners=24, obs_mode=O.PARTIAL,
                               k_nearest=3, episode_length=35, world_length=6.0, seed=8), 9),
    "cont_part_2x300_k8": (dict(variant=O.CONTINUOUS, num_taggers=60, num_runners=240, obs_mode=O.PARTIAL,
                                k_nearest=8, episode_length=30, world_length=14.0, tag_radius=0.6,
                                seed=10), 2),
    "cont_part_2x400_k12": (dict(variant=O.CONTINUOUS, num_taggers=80, num_runners=320, obs_mode=O.PARTIAL,
                                 k_nearest=12, episode_length=30, world_length=16.0, tag_radius=0.6,
                                 seed=9), 2),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CONT))
def test_continuous_free_running_bit_exact(name):
    """Continuous Tag, fused rollout with random logits, free-running (no
    state pushed back): every array bit-exact against the oracle at every
    step, resets included."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not O.libm_matches_replica():
        pytest.skip("host libm is not the glibc FMA variant the device replicates")
    kw, envs = CONT[name]
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    ws = W.Workspace(dc, envs)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, envs)
    A = dc.num_agents()
    rng = np.random.default_rng(11)
    lg = rng.normal(0, 1.5, (envs, A, 2, 3))
    dlg = torch.from_numpy(lg).cuda()  # must outlive the rollout's use of it
    drv.set_logits(dlg, lg.size)
    for t in range(100):
        drv.step()
        o.rollout(t, 1, oc.seed, lg.reshape(-1))
        d = O.first_divergence({n: ws.store.pull(n) for n in o.layout}, o.snapshot())
        assert d is None, f"{name} step {t}: first divergence {d}"
    drv.check()
    ws.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cont_full_20x12", "cont_part_5x100", "cont_part_2x200", "cont_part_3x300"])
def test_continuous_multistep_equals_single_steps(name):
    """RolloutDriver::run keeps up to 64 steps resident in one launch; with
    resets inside the window it must equal one launch per step bit-for-bit."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    kw, envs = CONT[name]
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    ws1, ws2 = W.Workspace(dc, envs), W.Workspace(dc, envs)
    d1 = W.RolloutDriver(ws1.store, ws1.plan, ws1.resets, 9)
    d2 = W.RolloutDriver(ws2.store, ws2.plan, ws2.resets, 9)
    d1.run(70)
    for _ in range(70):
        d2.step()
    names = list(O.array_layout(oc, envs).keys())
    d = O.first_divergence({n: ws1.store.pull(n) for n in names}, {n: ws2.store.pull(n) for n in names})
    assert d is None, f"{name}: run(70) vs 70 steps, first divergence {d}"
    np.testing.assert_array_equal(d1.stats(), d2.stats())
    ws1.close()
    ws2.close()


@pytest.mark.gpu
def test_continuous_half_warp_staging_bit_exact():
    """Wide continuous rows staged by half-warps (chosen automatically when it
    fits more CTAs per SM, as at A = 1000; forced here at A = 300): bit-exact."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not O.libm_matches_replica():
        pytest.skip("host libm is not the glibc FMA variant the device replicates")
    kw, envs = CONT["cont_part_3x300"]
    oc = O.make_config(**{**kw, "episode_length": 25})
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    W.set_tuning("stage_rows", 16)
    try:
        ws = W.Workspace(dc, envs)
    finally:
        W.set_tuning("reset")
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, oc.seed)
    o = O.OracleWorld(oc, envs)
    for t in range(40):
        drv.step()
        o.rollout(t, 1, oc.seed)
        d = O.first_divergence({n: ws.store.pull(n) for n in o.layout}, o.snapshot())
        assert d is None, f"half-warp staging step {t}: first divergence {d}"
    ws2 = W.Workspace(dc, envs)  # multi-step windows on the same plan choice
    W.set_tuning("stage_rows", 16)
    try:
        ws3 = W.Workspace(dc, envs)
    finally:
        W.set_tuning("reset")
    d2 = W.RolloutDriver(ws2.store, ws2.plan, ws2.resets, 4)
    d3 = W.RolloutDriver(ws3.store, ws3.plan, ws3.resets, 4)
    d2.run(50)
    d3.run(50)
    names = list(o.layout)
    d = O.first_divergence({n: ws2.store.pull(n) for n in names}, {n: ws3.store.pull(n) for n in names})
    assert d is None, f"half vs full staging after run(50): first divergence {d}"
    for w in (ws, ws2, ws3):
        w.close()
