"""The host-buffer integration (wdg_rollout_step_host / _obs): the path behind
bench.py's `e2e` number, checked against the oracle.

A host learner reads, after RolloutDriver::step, the step's rewards and done
as the post_step hook sees them — BEFORE auto_reset (trainer.cpp:382-394,
harness.cpp:478-490) — and then the observations the next policy_forward
reads, i.e. AFTER the reset (trainer.cpp:358-360). The oracle is stepped the
same way (sample -> step -> track -> [capture rewards/done] -> reset_done ->
[capture observations]) with the same random host logits, and everything the
call returns plus the whole device store must be bit-exact (discrete Tag).

Also here: launch-overlap transitions: a flag-waiting overlapped
step right after a kernel that released it early without publishing env
flags (a bf16 policy step, collect's bootstrap forward) must equal the same
sequence launched serially."""
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


def pinned(shape, dtype):
    return torch.empty(shape, dtype=dtype, pin_memory=True)


HOST_CASES = {
    # dense: tags and resets inside the window (episode 15), partial K=5
    "disc_partial_24x12": (dict(num_taggers=2, num_runners=10, obs_mode=O.PARTIAL, episode_length=15,
                                grid_size=8, seed=3), 24),
    # one env per CTA (grid path), several chunks of CTAs
    "disc_partial_40x200": (dict(num_taggers=40, num_runners=160, obs_mode=O.PARTIAL, episode_length=12,
                                 seed=17), 40),
    # full observations, packed envs (several envs per CTA)
    "disc_full_30x20": (dict(num_taggers=4, num_runners=16, episode_length=10, grid_size=6, seed=8), 30),
    # C4's 1 + 4 agents: 95-float rows, so chunk starts must keep 16-byte alignment
    "disc_full_43x5": (dict(num_taggers=1, num_runners=4, episode_length=7, grid_size=4, seed=9), 43),
    # continuous partial on the one-env grid path
    "cont_partial_12x300": (dict(variant=O.CONTINUOUS, num_taggers=60, num_runners=240, obs_mode=O.PARTIAL,
                                 episode_length=8, world_length=12.0, tag_radius=0.6, seed=10), 12),
}


@pytest.mark.parametrize("name", list(HOST_CASES))
@pytest.mark.parametrize("mode", ["fused_auto", "fused_5chunks", "unfused"])
@pytest.mark.parametrize("with_obs", [True, False])
def test_step_host_matches_oracle(name, mode, with_obs):
    kw, E = HOST_CASES[name]
    if kw.get("variant") == O.CONTINUOUS and not O.libm_matches_replica():
        pytest.skip("host libm is not the glibc FMA variant the device replicates")
    dc, oc = cfg_pair(**kw)
    A = oc.num_taggers + oc.num_runners
    C, V, D = dc.action_categories(), dc.action_choices(), dc.obs_dim()
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, kw["seed"])
    if mode == "unfused":
        drv.set_fused(False)
    if mode == "fused_5chunks":
        drv.set_host_chunks(5)
    ow = O.OracleWorld(oc, E)
    rng = np.random.default_rng(99)
    h_logits = pinned((E, A, C, V), torch.float64)
    h_rew = pinned((E, A), torch.float32)
    h_done = pinned((E,), torch.uint8)
    h_obs = pinned((E, A, D), torch.float32) if with_obs else None
    dones = 0
    for t in range(36):
        lg = rng.normal(0.0, 2.0, (E, A, C, V))
        h_logits.numpy()[...] = lg
        h_rew.fill_(np.nan)
        h_done.fill_(7)
        if with_obs:
            h_obs.fill_(np.nan)
            drv.step_host(h_logits, lg.size, h_rew, h_done, h_obs, E * A * D)
        else:
            drv.step_host(h_logits, lg.size, h_rew, h_done)
        ws.store.synchronize()
        assert ow.sample(t, kw["seed"], lg) == 0
        ow.step(t)
        ow.track()
        want_r, want_d = ow.pull("rewards"), ow.pull("done")
        ow.reset_done()
        np.testing.assert_array_equal(h_rew.numpy().view(np.uint32), want_r.view(np.uint32).reshape(E, A),
                                      err_msg=f"step {t}: rewards (before reset)")
        np.testing.assert_array_equal(h_done.numpy(), want_d.reshape(E), err_msg=f"step {t}: done (before reset)")
        if with_obs:
            np.testing.assert_array_equal(h_obs.numpy().view(np.uint32),
                                          ow.pull("observations").view(np.uint32).reshape(E, A, D),
                                          err_msg=f"step {t}: observations (after reset)")
        d = O.first_divergence({n: ws.store.pull(n) for n in ow.layout}, ow.snapshot())
        assert d is None, f"step {t}: store diverged at {d}"
        dones += int(want_d.sum())
    drv.check()
    if mode != "unfused":  # the episode tracker runs inside the fused step
        np.testing.assert_array_equal(drv.stats()[:5], ow.stats()[:5])
    assert dones > 0, "the window must contain episode ends"
    for e in (0, E - 1):
        assert ws.resets.episodes_started(e) == ow.episodes(e)
    ws.close()


def test_step_host_errors():
    dc, _ = cfg_pair(num_taggers=2, num_runners=10, obs_mode=O.PARTIAL, episode_length=15, grid_size=8)
    ws = W.Workspace(dc, 4)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
    lg = np.zeros((4, 12, 1, 5))
    with pytest.raises(W.WarpError) as e:
        drv.step_host(lg, lg.size - 1)
    assert e.value.code == W.SHAPE_MISMATCH
    obs = np.zeros((4, 12, dc.obs_dim()), np.float32)
    with pytest.raises(W.WarpError) as e:
        drv.step_host(lg, lg.size, None, None, obs, obs.size - 1)
    assert e.value.code == W.SHAPE_MISMATCH
    with pytest.raises(W.WarpError) as e:
        drv.set_host_chunks(-1)
    assert e.value.code == W.INVALID_ARGUMENT
    assert drv.next_step() == 0  # nothing was stepped
    ws.close()


def test_step_host_headline_shape_sampled_envs():
    """C2 shape (2000 x 1000, partial K=5) through the pipelined host path
    (8 chunks of 250 envs): two steps with random host logits; sampled envs
    (global ids at both ends and across chunk borders) against the oracle."""
    kw = dict(num_taggers=200, num_runners=800, obs_mode=O.PARTIAL, seed=0)
    E, A, D = 2000, 1000, 23
    dc, oc = cfg_pair(**kw)
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
    rng = np.random.default_rng(5)
    h_logits = pinned((E, A, 1, 5), torch.float64)
    h_rew = pinned((E, A), torch.float32)
    h_done = pinned((E,), torch.uint8)
    h_obs = pinned((E, A, D), torch.float32)
    picks = [0, 249, 250, 1000, 1999]
    worlds = {e: O.OracleWorld(oc, 1, env_offset=e) for e in picks}  # global env e
    for t in range(2):
        lg = rng.normal(0.0, 1.0, (E, A, 1, 5))
        h_logits.numpy()[...] = lg
        drv.step_host(h_logits, lg.size, h_rew, h_done, h_obs, E * A * D)
        ws.store.synchronize()
        for e, w in worlds.items():
            assert w.sample(t, 0, lg[e:e + 1]) == 0
            w.step(t)
            w.track()
            np.testing.assert_array_equal(h_rew.numpy()[e], w.pull("rewards").reshape(A), err_msg=f"env {e} t {t}")
            np.testing.assert_array_equal(h_done.numpy()[e], w.pull("done").reshape(()))
            w.reset_done()
            np.testing.assert_array_equal(h_obs.numpy()[e], w.pull("observations").reshape(A, D),
                                          err_msg=f"env {e} t {t} obs")
    drv.check()
    ws.close()


# ---- launch-overlap transitions (programmatic dependent launch) ------------

def _pair(kw, E):
    dc, oc = cfg_pair(**kw)
    out = []
    for overlap in (True, False):
        ws = W.Workspace(dc, E)
        drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, kw["seed"])
        drv.set_overlap(overlap)
        out.append((ws, drv))
    return dc, oc, out


def _compare(oc, E, a, b, where):
    names = list(O.array_layout(oc, E).keys())
    d = O.first_divergence({n: a.store.pull(n) for n in names}, {n: b.store.pull(n) for n in names})
    assert d is None, f"{where}: overlapped vs serial, first divergence {d}"


@pytest.mark.parametrize("E", [600, 2000])
def test_overlap_after_bf16_policy_steps_equals_serial(E):
    """bf16 policy steps (plain PDL, released at entry, no env flags) ->
    set_policies(None) / set_logits -> flag-waiting overlapped steps: equal to
    the same sequence with overlap off, at the C2 agent count."""
    kw = dict(num_taggers=200, num_runners=800, obs_mode=O.PARTIAL, episode_length=9, seed=4)
    dc, oc, ((wa, da), (wb, db)) = _pair(kw, E)
    pol_t, pol_r = W.Policy.for_tag(dc, seed=1), W.Policy.for_tag(dc, seed=2)
    rng = np.random.default_rng(3)
    lg = torch.from_numpy(rng.normal(0, 1, (E, 1000, 1, 5))).cuda()
    for d in (da, db):
        d.set_policies(pol_t, pol_r, W.POLICY_BF16)
        for _ in range(3):
            d.step()
        d.set_policies(None)
        for _ in range(3):
            d.step()  # uniform policy right behind the bf16 steps
        d.set_policies(pol_t, pol_r, W.POLICY_BF16)
        d.step()
        d.set_logits(lg, lg.numel())  # explicit logits right behind a bf16 step
        for _ in range(3):
            d.step()
        d.set_policies(pol_t, pol_r, W.POLICY_BF16)
        d.step()
        d.set_policies(None)
        d.run(40)  # graph / multi-step windows right behind a bf16 step
    _compare(oc, E, wa, wb, "bf16 -> logits transitions")
    np.testing.assert_array_equal(da.stats(), db.stats())
    for w in (wa, wb):
        w.close()


def test_overlap_after_collect_equals_serial():
    """collect() ends with a bf16 bootstrap forward that releases its
    dependents at entry; the next overlapped uniform-policy steps must wait
    for it (it reads the observations those steps overwrite)."""
    kw = dict(num_taggers=200, num_runners=800, obs_mode=O.PARTIAL, episode_length=9, seed=6)
    E, T = 800, 4
    dc, oc, ((wa, da), (wb, db)) = _pair(kw, E)
    pol = W.Policy.for_tag(dc, seed=9)
    boots = []
    for ws, d in ((wa, da), (wb, db)):
        d.set_policies(pol, pol, W.POLICY_BF16)
        batch = W.RolloutBatch(ws.store, T)
        d.collect(batch)
        d.set_policies(None)
        for _ in range(4):
            d.step()
        torch.cuda.synchronize()
        boots.append(batch.pull("bootstrap"))
        batch.close()
    np.testing.assert_array_equal(boots[0], boots[1])
    _compare(oc, E, wa, wb, "collect -> uniform steps")
    for w in (wa, wb):
        w.close()
