"""Rollout-capture row: RolloutBatch + Trainer::collect
hooks + compute_returns (proj/src/trainer.cpp:58-88,315-403) on device.

CPU: the oracle's compute_returns / logp restatement is pinned bit-for-bit to
the reference (trainer.cpp compiled in oracle/_ref).
GPU: RolloutDriver.collect with device policies against oracle.collect on the
same seeds — obs, actions, active, rewards, done bit-exact; values, logp and
bootstrap within LOGIT_RTOL (CUDA vs glibc tanh/exp/log ulps); device
compute_returns bit-exact given the batch."""
import numpy as np
import pytest

import oracle as O
import paper_2108_13976_b200 as W

LOGIT_RTOL = 1e-12


@pytest.mark.parametrize("gamma", [0.5, 0.97, 0.999])
def test_oracle_returns_match_reference(gamma):
    if not O.ref_available():
        pytest.skip("reference build oracle/_ref not available")
    rng = np.random.default_rng(int(gamma * 1000))
    T, E, A = 23, 7, 9
    r = rng.choice(np.array([-1.0, 0.0, 1.0, 2.0, 0.25], dtype=np.float32), size=(T, E, A))
    d = (rng.random((T, E)) < 0.15).astype(np.uint8)
    b = rng.normal(size=(E, A))
    a = O.compute_returns(r, d, b, gamma)
    c = O.compute_returns(r, d, b, gamma, ref=True)
    np.testing.assert_array_equal(a.view(np.uint64), c.view(np.uint64))


def test_oracle_logp_properties():
    rng = np.random.default_rng(2)
    z = rng.normal(0, 2, size=(50, 2, 3))
    acts = rng.integers(0, 3, size=(50, 2)).astype(np.int32)
    lp = O.logp_of(z.reshape(-1), acts.reshape(-1), 2, 3)
    zs = z - z.max(axis=2, keepdims=True)
    want = (np.take_along_axis(zs, acts[:, :, None], 2)[:, :, 0] - np.log(np.exp(zs).sum(2))).sum(1)
    np.testing.assert_allclose(lp, want, rtol=1e-13, atol=1e-13)


def rel_err(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("shared", [True, False])
def test_collect_matches_oracle(shared):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    kw = dict(num_taggers=12, num_runners=48, obs_mode=O.PARTIAL, episode_length=12, grid_size=10, seed=7)
    E, T = 9, 20
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    dims = O.PolicyDims(dc.obs_dim(), (64, 64), 1, 5)
    pt = O.policy_init(31, dims)
    pr = pt if shared else O.policy_init(32, dims)
    dev_t = W.Policy.for_tag(dc, seed=31)
    dev_r = dev_t if shared else W.Policy.for_tag(dc, seed=32)
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, kw["seed"])
    drv.set_policies(dev_t, None if shared else dev_r)
    ow = O.OracleWorld(oc, E)
    # two consecutive collects: the second starts at global step T
    for first in (0, T):
        batch = W.RolloutBatch(ws.store, T)
        drv.collect(batch)
        want = O.collect(ow, oc, pt, pr, dims, T, first, kw["seed"])
        for name in ("obs", "actions", "active", "rewards", "done"):
            got = batch.pull(name)
            np.testing.assert_array_equal(got, want[name].reshape(got.shape), err_msg=f"{name} (from {first})")
        for name in ("values", "logp", "bootstrap"):
            got = batch.pull(name)
            assert rel_err(got, want[name].reshape(got.shape)) <= LOGIT_RTOL, name
        # done flags actually occur (episode_length 12 < T)
        assert want["done"].sum() > 0
        # compute_returns on device == oracle on the device batch's own arrays
        ret = torch.empty(batch.shapes["rewards"], dtype=torch.float64, device="cuda")
        batch.compute_returns(0.95, ret)
        oret = O.compute_returns(batch.pull("rewards"), batch.pull("done"), batch.pull("bootstrap"), 0.95)
        np.testing.assert_array_equal(ret.cpu().numpy().view(np.uint64), oret.view(np.uint64))
        batch.close()
    d = O.first_divergence({n: ws.store.pull(n) for n in ow.layout}, ow.snapshot())
    assert d is None, d
    ws.close()


@pytest.mark.gpu
def test_collect_requires_policies():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    dc = W.TagConfig(num_taggers=2, num_runners=6)
    ws = W.Workspace(dc, 3)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
    batch = W.RolloutBatch(ws.store, 4)
    with pytest.raises(W.WarpError) as e:
        drv.collect(batch)
    assert e.value.code == W.STATE
    ws.close()
