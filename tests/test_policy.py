"""Policy forward row: the reference MLP
(proj/src/policy_model.cpp) as the producer of the rollout's logits.

CPU (not gpu): the C restatement (oracle/tag_oracle.c) is pinned bit-for-bit
to the reference (oracle/_ref, policy_model.cpp compiled from the reference
sources) for init_policy and forward; the product library's host-side
init_policy equals the reference bit-for-bit (no GPU needed).

GPU: the device f64 forward against the oracle forward (tolerance LOGIT_RTOL:
CUDA's tanh and glibc's tanh may round an activation differently by 1 ulp,
nothing else differs), and full rollouts driven by device policies against
the oracle driven by the oracle forward — bit-exact on every store array."""
import numpy as np
import pytest

import oracle as O
import paper_2108_13976_b200 as W

LOGIT_RTOL = 1e-12  # relative |device - oracle| of f64 logits / values (tanh ulps only)

DIMS = [
    O.PolicyDims(23, (64, 64), 1, 5),    # discrete partial K=5 (the C2 shape)
    O.PolicyDims(41, (64, 64), 2, 3),    # continuous partial K=5
    O.PolicyDims(19, (33, 7, 70), 1, 5),  # odd widths, 3 layers
]


def need_ref():
    if not O.ref_available():
        pytest.skip("reference build oracle/_ref not available")


@pytest.mark.parametrize("dims", DIMS, ids=lambda d: f"D{d.obs_dim}_{'x'.join(map(str, d.hidden))}")
@pytest.mark.parametrize("seed", [0, 7, 2**40 + 3])
def test_oracle_policy_init_matches_reference(dims, seed):
    need_ref()
    a = O.policy_init(seed, dims)
    b = O.policy_init(seed, dims, ref=True)
    assert a.shape == b.shape and a.size == O.policy_param_count(dims)
    np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("dims", DIMS, ids=lambda d: f"D{d.obs_dim}_{'x'.join(map(str, d.hidden))}")
def test_oracle_policy_forward_matches_reference(dims):
    need_ref()
    rng = np.random.default_rng(11)
    params = O.policy_init(5, dims) + rng.normal(0, 0.05, O.policy_param_count(dims))
    obs = rng.normal(0, 1.5, (300, dims.obs_dim)).astype(np.float32)
    la, va = O.policy_forward(params, dims, obs)
    lb, vb = O.policy_forward(params, dims, obs, ref=True)
    np.testing.assert_array_equal(la.view(np.uint64), lb.view(np.uint64))
    np.testing.assert_array_equal(va.view(np.uint64), vb.view(np.uint64))


def test_oracle_policy_forward_non_finite():
    dims = DIMS[0]
    obs = np.zeros((2, dims.obs_dim), dtype=np.float32)
    obs[1, 3] = np.nan
    with pytest.raises(ValueError, match="status 10"):
        O.policy_forward(O.policy_init(0, dims), dims, obs)


@pytest.mark.parametrize("dims", DIMS, ids=lambda d: f"D{d.obs_dim}_{'x'.join(map(str, d.hidden))}")
def test_library_policy_init_matches_reference(dims):
    """Host-side init_policy of the product library (no device work)."""
    p = W.Policy(dims.obs_dim, dims.hidden, dims.num_categories, dims.num_choices, seed=123)
    got = p.get_params()
    want = O.policy_init(123, dims, ref=O.ref_available())
    assert p.param_count() == want.size
    np.testing.assert_array_equal(got.view(np.uint64), want.view(np.uint64))
    p.close()


def test_library_policy_params_roundtrip_and_errors():
    p = W.Policy(23, (64, 64), 1, 5)
    v = np.arange(p.param_count(), dtype=np.float64) * 0.001
    p.set_params(v)
    np.testing.assert_array_equal(p.get_params(), v)
    with pytest.raises(W.WarpError) as e:
        p.set_params(v[:-1])
    assert e.value.code == W.SHAPE_MISMATCH
    with pytest.raises(W.WarpError) as e:
        W.Policy(23, (), 1, 5)
    assert e.value.code == W.INVALID_ARGUMENT
    p.close()


# ---- GPU ---------------------------------------------------------------------
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


def rel_err(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("dims", DIMS, ids=lambda d: f"D{d.obs_dim}_{'x'.join(map(str, d.hidden))}")
def test_device_f64_forward_matches_oracle(dims):
    torch = _gpu()
    rng = np.random.default_rng(3)
    E, A = 37, 29
    params = O.policy_init(9, dims) + rng.normal(0, 0.05, O.policy_param_count(dims))
    obs = rng.normal(0, 1.5, (E, A, dims.obs_dim)).astype(np.float32)
    p = W.Policy(dims.obs_dim, dims.hidden, dims.num_categories, dims.num_choices)
    p.set_params(params)
    d_obs = torch.from_numpy(obs).cuda()
    Wd = dims.logits_width()
    d_lg = torch.full((E, A, Wd), -7.0, dtype=torch.float64, device="cuda")
    d_v = torch.full((E, A), -7.0, dtype=torch.float64, device="cuda")
    # two agent ranges, like the tagger / runner policy groups
    p.forward(d_obs, E, A, d_lg, d_v, 0, 11)
    p.forward(d_obs, E, A, d_lg, d_v, 11, A)
    lg, v = O.policy_forward(params, dims, obs.reshape(-1, dims.obs_dim))
    assert rel_err(d_lg.cpu().numpy().reshape(-1, Wd), lg) <= LOGIT_RTOL
    assert rel_err(d_v.cpu().numpy().reshape(-1), v) <= LOGIT_RTOL
    # a sub-range leaves the other rows untouched
    d_lg2 = torch.full((E, A, Wd), -7.0, dtype=torch.float64, device="cuda")
    p.forward(d_obs, E, A, d_lg2, None, 5, 9)
    out = d_lg2.cpu().numpy()
    assert np.all(out[:, :5] == -7.0) and np.all(out[:, 9:] == -7.0)
    assert rel_err(out[:, 5:9].reshape(-1, Wd), lg.reshape(E, A, Wd)[:, 5:9].reshape(-1, Wd)) <= LOGIT_RTOL
    # non-finite observation -> non_finite (policy_model.cpp:152-154)
    obs[3, 4, 1] = np.inf
    with pytest.raises(W.WarpError) as e:
        p.forward(torch.from_numpy(obs).cuda(), E, A, d_lg, None)
    assert e.value.code == W.NON_FINITE
    p.close()


POLICY_ROLLOUTS = {
    "disc_part_12x60_shared": (dict(num_taggers=12, num_runners=48, obs_mode=O.PARTIAL, episode_length=30,
                                    grid_size=12, seed=4), 12, True),
    "disc_part_6x300_split": (dict(num_taggers=60, num_runners=240, obs_mode=O.PARTIAL, episode_length=25,
                                   grid_size=14, seed=6), 6, False),
    "disc_full_20x8_split": (dict(num_taggers=2, num_runners=6, episode_length=20, seed=2), 20, False),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(POLICY_ROLLOUTS))
@pytest.mark.parametrize("fused", [True, False])
def test_policy_rollout_matches_oracle(name, fused):
    """RolloutDriver::step with policies (harness.cpp:478-490): forward on the
    current obs -> sample(t) -> step -> reset, device vs oracle, bit-exact."""
    torch = _gpu()
    kw, E, shared = POLICY_ROLLOUTS[name]
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    dims = O.PolicyDims(dc.obs_dim(), (64, 64), dc.action_categories(), dc.action_choices())
    # the Trainer seeds tag i with mix64(seed) + i over the sorted tags (trainer.cpp:286-291);
    # any distinct seeds exercise the two groups
    pt = O.policy_init(101, dims)
    pr = pt if shared else O.policy_init(202, dims)
    dev_t = W.Policy.for_tag(dc, seed=101)
    dev_r = dev_t if shared else W.Policy.for_tag(dc, seed=202)
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, kw["seed"])
    drv.set_fused(fused)
    drv.set_policies(dev_t, None if shared else dev_r)
    ow = O.OracleWorld(oc, E)
    seed = kw["seed"]
    for t in range(45):
        logits = O.tag_policy_logits(ow, oc, pt, pr, dims)
        drv.step()
        ow.rollout(t, 1, seed, logits)
        if t % 5 == 0 or t == 44:
            dev = {n: ws.store.pull(n) for n in ow.layout}
            d = O.first_divergence(dev, ow.snapshot())
            assert d is None, f"{name} step {t}: first divergence {d}"
            lg_ptr, _ = drv.policy_outputs()
            got = np.zeros(logits.size, dtype=np.float64)
            W.copy_to_host(lg_ptr, got)
            assert rel_err(got, logits) <= LOGIT_RTOL, f"{name} step {t}: policy logits"
    drv.check()
    ws.close()


# ---- bf16 tensor-core path -----------------------------------------------------
BF16_EMU_ATOL = 5e-3   # vs a torch fp32 forward that rounds operands/activations to bf16 like the kernel
BF16_F32_ATOL = 6e-2   # vs the plain torch fp32 forward of the same parameters (bf16 quantisation error)


def torch_mlp(torch, params, dims, obs, emulate_bf16):
    """Plain PyTorch fp32 forward of the reference MLP (policy_model.cpp:146-197)."""
    p = torch.as_tensor(params, dtype=torch.float32)
    q = (lambda t: t.to(torch.bfloat16).to(torch.float32)) if emulate_bf16 else (lambda t: t)
    D, W = dims.obs_dim, dims.logits_width()
    off = 0
    x = q(torch.as_tensor(obs, dtype=torch.float32))
    in_w = D
    for h in dims.hidden:
        w = p[off:off + h * in_w].reshape(h, in_w)
        b = p[off + h * in_w: off + h * in_w + h]
        x = q(torch.tanh(x @ q(w).T + b))
        off += h * in_w + h
        in_w = h
    hw = p[off:off + W * in_w].reshape(W, in_w)
    hb = p[off + W * in_w: off + W * in_w + W]
    vw = p[off + W * in_w + W: off + W * in_w + W + in_w]
    vb = p[off + W * in_w + W + in_w]
    return (x @ q(hw).T + hb).numpy(), (x @ q(vw) + vb).numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("dims", DIMS[:2], ids=lambda d: f"D{d.obs_dim}")
def test_device_bf16_forward_matches_torch(dims):
    torch = _gpu()
    rng = np.random.default_rng(5)
    E, A = 53, 37  # 1961 rows: 16 tiles of 128, the last partial
    params = O.policy_init(4, dims) + rng.normal(0, 0.05, O.policy_param_count(dims))
    obs = rng.uniform(-1, 1, (E, A, dims.obs_dim)).astype(np.float32)
    p = W.Policy(dims.obs_dim, dims.hidden, dims.num_categories, dims.num_choices)
    p.set_params(params)
    Wd = dims.logits_width()
    d_lg = torch.full((E, A, Wd), -7.0, dtype=torch.float64, device="cuda")
    d_v = torch.full((E, A), -7.0, dtype=torch.float64, device="cuda")
    p.forward(torch.from_numpy(obs).cuda(), E, A, d_lg, d_v, 0, 10, precision=W.POLICY_BF16)
    p.forward(torch.from_numpy(obs).cuda(), E, A, d_lg, d_v, 10, A, precision=W.POLICY_BF16)
    lg = d_lg.cpu().numpy().reshape(-1, Wd)
    v = d_v.cpu().numpy().reshape(-1)
    el, ev = torch_mlp(torch, params, dims, obs.reshape(-1, dims.obs_dim), True)
    fl, fv = torch_mlp(torch, params, dims, obs.reshape(-1, dims.obs_dim), False)
    assert np.max(np.abs(lg - el)) <= BF16_EMU_ATOL, np.max(np.abs(lg - el))
    assert np.max(np.abs(v - ev)) <= BF16_EMU_ATOL
    assert np.max(np.abs(lg - fl)) <= BF16_F32_ATOL, np.max(np.abs(lg - fl))
    assert np.max(np.abs(v - fv)) <= BF16_F32_ATOL
    p.close()


@pytest.mark.gpu
@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("shared", [True, False])
def test_bf16_policy_rollout_samples_its_logits_exactly(fused, shared):
    """The bf16 kernel samples in its epilogue from f64(its f32 logits): the
    oracle stepped with those very logits (sampler.cpp + TagReference) must
    reproduce the device store bit-for-bit; the actions also agree with the
    f64 policy's for the overwhelming majority of agents."""
    _gpu()
    kw = dict(num_taggers=20, num_runners=80, obs_mode=O.PARTIAL, episode_length=25, grid_size=12, seed=5)
    E = 10
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    dims = O.PolicyDims(dc.obs_dim(), (64, 64), 1, 5)
    dev_t = W.Policy.for_tag(dc, seed=11)
    dev_r = dev_t if shared else W.Policy.for_tag(dc, seed=12)
    pt = O.policy_init(11, dims)
    pr = pt if shared else O.policy_init(12, dims)
    ws = W.Workspace(dc, E)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, kw["seed"])
    drv.set_fused(fused)
    drv.set_policies(dev_t, None if shared else dev_r, W.POLICY_BF16)
    drv.set_keep_policy_outputs(True)
    ow = O.OracleWorld(oc, E)
    agree = total = 0
    for t in range(40):
        f64_logits = O.tag_policy_logits(ow, oc, pt, pr, dims)
        f64_actions = ow.pull("sampled_actions").copy()
        drv.step()
        lg_ptr, _ = drv.policy_outputs()
        dev_logits = W.copy_to_host(lg_ptr, np.zeros(f64_logits.size, dtype=np.float64))
        assert np.max(np.abs(dev_logits - f64_logits)) <= BF16_F32_ATOL
        # what the f64 policy would have sampled at this step
        probe = O.OracleWorld(oc, E)  # sampling depends only on (seed, step, env, agent, logits)
        probe.sample(t, kw["seed"], f64_logits)
        want = probe.pull("sampled_actions").copy()
        del probe, f64_actions
        ow.rollout(t, 1, kw["seed"], dev_logits)
        got = ws.store.pull("sampled_actions")
        agree += int(np.sum(got == want))
        total += got.size
        d = O.first_divergence({n: ws.store.pull(n) for n in ow.layout}, ow.snapshot())
        assert d is None, f"step {t}: first divergence {d}"
    drv.check()
    assert agree / total >= 0.95, agree / total
    ws.close()
