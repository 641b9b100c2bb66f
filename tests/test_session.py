"""Session-ABI row: the reference's wd_session_* entry
points (proj/include/warp/warp_c.h, proj/src/c_api.cpp) on the device path.

CPU: the strict RunConfig parser, canonical JSON and FNV-1a config hash equal
the reference's own (harness.cpp compiled in oracle/_ref against the same
nlohmann/json 3.11.3), including error codes for malformed configs.
GPU: check / bench-envs / bench-agents run on the B200 kernels and report in
the reference's JSON shape; dump_array writes the store CSV."""
import json
import os

import pytest

import oracle as O
import paper_2108_13976_b200 as W

CONFIGS = [
    "{}",
    '{"env": {"num_taggers": 3, "obs_mode": "partial", "seed": 7}, "run": {"env_counts": [1, 8]}}',
    '{"env": {"variant": "continuous", "world_length": 12.5, "tag_radius": 0.75, "turn_delta": 0.1,'
    ' "k_nearest": 3, "obs_mode": "partial", "num_runners": 20, "seed": 18446744073709551615},'
    ' "engine": {"num_envs": 16, "worker_count": 0, "deterministic": false},'
    ' "trainer": {"algorithm": "ppo", "gamma": 0.95, "hidden_sizes": [32, 16, 8], "seed": 5},'
    ' "run": {"mode": "check", "check_steps": 7, "bench_obs_modes": ["full"], "bench_budget_ms": 12.5,'
    ' "dump_arrays": ["loc_x", "rewards"], "output_dir": "x"}}',
]

BAD = [
    ('{"env": {"bogus": 1}}', 11),            # unknown key -> parse_error
    ('{"env": {"grid_size": "20"}}', 11),      # wrong type -> parse_error
    ('{"env": {"variant": "hex"}}', 11),       # bad enum -> parse_error
    ('{"engine": {"num_envs": 0}}', 8),        # invalid_config
    ('{"trainer": {"gamma": 1.5}}', 8),        # invalid_config
    ('{"env": {"obs_mode": "partial", "num_taggers": 1, "num_runners": 2, "k_nearest": 3}}', 8),
    ('[1, 2]', 11),
    ('{"env": ', 11),
]


def need_ref():
    if not O.ref_available() or O.ref_config_canonical("{}")[0] is None:
        pytest.skip("reference harness build (oracle/_ref + json.hpp) not available")


@pytest.mark.parametrize("text", CONFIGS)
def test_canonical_config_and_hash_match_reference(text):
    need_ref()
    s = W.Session(text)
    assert s.config_json() == O.ref_config_canonical(text)[1]
    assert s.config_hash() == O.ref_config_canonical(text, hash=True)[1]
    s.close()


@pytest.mark.parametrize("text,code", BAD)
def test_config_errors_match_reference(text, code):
    with pytest.raises(W.WarpError) as e:
        W.Session(text)
    assert e.value.code == code
    if O.ref_available() and O.ref_config_canonical("{}")[0] is not None:
        assert O.ref_config_canonical(text)[0] == code


def test_overrides_and_training_out_of_scope(tmp_path):
    need_ref()
    s = W.Session('{"env": {"seed": 1}, "trainer": {"seed": 2}}')
    s.set_seed(99)  # sets env and trainer seeds (c_api.cpp:128-133)
    assert s.config_hash() == O.ref_config_canonical('{"env": {"seed": 99}, "trainer": {"seed": 99}}', True)[1]
    s.set_workers(3)
    s.set_output_dir(str(tmp_path))
    cfg = json.loads(s.config_json())
    assert cfg["engine"]["worker_count"] == 3 and cfg["run"]["output_dir"] == str(tmp_path)
    with pytest.raises(W.WarpError) as e:
        s.run_training()
    assert e.value.code == W.STATE
    assert s.report_json() is None and s.summary() is None
    s.close()
    p = tmp_path / "cfg.json"
    p.write_text(CONFIGS[1])
    s2 = W.Session(path=str(p))
    assert s2.config_hash() == O.ref_config_canonical(CONFIGS[1], True)[1]
    with pytest.raises(W.WarpError) as e:
        W.Session(path=str(tmp_path / "missing.json"))
    assert e.value.code == W.IO


@pytest.mark.gpu
def test_session_modes_on_device(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = {"env": {"num_taggers": 2, "num_runners": 8, "k_nearest": 4, "episode_length": 15, "seed": 3},
           "engine": {"num_envs": 6},
           "trainer": {"seed": 4},
           "run": {"check_steps": 40, "env_counts": [1, 64], "agent_counts": [10, 100],
                   "bench_budget_ms": 60, "bench_reps": 2, "output_dir": str(tmp_path)}}
    s = W.Session(json.dumps(cfg))
    s.run_check()
    rep = json.loads(s.report_json())
    assert rep["passed"] is True and len(rep["combos"]) == 4
    assert {(c["variant"], c["obs_mode"]) for c in rep["combos"]} == {
        ("discrete", "full"), ("discrete", "partial"), ("continuous", "full"), ("continuous", "partial")}
    assert rep["meta"]["config_hash"] == s.config_hash() and rep["meta"]["mode"] == "check"
    assert s.summary().startswith("check: PASS (4/4 combos)")
    # both legs ran: production plan vs the device TagReference twin, fused vs unfused
    assert all(c["legs"]["reference"]["passed"] and c["legs"]["fused"]["passed"] for c in rep["combos"])
    assert (tmp_path / "check.csv").exists() and (tmp_path / "report.json").exists()
    s.dump_array("observations", str(tmp_path / "obs.csv"))
    lines = (tmp_path / "obs.csv").read_text().splitlines()
    assert lines[0].startswith("env,v0,") and len(lines) == 1 + 6

    s.run_bench_envs()
    rep = json.loads(s.report_json())
    assert [r["env_count"] for r in rep["rows"]] == [1, 64]
    assert all(r["steps_per_sec"] > 0 for r in rep["rows"])

    s.run_bench_agents()
    rep = json.loads(s.report_json())
    assert len(rep["rows"]) == 4 and set(rep["slopes"]) == {"partial", "full"}
    assert all(r["per_env_step_us"] > 0 for r in rep["rows"])
    assert os.path.exists(tmp_path / "bench_agents.csv")
    s.close()


@pytest.mark.gpu
def test_session_check_catches_fault_hook(tmp_path):
    """Mutation test of the device check: the fault hook biases
    the production plan's tag radius only; the independent TagReference twin
    is unaffected, so the reference leg reports the first divergence, in
    rewards, as the reference's checker does (harness.cpp:619-629)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = {"env": {"num_taggers": 2, "num_runners": 10, "k_nearest": 5, "episode_length": 100, "seed": 1},
           "engine": {"num_envs": 60}, "trainer": {"seed": 4},
           "run": {"check_steps": 100, "output_dir": str(tmp_path)}}
    s = W.Session(json.dumps(cfg))
    W.set_fault_tag_radius_bias(1.0)
    try:
        with pytest.raises(W.WarpError) as ei:  # a failed check is WD_ERR_STATE (c_api.cpp:205-212)
            s.run_check()
        assert ei.value.code == W.STATE
    finally:
        W.set_fault_tag_radius_bias(0.0)
    rep = json.loads(s.report_json())
    assert rep["passed"] is False
    failing = [c for c in rep["combos"] if not c["passed"]]
    assert failing
    for c in failing:
        assert c["divergence"]["leg"] == "reference"
        assert c["divergence"]["array"] == "rewards"
    assert "FAIL" in s.summary()
    s.close()
