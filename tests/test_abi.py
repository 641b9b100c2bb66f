"""CPU-side checks of the drop-in boundary: the product library loads, exports
every symbol include/wdg_b200.h declares, keeps the reference's status
numbering, validates configs like TagConfig::validate (no device needed), and
fails loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2108_13976_b200 as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wdg_b200.h")
REF_HEADER = "/root/reference/proj/include/warp/warp_c.h"


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"WDG_API\s+[\w\s\*]+?\b(wdg_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = W.lib()
    syms = declared_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(W.EXPORTED_SYMBOLS) == syms


def test_library_is_sm100a_and_has_no_oracle_code():
    so = W.library_path()
    nm = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    assert "oracle_" not in nm and "ref_world" not in nm
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    pkg = os.path.join(ROOT, "paper_2108_13976_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".hpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "tag_oracle" not in src, f


def test_status_names_match_reference_numbering():
    lib = W.lib()
    for code, name in enumerate(W.STATUS_NAMES):
        assert lib.wdg_status_name(code).decode() == name
    if os.path.exists(REF_HEADER):  # wd_status order, warp_c.h:22-38
        body = open(REF_HEADER).read().split("typedef enum wd_status {")[1].split("}")[0]
        ref = [t.strip().split("=")[0].strip() for t in body.split(",") if t.strip()]
        assert ref == W.STATUS_NAMES[:15]


@pytest.mark.parametrize("kw,ok", [
    (dict(), True),
    (dict(num_taggers=0), False),
    (dict(num_runners=0), False),
    (dict(episode_length=0), False),
    (dict(tag_reward=0.0), False),
    (dict(tagged_penalty=0.0), False),
    (dict(grid_size=0), False),
    (dict(variant=W.CONTINUOUS, world_length=0.0), False),
    (dict(variant=W.CONTINUOUS, tag_radius=-1.0), False),
    (dict(variant=W.CONTINUOUS, accel_delta=0.0), False),
    (dict(variant=W.CONTINUOUS, max_speed_runner=0.0), False),
    (dict(obs_mode=W.PARTIAL, k_nearest=0), False),
    (dict(obs_mode=W.PARTIAL, k_nearest=12), False),   # SPEC.md: k >= agents
    (dict(obs_mode=W.PARTIAL, k_nearest=11), True),
])
def test_config_validation_matches_reference(kw, ok):
    cfg = W.TagConfig(**kw)
    if ok:
        cfg.validate()
    else:
        with pytest.raises(W.WarpError) as ei:
            cfg.validate()
        assert ei.value.code == W.INVALID_CONFIG


def test_obs_dim_and_zero_on_reset():
    assert W.TagConfig(num_taggers=1, num_runners=4).obs_dim() == 19
    assert W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL).obs_dim() == 23
    assert W.TagConfig(num_taggers=200, num_runners=800).obs_dim() == 3999
    assert W.TagConfig(variant=W.CONTINUOUS, num_taggers=200, num_runners=800,
                       obs_mode=W.PARTIAL).obs_dim() == 41
    assert W.tag_zero_on_reset() == ["step_count", "rewards", "done", "tag_credits", "was_tagged",
                                     "sampled_actions", "observations"]


def test_null_arguments_are_errors_not_crashes():
    lib = W.lib()
    assert lib.wdg_store_create(2, 2, None) == W.INVALID_ARGUMENT
    assert "null" in lib.wdg_last_error().decode()
    assert lib.wdg_run_step(None, 0) == W.INVALID_ARGUMENT
    assert lib.wdg_rollout_step(None) == W.INVALID_ARGUMENT


def test_no_gpu_fails_loudly():
    if W.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(W.WarpError) as ei:
        W.DataStore(2, 5)
    assert ei.value.code == W.CUDA_ERROR
    assert "no CPU fallback" in str(ei.value)


def build_cpp_example(tmp_dir):
    """Builds tests/cpp/facade_example.cpp against include/warp_b200.hpp and
    the product library (what a reference-side C++ integration compiles)."""
    lib_dir = os.path.dirname(W.library_path())
    exe = os.path.join(str(tmp_dir), "facade_example")
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_example.cpp"), "-L", lib_dir, "-lwdg_b200",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    return exe


def test_cpp_facade_builds_and_fails_loudly_without_gpu(tmp_path):
    exe = build_cpp_example(tmp_path)
    if W.device_count() > 0:
        pytest.skip("GPU present: the run is covered by test_parity_gpu")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "no CUDA device" in r.stderr


def test_tuning_keys_documented_and_accepted():
    """Every plan tuning key the header lists is accepted by wdg_set_tuning
    (host-side table, no device), an unknown key is an error, and "reset"
    restores the plan's own choices."""
    text = open(HEADER).read()
    block = text[text.index("Plan tuning overrides"):text.index("WDG_API wdg_status wdg_set_tuning")]
    keys = re.findall(r"\b([a-z][a-z0-9]*(?:_[a-z0-9]+)+|multistep)\b", block.split("Keys:")[1].split(";")[0])
    assert {"brute_max", "cont_keys", "packed_warps_max", "pdl_mode", "multistep"} <= set(keys)
    try:
        for k in keys:
            W.set_tuning(k, 1)
            W.set_tuning(k, -1)
        with pytest.raises(Exception):
            W.set_tuning("no_such_key", 1)
    finally:
        W.set_tuning("reset")
