"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, the
reference's own sources compiled by oracle/Makefile). Run here, where
/root/reference exists:  python tests/golden/make_golden.py

Each fixture holds, for a small config driven exactly like RolloutDriver::step
(harness.cpp:478-490) with zero logits (or fixed random logits):
  * init_<array>            the registration-time arrays (episode 0)
  * step_digest / reset_digest  blake2b-64 of every array after each step
                             (before reset) and after the reset, per step
  * final_<array>           the arrays after the last step + reset
  * episodes                episodes_started per env at the end
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

CONFIGS = {
    # C1: BASELINE.json configs[0] — 1 env x (1 tagger + 4 runners), full obs, 100 steps, seed 0
    "c1_discrete_full_1x5": dict(cfg=dict(num_taggers=1, num_runners=4), envs=1, steps=100),
    # dense configs so tags and resets actually occur
    "discrete_partial_60x12": dict(cfg=dict(num_taggers=2, num_runners=10, obs_mode=O.PARTIAL,
                                            episode_length=50, seed=7), envs=60, steps=120),
    "discrete_full_20x12": dict(cfg=dict(num_taggers=2, num_runners=10, obs_mode=O.FULL,
                                         episode_length=40, seed=3, grid_size=8), envs=20, steps=100),
    "discrete_partial_4x1000": dict(cfg=dict(num_taggers=200, num_runners=800, obs_mode=O.PARTIAL,
                                             seed=42), envs=4, steps=40),
    "discrete_partial_3x100_logits": dict(cfg=dict(num_taggers=20, num_runners=80, obs_mode=O.PARTIAL,
                                                   k_nearest=7, seed=11, grid_size=12), envs=3,
                                          steps=60, logits=True),
    "continuous_partial_20x12": dict(cfg=dict(variant=O.CONTINUOUS, num_taggers=2, num_runners=10,
                                              obs_mode=O.PARTIAL, episode_length=60, seed=5,
                                              world_length=8.0), envs=20, steps=80),
    "continuous_full_10x6": dict(cfg=dict(variant=O.CONTINUOUS, num_taggers=2, num_runners=4,
                                          obs_mode=O.FULL, episode_length=30, seed=9,
                                          world_length=6.0), envs=10, steps=60, logits=True),
}


def digest(snap):
    out = {}
    for k in sorted(snap):
        out[k] = hashlib.blake2b(snap[k].tobytes(), digest_size=8).hexdigest()
    return out


def logits_for(name, cfg, envs, t):
    rng = np.random.default_rng(abs(hash((name, t))) % (2**32) if False else 1000 + t)
    c = 2 if cfg.variant == O.CONTINUOUS else 1
    v = 3 if cfg.variant == O.CONTINUOUS else 5
    a = cfg.num_taggers + cfg.num_runners
    return rng.normal(0.0, 2.0, size=(envs, a, c, v))


def make(name, spec):
    cfg = O.make_config(**spec["cfg"])
    w = O.RefWorld(cfg, spec["envs"])
    out = {}
    for k, v in w.snapshot().items():
        out["init_" + k] = v
    step_dig, reset_dig = [], []
    for t in range(spec["steps"]):
        lg = logits_for(name, cfg, spec["envs"], t) if spec.get("logits") else None
        w.sample(t, cfg.seed, lg)
        w.step(t)
        step_dig.append(digest(w.snapshot()))
        w.reset_done()
        reset_dig.append(digest(w.snapshot()))
    for k, v in w.snapshot().items():
        out["final_" + k] = v
    out["episodes"] = np.array([w.episodes(e) for e in range(spec["envs"])], dtype=np.int64)
    out["step_digest"] = np.array(json.dumps(step_dig))
    out["reset_digest"] = np.array(json.dumps(reset_dig))
    out["config"] = np.array(json.dumps(spec, default=int))
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {os.path.getsize(path)} bytes, episodes={int(out['episodes'].sum())}")


if __name__ == "__main__":
    for n, s in CONFIGS.items():
        make(n, s)
