"""Scan plan tuning keys (wdg_set_tuning) on a few shapes: single-step
launches, device-timed.  python tools/tune_scan.py
Each line: shape, key=value, us/step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402


def time_shape(var, A, K, E, steps=100):
    T = round(A / 5)
    cfg = W.TagConfig(variant=var, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL if K else W.FULL,
                      k_nearest=K or 5)
    st = torch.cuda.current_stream()
    ws = W.Workspace(cfg, E, stream=st)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, cfg.seed)
    for _ in range(5):
        drv.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        drv.step()
    e1.record(st)
    torch.cuda.synchronize()
    geo = ws.plan.geometry()
    ws.close()
    return e0.elapsed_time(e1) * 1e3 / steps, geo


SCANS = [
    # discrete lattice shapes after the paired key insertion (thread cap per env)
    ("disc500", (W.DISCRETE, 500, 5, 2000), "combo", [None, {'threads_per_env_max': 128}, {'threads_per_env_max': 160}]),
    ("disc600", (W.DISCRETE, 600, 5, 2000), "combo", [None, {'threads_per_env_max': 128}, {'threads_per_env_max': 160}]),
    ("disc700", (W.DISCRETE, 700, 5, 2000), "combo", [None, {'threads_per_env_max': 128}, {'threads_per_env_max': 160}]),
    ("disc800", (W.DISCRETE, 800, 5, 2000), "combo", [None, {'threads_per_env_max': 128}, {'threads_per_env_max': 160}]),
    ("disc900", (W.DISCRETE, 900, 5, 2000), "combo", [None, {'threads_per_env_max': 128}, {'threads_per_env_max': 160}]),
    ("cont500", (W.CONTINUOUS, 500, 5, 2000), "combo", [None, {"threads_per_env_max": 128}]),
    ("cont700", (W.CONTINUOUS, 700, 5, 2000), "combo", [None, {"threads_per_env_max": 128}, {"threads_per_env_max": 192}]),
    ("cont1000", (W.CONTINUOUS, 1000, 5, 2000), "combo", [None, {"threads_per_env_max": 128}, {"threads_per_env_max": 192}]),
]
for name, shape, key, vals in SCANS:
    for v in vals:
        if key == "combo":
            for k2, v2 in (v or {}).items():
                W.set_tuning(k2, v2)
        else:
            W.set_tuning(key, v)
        try:
            us, geo = time_shape(*shape)
            print(f"{name} {key}={v}: {us:.1f} us/step  threads={geo['threads_per_cta']} smem={geo['smem_bytes']}",
                  flush=True)
        except Exception as exc:
            print(f"{name} {key}={v}: failed {exc}", flush=True)
        W.set_tuning("reset")
