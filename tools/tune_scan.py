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
    # re-tuning after the K-NN changes: lattice vs brute, thread caps, staging rows
    ("disc100", (W.DISCRETE, 100, 5, 2000), "combo", [None, {"brute_max": 64}]),
    ("disc128", (W.DISCRETE, 128, 5, 2000), "combo", [None, {"brute_max": 64}, {"brute_max": 256}]),
    ("disc160", (W.DISCRETE, 160, 5, 2000), "combo", [None, {"brute_max": 64}, {"brute_max": 256}]),
    ("disc200", (W.DISCRETE, 200, 5, 2000), "combo", [None, {"brute_max": 256}]),
    ("cont300", (W.CONTINUOUS, 300, 5, 2000), "combo", [None, {"threads_per_env_max": 192}, {"stage_rows": 32}]),
    ("cont400", (W.CONTINUOUS, 400, 5, 2000), "combo", [None, {"threads_per_env_max": 192}]),
    ("cont1000", (W.CONTINUOUS, 1000, 5, 2000), "combo", [None, {"stage_rows": 32}]),
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
