"""Continuous partial (K=5) µs/step with the exact and the keyed ring search
(tuning key cont_keys) over agent counts, 2000 envs, single-step launches.
  python tools/keys_scan.py [A ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402


def time_a(A, keys, E=2000, steps=100):
    W.set_tuning("cont_keys", keys)
    T = round(A / 5)
    cfg = W.TagConfig(variant=W.CONTINUOUS, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL, k_nearest=5)
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
    drv.check()
    ws.close()
    W.set_tuning("cont_keys", -1)
    return e0.elapsed_time(e1) * 1e3 / steps


for A in [int(x) for x in sys.argv[1:]] or [240, 300, 400, 500, 600, 700, 800, 1000]:
    r = [time_a(A, k) for k in (0, 1, 0, 1)]
    print(f"A={A}: exact {min(r[0], r[2]):.1f}  keyed {min(r[1], r[3]):.1f} us/step", flush=True)
