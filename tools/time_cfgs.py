"""Device-timed env-steps/s for a few Tag shapes (single-step launches and
run() windows): python tools/time_cfgs.py [shape ...]   shapes: name=var,A,K,envs"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.sweep import measure  # noqa: E402
import paper_2108_13976_b200 as W  # noqa: E402

SHAPES = {
    "c2": (W.DISCRETE, 1000, 5, 2000), "d500": (W.DISCRETE, 500, 5, 2000), "d100": (W.DISCRETE, 100, 5, 2000),
    "c1000": (W.CONTINUOUS, 1000, 5, 2000), "c300": (W.CONTINUOUS, 300, 5, 2000),
    "c100": (W.CONTINUOUS, 100, 5, 2000), "c150": (W.CONTINUOUS, 150, 5, 2000), "c20": (W.CONTINUOUS, 20, 5, 2000), "c20f": (W.CONTINUOUS, 20, 0, 2000), "d20": (W.DISCRETE, 20, 5, 2000),
    "d200": (W.DISCRETE, 200, 5, 2000), "d300": (W.DISCRETE, 300, 5, 2000), "d700": (W.DISCRETE, 700, 5, 2000), "d600": (W.DISCRETE, 600, 5, 2000),
    "c500": (W.CONTINUOUS, 500, 5, 2000),
    "c2_e1776": (W.DISCRETE, 1000, 5, 1776), "c2_e2368": (W.DISCRETE, 1000, 5, 2368),
    "c2_e1184": (W.DISCRETE, 1000, 5, 1184), "c2_e4000": (W.DISCRETE, 1000, 5, 4000),
    "d100f": (W.DISCRETE, 100, 0, 2000), "c4": (W.DISCRETE, 5, 0, 2000), "d500f": (W.DISCRETE, 500, 0, 400),
    "c4_e10000": (W.DISCRETE, 5, 0, 10000), "c4_e1": (W.DISCRETE, 5, 0, 1), "d10": (W.DISCRETE, 10, 5, 2000),
    "d10f": (W.DISCRETE, 10, 0, 2000), "c5f": (W.CONTINUOUS, 5, 0, 2000),
}
for name in (sys.argv[1:] or list(SHAPES)):
    var, A, K, E = SHAPES[name]
    T = round(A / 5)
    if A == 5:
        T = 1
    cfg = W.TagConfig(variant=var, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL if K else W.FULL,
                      k_nearest=K or 5)
    W.set_tuning("multistep", 0)
    sps1, ms1, _ = measure(cfg, E, 200, warmup=5)
    W.set_tuning("multistep", -1)
    sps2, ms2, _ = measure(cfg, E, 200, warmup=5)
    # RolloutDriver::step loop (the bench's per-step launches)
    import torch
    st = torch.cuda.current_stream()
    ws = W.Workspace(cfg, E, stream=st)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, cfg.seed)
    for _ in range(5):
        drv.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(200):
        drv.step()
    e1.record(st)
    torch.cuda.synchronize()
    ms3 = e0.elapsed_time(e1) / 200
    ws.close()
    print(f"{name}: graph {ms1 * 1e3:.1f} us/step ({sps1 / 1e6:.2f}M)  run {ms2 * 1e3:.1f} us/step "
          f"({sps2 / 1e6:.2f}M)  step {ms3 * 1e3:.1f} us/step ({E / ms3 / 1e3:.2f}M)", flush=True)
