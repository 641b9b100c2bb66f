"""Fused steps on non-uniform logits (bench.py's sampler_stress leg) for a few
shapes: python tools/sampler_stress.py [shape ...]  (c2, c1000, c4)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402

SHAPES = {"c2": (W.DISCRETE, 200, 800, W.PARTIAL, 2000), "c1000": (W.CONTINUOUS, 200, 800, W.PARTIAL, 2000),
          "c4": (W.DISCRETE, 1, 4, W.FULL, 2000)}
for name in sys.argv[1:] or list(SHAPES):
    var, T, R, obs, E = SHAPES[name]
    cfg = W.TagConfig(variant=var, num_taggers=T, num_runners=R, obs_mode=obs, k_nearest=5)
    st = torch.cuda.current_stream()
    ws = W.Workspace(cfg, E, stream=st)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, cfg.seed)
    C, V = (2, 3) if var == W.CONTINUOUS else (1, 5)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    lg = torch.randn(E * (T + R) * C * V, dtype=torch.float64, device="cuda", generator=gen) * 3.0
    drv.set_logits(lg, lg.numel())
    drv.run(5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    drv.run(200)
    e1.record(st)
    torch.cuda.synchronize()
    drv.check()
    ms = e0.elapsed_time(e1) / 200
    print(f"{name} stress: {ms * 1e3:.1f} us/step ({E / ms / 1e3:.2f}M)", flush=True)
    ws.close()
