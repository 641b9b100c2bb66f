"""A few fused steps (with resets) of every kernel layout, small E, for
compute-sanitizer (memcheck / racecheck / synccheck):
  compute-sanitizer --tool racecheck python tools/sanitize_cfgs.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13976_b200 as W  # noqa: E402

D, C, P, F = W.DISCRETE, W.CONTINUOUS, W.PARTIAL, W.FULL
SHAPES = [  # (variant, taggers, runners, obs, K, grid/world, envs)
    (D, 1, 4, F, 5, 20, 7),        # packed, full obs
    (D, 3, 20, P, 5, 20, 9),       # packed brute K-NN
    (D, 20, 80, P, 5, 20, 3),      # brute, 2 envs per CTA
    (D, 30, 120, P, 5, 20, 2),     # one-env brute CTA with idle lanes
    (D, 40, 160, P, 5, 20, 2),     # lattice cells, 128 threads
    (D, 50, 200, P, 5, 30, 2),     # ring search
    (D, 200, 800, P, 5, 20, 2),    # C2 layout (TMA bulk, 256 threads)
    (D, 20, 80, F, 5, 10, 2),      # grid, full obs
    (D, 3, 30, P, 20, 50, 3),      # K=20 brute
    (C, 1, 4, F, 5, 20.0, 5),      # continuous packed full
    (C, 20, 80, P, 5, 10.0, 3),    # continuous brute
    (C, 60, 240, P, 5, 12.0, 2),   # continuous ring
    (C, 200, 800, P, 5, 20.0, 2),  # continuous ring, half-warp staging
    (C, 80, 320, P, 12, 16.0, 2),  # continuous K=12
    (D, 2, 8, F, 5, 8, 13),        # SMALL: 3 envs per warp, partial last warp
]
for var, t, r, obs, k, g, envs in SHAPES:
    kw = dict(variant=var, num_taggers=t, num_runners=r, obs_mode=obs, k_nearest=k, episode_length=4, seed=3)
    if var == D:
        kw["grid_size"] = g
    else:
        kw["world_length"] = g
    cfg = W.TagConfig(**kw)
    ws = W.Workspace(cfg, envs)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 1)
    for _ in range(6):
        drv.step()
    drv.run(6)
    ws.store.synchronize()
    drv.check()
    print("ok", var, t + r, obs, k, ws.plan.geometry(), flush=True)
    ws.close()

# the device TagReference twin (unfused sample -> run_step -> auto_reset)
for var, t, r, obs, g in ((D, 3, 20, P, 8), (D, 20, 80, F, 10), (C, 10, 40, P, 10.0)):
    kw = dict(variant=var, num_taggers=t, num_runners=r, obs_mode=obs, k_nearest=5, episode_length=4, seed=3)
    kw["grid_size" if var == D else "world_length"] = g
    cfg = W.TagConfig(**kw)
    ws = W.Workspace(cfg, 3, reference=True)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 1)
    for _ in range(6):
        drv.step()
    ws.store.synchronize()
    drv.check()
    print("ok twin", var, t + r, obs, flush=True)
    ws.close()

# the pipelined host step (env-range launches) with observations
import numpy as np  # noqa: E402
cfg = W.TagConfig(num_taggers=20, num_runners=80, obs_mode=P, k_nearest=5, episode_length=4, seed=3)
ws = W.Workspace(cfg, 7)
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 1)
drv.set_host_chunks(3)
lg = np.zeros((7, 100, 1, 5))
rw, dn, ob = np.zeros((7, 100), np.float32), np.zeros(7, np.uint8), np.zeros((7, 100, cfg.obs_dim()), np.float32)
for _ in range(6):
    drv.step_host(lg, lg.size, rw, dn, ob, ob.size)
    ws.store.synchronize()
drv.check()
print("ok step_host", flush=True)
ws.close()
