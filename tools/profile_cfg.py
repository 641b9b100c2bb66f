"""Single-step fused launches of an arbitrary Tag config for ncu:
  python tools/profile_cfg.py STEPS ENVS key=value ...   (TagConfig fields)
Launch 0 = registration; launches 1..STEPS = RolloutDriver::step."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13976_b200 as W
steps, envs = int(sys.argv[1]), int(sys.argv[2])
kw = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    kw[k] = float(v) if "." in v else int(v)
cfg = W.TagConfig(**kw)
ws = W.Workspace(cfg, envs)
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, cfg.seed)
for _ in range(steps):
    drv.step()
ws.store.synchronize()
print("done", ws.plan.geometry())
