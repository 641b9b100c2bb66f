"""Fused C2 launches for ncu.
  python tools/profile_c2.py [steps] [envs] [single|multi]
single (default): registration (launch 0), then `steps` single-step launches
  (RolloutDriver::step) — ncu -s 6 -c 1 profiles the 6th step launch.
multi: registration, a warm-up run(16) (launch 1), then one run(steps)
  multi-step residency launch (launch 2: ncu -s 2 -c 1)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13976_b200 as W
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
envs = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
mode = sys.argv[3] if len(sys.argv) > 3 else "single"
cfg = W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL, k_nearest=5, seed=0)
ws = W.Workspace(cfg, envs)
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
if mode == "multi":
    drv.run(16)
    drv.run(steps)
else:
    for _ in range(steps):
        drv.step()
ws.store.synchronize()
print("done", drv.stats())
