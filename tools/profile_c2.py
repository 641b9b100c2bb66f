"""Runs a few fused C2 steps (for ncu): python tools/profile_c2.py [steps] [envs]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13976_b200 as W
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
envs = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
cfg = W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL, k_nearest=5, seed=0)
ws = W.Workspace(cfg, envs)
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
drv.run(steps)
ws.store.synchronize()
print("done", drv.stats())
