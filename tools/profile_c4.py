"""C4 (5 agents, full obs) fused steps for ncu: python tools/profile_c4.py ENVS STEPS [graphs]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13976_b200 as W
envs, steps = int(sys.argv[1]), int(sys.argv[2])
cfg = W.TagConfig(num_taggers=1, num_runners=4)
ws = W.Workspace(cfg, envs)
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
drv.set_graphs(len(sys.argv) > 3 and sys.argv[3] == "1")
drv.run(steps)
ws.store.synchronize()
