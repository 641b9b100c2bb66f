"""Policy rollout at C2 for ncu: 20 uniform steps, then `steps` bf16 policy
steps (tagger + runner policy launches per step).
  ncu -k regex:policy_bf16 -s 5 -c 1 python tools/profile_policy.py 4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL, k_nearest=5, seed=0)
ws = W.Workspace(cfg, 2000, stream=torch.cuda.current_stream())
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
drv.run(20)
drv.set_policies(W.Policy.for_tag(cfg, seed=1), W.Policy.for_tag(cfg, seed=2), W.POLICY_BF16)
drv.run(steps)
torch.cuda.synchronize()
drv.check()
ws.close()
