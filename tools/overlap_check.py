"""Full-size ordering check (GPU): the C2 shape stepped N times with
overlapped launches (programmatic dependent launch) vs serial launches;
every store array must match bit for bit.  python tools/overlap_check.py [N]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13976_b200 as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
cfg = W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL, k_nearest=5, episode_length=40, seed=7)
ws1 = W.Workspace(cfg, 2000)
d1 = W.RolloutDriver(ws1.store, ws1.plan, ws1.resets, 3)
ws2 = W.Workspace(cfg, 2000)
d2 = W.RolloutDriver(ws2.store, ws2.plan, ws2.resets, 3)
d2.set_overlap(False)
for d in (d1, d2):
    for _ in range(n):
        d.step()
    d.run(n)
names = ["loc_x", "loc_y", "is_tagger", "active", "was_tagged", "tag_credits", "rewards", "observations",
         "sampled_actions", "step_count", "done"]
bad = [k for k in names if not np.array_equal(ws1.store.pull(k), ws2.store.pull(k))]
print("overlap check", n, "steps + run(", n, "):", "MISMATCH " + str(bad) if bad else "identical",
      "stats equal:", bool(np.array_equal(d1.stats(), d2.stats())))
sys.exit(1 if bad else 0)
