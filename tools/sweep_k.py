"""K (k_nearest) sweep at the C2 shape (2000 envs x 1000 agents, discrete,
partial obs): per-step launches (RolloutDriver::step, overlapped) and the
roofline fraction of SURVEY §8(d)'s algorithmic bytes.
  python tools/sweep_k.py [--out profiles/sweep_k_r01.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402
from tools.sweep import algo_bytes, hbm_peak  # noqa: E402

rows = []
for K in (1, 3, 5, 8, 12, 20, 32):
    cfg = W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL, k_nearest=K)
    st = torch.cuda.current_stream()
    ws = W.Workspace(cfg, 2000, stream=st)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
    for _ in range(5):
        drv.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(200):
        drv.step()
    e1.record(st)
    torch.cuda.synchronize()
    drv.check()
    ms = e0.elapsed_time(e1) / 200
    sps = 2000 / (ms / 1e3)
    row = dict(k_nearest=K, obs_dim=cfg.obs_dim(), us_per_step=ms * 1e3, env_steps_per_s=sps,
               hbm_frac=sps * algo_bytes(cfg) / 1e9 / hbm_peak(), geometry=ws.plan.geometry())
    rows.append(row)
    print(json.dumps(row), flush=True)
    ws.close()
if "--out" in sys.argv:
    json.dump(rows, open(sys.argv[sys.argv.index("--out") + 1], "w"), indent=1)
