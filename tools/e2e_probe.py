"""e2e host-path probe at C2: closed-loop / open-loop step_host rates per
env-chunk count (wdg_rollout_set_host_chunks), with and without observations.

  python tools/e2e_probe.py [steps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402
from bench import C2  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
cfg = W.TagConfig(**C2)
E = 2000
A, D = cfg.num_agents(), cfg.obs_dim()
ws = W.Workspace(cfg, E, stream=torch.cuda.current_stream())
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
n = E * A * 5
hl = torch.zeros(n, dtype=torch.float64).pin_memory()
hr = torch.empty(E * A, dtype=torch.float32).pin_memory()
hd = torch.empty(E, dtype=torch.uint8).pin_memory()
ho = torch.empty(E * A * D, dtype=torch.float32).pin_memory()
out = []
for chunks in (1, 2, 4, 8, 16):
    drv.set_host_chunks(chunks)
    for obs in (False, True):
        for closed in (True, False):
            o, no = (ho, E * A * D) if obs else (None, 0)
            for _ in range(5):
                drv.step_host(hl, n, hr, hd, o, no)
            ws.store.synchronize()
            t0 = time.perf_counter()
            for _ in range(steps):
                drv.step_host(hl, n, hr, hd, o, no)
                if closed:
                    ws.store.synchronize()
            ws.store.synchronize()
            dt = time.perf_counter() - t0
            r = {"chunks": chunks, "obs": obs, "closed": closed, "ms_per_step": 1e3 * dt / steps,
                 "env_steps_per_s": E * steps / dt}
            out.append(r)
            print(json.dumps(r), flush=True)
# raw copy rates for reference
dev = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("h2d_80MB", lambda: dev.copy_(hl, non_blocking=True)),
                 ("d2h_80MB", lambda: hl.copy_(dev, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print(json.dumps({"copy": name, "ms": 1e3 * dt, "gbs": n * 8 / dt / 1e9}), flush=True)
ws.close()
