"""Rollout with device policies at C2 (2000 envs x 1000 agents): ms per
policy forward and env-steps/s of forward + fused step, per precision.
  python tools/policy_bench.py [steps] [precisions...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
precs = [int(x) for x in sys.argv[2:]] or [W.POLICY_F64]
cfg = W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL, k_nearest=5, seed=0)
E, A = 2000, 1000
stream = torch.cuda.current_stream()
ws = W.Workspace(cfg, E, stream=stream)
drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, 0)
pt, pr = W.Policy.for_tag(cfg, seed=1), W.Policy.for_tag(cfg, seed=2)
obs = ws.store.device_ptr("observations")
for prec in precs:
    lg = torch.empty((E, A, 5), dtype=torch.float64, device="cuda")
    for _ in range(3):
        pt.forward(obs, E, A, lg, None, 0, A, precision=prec, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        pt.forward(obs, E, A, lg, None, 0, A, precision=prec, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    fwd_ms = e0.elapsed_time(e1) / 10
    drv.set_policies(pt, pr, prec)
    drv.run(3)
    torch.cuda.synchronize()
    e0.record(stream)
    drv.run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    drv.check()
    print(f"precision={prec}: forward {fwd_ms:.3f} ms (2M rows), rollout {ms:.3f} ms/step = "
          f"{E / (ms / 1e3) / 1e6:.3f} M env-steps/s", flush=True)
ws.close()
