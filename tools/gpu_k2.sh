#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
WDG_STAGE_HALF_WARP=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_trig.py -m gpu -x -q -k "k8 or k3 or 7x100 or fused_rollout" 2>&1 | tail -1
timeout 600 python tools/sweep_k.py --out gpurun_out/sweep_k.json | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('K=%d D=%d %.1f us %.2fM frac %.3f smem %d' % (d['k_nearest'], d['obs_dim'], d['us_per_step'], d['env_steps_per_s']/1e6, d['hbm_frac'], d['geometry']['smem_bytes']))"
echo "--- full-warp staging forced"; WDG_STAGE_FULL_WARP=1 timeout 600 python tools/sweep_k.py | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('K=%d %.1f us smem %d' % (d['k_nearest'], d['us_per_step'], d['geometry']['smem_bytes']))" | head -4
