#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/sweep_k.py --out gpurun_out/sweep_k.json | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('K=%d D=%d %.1f us %.2fM frac %.3f smem %d' % (d['k_nearest'], d['obs_dim'], d['us_per_step'], d['env_steps_per_s']/1e6, d['hbm_frac'], d['geometry']['smem_bytes']))"
