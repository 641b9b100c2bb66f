#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python - <<PY
import sys, os
sys.path.insert(0, os.getcwd())
import paper_2108_13976_b200 as W
for A in (300, 1000):
    T = round(A / 5)
    cfg = W.TagConfig(variant=W.CONTINUOUS, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL, k_nearest=5)
    ws = W.Workspace(cfg, 64); print(A, ws.plan.geometry()); ws.close()
PY
timeout 900 python tools/time_cfgs.py c1000 c300 c100
