#!/bin/bash
export WDG_NO_MULTISTEP=1
timeout 600 python - <<PY
import sys, os
sys.path.insert(0, os.getcwd())
from tools.sweep import measure
import paper_2108_13976_b200 as W
cfg = W.TagConfig(num_taggers=200, num_runners=800, obs_mode=W.PARTIAL, k_nearest=5)
for rep in range(2):
    for g in (False, True):
        sps, ms, geo = measure(cfg, 2000, 400, warmup=10, graphs=g)
        print("graphs=%s: %.2fM %.1f us" % (g, sps / 1e6, ms * 1e3))
PY
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
