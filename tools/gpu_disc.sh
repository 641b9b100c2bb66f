#!/bin/bash
for g in 0 5 7 10 20; do
if [ $g == 0 ]; then unset WDG_DISC_GC; else export WDG_DISC_GC=$g; fi
timeout 600 python - <<PY
import sys, os
sys.path.insert(0, os.getcwd())
from tools.sweep import measure
import paper_2108_13976_b200 as W
for A in (100, 500):
    T = round(A / 5)
    cfg = W.TagConfig(num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL, k_nearest=5)
    sps, ms, geo = measure(cfg, 2000, 200, warmup=5, graphs=False)
    print("gc=$g A=%d partial: %.2fM env-steps/s %.1f us/step" % (A, sps / 1e6, ms * 1e3))
PY
done
