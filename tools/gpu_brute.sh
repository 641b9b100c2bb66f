#!/bin/bash
# Brute-force vs bucket-grid K-NN crossover (WDG_BRUTE_MAX) and discrete gc.
for v in "64 0" "128 0" "512 0" "64 20" "64 14"; do
read bm g <<< "$v"
export WDG_BRUTE_MAX=$bm
if [ $g == 0 ]; then unset WDG_DISC_GC; else export WDG_DISC_GC=$g; fi
timeout 600 python - <<PY
import sys, os
sys.path.insert(0, os.getcwd())
from tools.sweep import measure
import paper_2108_13976_b200 as W
for var in (W.DISCRETE, W.CONTINUOUS):
  for A in (100, 200, 300, 500):
    if $g and var == W.CONTINUOUS: continue
    T = round(A / 5)
    cfg = W.TagConfig(variant=var, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL, k_nearest=5)
    try:
        sps, ms, geo = measure(cfg, 2000, 200, warmup=5)
    except Exception as e:
        print("brute_max=$bm gc=$g", var, A, "ERR", e); continue
    print("brute_max=$bm gc=$g var=%d A=%d partial: %.2fM env-steps/s %.1f us/step thr=%d grid=%d" % (var, A, sps / 1e6, ms * 1e3, geo['threads_per_cta'], geo['uses_grid']))
PY
done
