#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for bm in 0 256; do
if [ $bm == 0 ]; then unset WDG_BRUTE_MAX; else export WDG_BRUTE_MAX=$bm; fi
timeout 600 python - <<PY
import sys, os, time
sys.path.insert(0, os.getcwd())
from tools.sweep import measure
import paper_2108_13976_b200 as W
for var in (W.CONTINUOUS,):
  for A in (100, 160, 200, 256):
    T = round(A / 5)
    t0 = time.time()
    cfg = W.TagConfig(variant=var, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL, k_nearest=5)
    sps, ms, geo = measure(cfg, 2000, 100, warmup=3)
    print("bm=$bm var=%d A=%d partial: %.2fM env-steps/s %.1f us/step thr=%d grid=%d (%.0fs)" % (var, A, sps / 1e6, ms * 1e3, geo['threads_per_cta'], geo['uses_grid'], time.time() - t0), flush=True)
PY
done
