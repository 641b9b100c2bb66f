#!/bin/bash
for v in main old main; do
  if [ $v == main ]; then unset WDG_LIB_VARIANT; else export WDG_LIB_VARIANT=$v; fi
  WDG_NO_MULTISTEP=1 timeout 600 python - <<PY
import sys, os
sys.path.insert(0, os.getcwd())
from tools.sweep import measure
import paper_2108_13976_b200 as W
for A, mode in ((100, W.FULL), (500, W.FULL), (1000, W.PARTIAL)):
    T = round(A / 5)
    cfg = W.TagConfig(num_taggers=T, num_runners=A - T, obs_mode=mode, k_nearest=5)
    sps, ms, geo = measure(cfg, 2000, 40 if A == 500 else 200, warmup=5, graphs=True)
    print("$v A=%d mode=%d: %.1f us/step" % (A, mode, ms * 1e3))
PY
done
