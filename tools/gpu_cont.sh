#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python - <<PY
import sys, os
sys.path.insert(0, os.getcwd())
from tools.sweep import measure
import paper_2108_13976_b200 as W
for A in (100, 1000):
    T = round(A / 5)
    cfg = W.TagConfig(variant=W.CONTINUOUS, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL, k_nearest=5)
    sps, ms, geo = measure(cfg, 2000, 100, warmup=5, graphs=False)
    print("continuous A=%d partial: %.2fM env-steps/s %.1f us/step" % (A, sps / 1e6, ms * 1e3))
PY
