#!/bin/bash
# Full GPU suite, then tools/run_scan.py's default-plan rows (SMALL-kernel shapes) for the
# product build and lib/variants/base, two alternating reps. usage: tools/gpu_ab_small.sh TAG
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
for rep in 1 2; do for v in main base; do
  if [ $v == main ]; then timeout 300 python tools/run_scan.py 2>&1 | grep -E "=8:" | sed "s/^/$v /";
  else WDG_LIB_VARIANT=base timeout 300 python tools/run_scan.py 2>&1 | grep -E "=8:" | sed "s/^/$v /"; fi
done; done
