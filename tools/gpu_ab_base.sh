#!/bin/bash
# Full GPU suite, then time_cfgs.py shapes for the product build and lib/variants/base
# (tools/build_variant.sh base PATCH.py). usage: tools/gpu_ab_base.sh TAG "shape ..."
TAG=$1; SH=$2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for v in main base; do
  if [ $v == main ]; then timeout 300 python tools/time_cfgs.py $SH 2>&1 | cut -c1-200;
  else WDG_LIB_VARIANT=base timeout 300 python tools/time_cfgs.py $SH 2>&1 | cut -c1-200; fi
done > gpurun_out/${TAG}_ab.log
cat gpurun_out/${TAG}_ab.log
