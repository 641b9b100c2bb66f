#!/bin/bash
# A/B the product build against tuning variants (lib/variants/<name>) on one
# box: tools/gpu_ab_variants.sh "shape ..." name1 name2 ...   (3 alternating reps)
SHAPES=$1; shift
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in main "$@"; do
    if [ "$v" == "main" ]; then
      out=$(timeout 300 python tools/time_cfgs.py $SHAPES 2>&1 | tr '\n' ' ')
    else
      out=$(WDG_LIB_VARIANT=$v timeout 300 python tools/time_cfgs.py $SHAPES 2>&1 | tr '\n' ' ')
    fi
    echo "rep$rep $v: $out"
  done
done
