#!/bin/bash
# A/B the bf16 policy rollout (bench.py policy leg) between the product build and variants
for rep in 1 2 3; do
  for v in main "$@"; do
    if [ "$v" == "main" ]; then env=""; else env="WDG_LIB_VARIANT=$v"; fi
    out=$(env $env timeout 300 python tools/policy_bench.py 200 1 2>&1 | tail -2 | tr '\n' ' ')
    echo "rep$rep $v: $out"
  done
done
