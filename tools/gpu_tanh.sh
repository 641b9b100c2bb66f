#!/bin/bash
timeout 600 python -m pytest tests/test_policy.py -m gpu -x -q --timeout 120 2>&1 | tail -2
for v in main tp0 tp4; do
  if [ $v == main ]; then unset WDG_LIB_VARIANT; else export WDG_LIB_VARIANT=$v; fi
  echo "variant $v"; timeout 300 python tools/policy_bench.py 40 1 2>&1 | tail -1
done
