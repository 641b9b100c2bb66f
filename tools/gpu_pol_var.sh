#!/bin/bash
for v in main p7r2 p6r2 main; do
  if [ $v == main ]; then unset WDG_LIB_VARIANT; else export WDG_LIB_VARIANT=$v; fi
  echo "variant $v"; WDG_DEBUG_POLICY=1 timeout 300 python tools/policy_bench.py 40 1 2>&1 | sort | uniq -c | tail -2
done
