#!/bin/bash
# A/B: product build vs lib/variants/base at C2 (graph / run / step columns), 2 reps
for rep in 1 2; do
  echo "main:"; timeout 300 python tools/time_cfgs.py c2 | tail -1
  echo "base:"; WDG_LIB_VARIANT=base timeout 300 python tools/time_cfgs.py c2 | tail -1
done
