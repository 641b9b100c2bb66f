#!/bin/bash
mkdir -p gpurun_out
for v in cbeaf1ed main; do
  if [ $v == main ]; then unset WDG_LIB_VARIANT; else export WDG_LIB_VARIANT=$v; fi
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:tag_env -s 6 -c 1 -o gpurun_out/ab_full_$v python tools/profile_cfg.py 8 2000 num_taggers=20 num_runners=80 obs_mode=0 > /dev/null 2>&1
done
ls gpurun_out/ab_full_*
