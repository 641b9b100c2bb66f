#!/bin/bash
# Round evidence — tools/gpu_round.sh (tests, smoke, both bench arms,
# launch list, ncu C2) + sweep, then ncu of the continuous A=1000 step
TAG=$1
bash tools/gpu_round.sh $TAG sweep
timeout 600 ncu --set full --clock-control none --import-source on -s 3 -c 1 -k regex:tag_env \
  -o gpurun_out/${TAG}_cont1000 python tools/profile_cfg.py 5 2000 variant=1 num_taggers=200 num_runners=800 \
  obs_mode=1 k_nearest=5 > gpurun_out/${TAG}_cont1000.log 2>&1
tail -1 gpurun_out/${TAG}_cont1000.log
