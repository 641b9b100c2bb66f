#!/bin/bash
# ncu --set full of the C4 run window (SMALL kernel, 64-step launch) and of the
# continuous A=1000 LEAN step: tools/gpu_prof_final.sh TAG
TAG=$1
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tag_small -s 1 -c 1 \
  -o gpurun_out/${TAG}_c4small python tools/profile_c4.py 2000 192 0 > gpurun_out/${TAG}_c4small.log 2>&1
tail -1 gpurun_out/${TAG}_c4small.log
timeout 600 ncu --set full --clock-control none --import-source on -s 3 -c 1 -k regex:tag_env \
  -o gpurun_out/${TAG}_cont1000 python tools/profile_cfg.py 5 2000 variant=1 num_taggers=200 num_runners=800 \
  obs_mode=1 k_nearest=5 > gpurun_out/${TAG}_cont1000.log 2>&1
tail -1 gpurun_out/${TAG}_cont1000.log
