#!/bin/bash
# ncu --set full of the C2 fused kernel (6th step launch): tools/gpu_prof.sh TAG
TAG=$1
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tag_env_kernel -s 6 -c 1 \
  -o gpurun_out/${TAG}_prof_c2 python tools/profile_c2.py 8 > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -1 gpurun_out/${TAG}_ncu_full.log
