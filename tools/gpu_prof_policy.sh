#!/bin/bash
# ncu --set full of the runner-policy launch of the third policy step at C2:
#   tools/gpu_prof_policy.sh TAG
TAG=$1
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:policy_bf16 -s 5 -c 1 \
  -o gpurun_out/${TAG}_pol python tools/profile_policy.py 4 > gpurun_out/${TAG}_pol.log 2>&1
tail -1 gpurun_out/${TAG}_pol.log
