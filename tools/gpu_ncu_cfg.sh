#!/bin/bash
# ncu --set full of one fused launch of a Tag config: tools/gpu_ncu_cfg.sh NAME ENVS key=value ...
NAME=$1; shift
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -s 3 -c 1 -k regex:tag_env -o gpurun_out/$NAME -f python tools/profile_cfg.py 5 "$@" > gpurun_out/$NAME.log 2>&1; tail -2 gpurun_out/$NAME.log
