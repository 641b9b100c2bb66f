#!/bin/bash
mkdir -p gpurun_out
for E in 1 2000; do
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,smsp__inst_executed.sum --clock-control none -c 30 --csv python tools/profile_c4.py $E 20 0 2>/dev/null | grep tag_env | tail -3
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tag_env -s 10 -c 1 -o gpurun_out/c4_e2000 python tools/profile_c4.py 2000 20 0 > /dev/null 2>&1
ls gpurun_out/c4_e2000*
