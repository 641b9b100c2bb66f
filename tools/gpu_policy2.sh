#!/bin/bash
TAG=$1
mkdir -p gpurun_out
WDG_DEBUG_POLICY=1 timeout 300 python tools/policy_bench.py 30 1 2>&1 | sort | uniq -c | tail -5
timeout 600 python -m pytest tests/test_policy.py -m gpu -x -q --timeout 120 2>&1 | tail -3
timeout 300 ncu --set full --import-source on --clock-control none -k regex:policy_bf16 -s 2 -c 1 -o gpurun_out/${TAG}_bf16 python tools/policy_bench.py 3 1 > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
