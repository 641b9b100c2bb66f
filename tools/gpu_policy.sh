#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_policy.py -m gpu -x -q --timeout 120 > gpurun_out/${TAG}_pytest_policy.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_policy.log
tail -40 gpurun_out/${TAG}_pytest_policy.log
timeout 300 python tools/policy_bench.py 30 1 2>&1 | tail -5
timeout 300 ncu --set full --import-source on --clock-control none -k regex:policy_bf16 -s 2 -c 1 -o gpurun_out/${TAG}_bf16 python tools/policy_bench.py 3 1 > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
