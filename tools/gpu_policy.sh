#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_policy.py -m gpu -x -q > gpurun_out/${TAG}_pytest_policy.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_policy.log
tail -30 gpurun_out/${TAG}_pytest_policy.log
timeout 600 python tools/policy_bench.py 30 0 2>&1 | tail -5
