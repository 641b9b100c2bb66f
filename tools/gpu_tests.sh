#!/bin/bash
# usage: tools/gpu_tests.sh TAG [pytest args...]
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest "$@" -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -30 gpurun_out/${TAG}_pytest.log
