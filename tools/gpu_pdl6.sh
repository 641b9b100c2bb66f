#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python tools/policy_bench.py 50 1 2>&1 | tail -1
WDG_NO_PDL=1 timeout 200 python tools/policy_bench.py 50 1 2>&1 | tail -1
