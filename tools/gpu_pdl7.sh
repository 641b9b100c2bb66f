#!/bin/bash
for m in 0 3; do echo "WDG_PDL=$m"; WDG_PDL=$m timeout 300 python tools/time_cfgs.py c4 d100f d100; done
WDG_PDL=3 timeout 300 python -m pytest tests/test_parity_gpu.py -q -k "graph_replay or overlapped or fused_rollout" 2>&1 | tail -1
