#!/bin/bash
# Repeat the overlap / graph / fused parity tests to shake out ordering races.
for i in $(seq 1 8); do
  timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "overlapped or graph_replay or fused_rollout or headline or multistep" 2>&1 | tail -1
done
timeout 600 python -m pytest tests/test_trig.py -q -x -m gpu 2>&1 | tail -1
