#!/bin/bash
# parity tests + single-step and run() sweeps merged into gpurun_out/${TAG}_sweep.json
TAG=${1:-cur}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
WDG_NO_MULTISTEP=1 timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep_single.json > gpurun_out/${TAG}_sweep_single.log 2>&1
timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep_run.json > gpurun_out/${TAG}_sweep_run.log 2>&1
python tools/merge_sweeps.py gpurun_out/${TAG}_sweep_single.json gpurun_out/${TAG}_sweep_run.json gpurun_out/${TAG}_sweep.json
