#!/bin/bash
# full round + single-step and run() sweeps
TAG=$1
bash tools/gpu_round.sh $TAG > /dev/null 2>&1
WDG_NO_MULTISTEP=1 timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep_single.json > /dev/null 2>&1
timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep_run.json > /dev/null 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_smoke.log; tail -1 gpurun_out/${TAG}_ncu_full.log
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(d['value'], d['roofline']['frac'], d['run_multistep']['env_steps_per_s'], d['policy_rollout']['env_steps_per_s'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
