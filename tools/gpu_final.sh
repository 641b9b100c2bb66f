#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 200 --warmup 5 --e2e-steps 20 --same-device > gpurun_out/${TAG}_bench2.json 2> gpurun_out/${TAG}_bench2.err
echo "N=2 same-device:"; cat gpurun_out/${TAG}_bench2.json | head -c 700; echo; tail -2 gpurun_out/${TAG}_bench2.err
timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1
WDG_NO_MULTISTEP=1 timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep_single.json > /dev/null 2>&1
python - <<PY
import json
a=json.load(open('gpurun_out/${TAG}_sweep.json')); b=json.load(open('gpurun_out/${TAG}_sweep_single.json'))
for r,q in zip(a,b):
    print(r['sweep'], r['agents'], r['envs'], r['obs'], 'run %.2fus' % (r['ms_per_step']*1e3), 'single %.2fus' % (q['ms_per_step']*1e3), '%.2fM' % (q['env_steps_per_s']/1e6))
PY
