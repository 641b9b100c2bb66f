timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"
timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/sweep_r01.json 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['sweep'], d['agents'], d['envs'], d['obs'], round(d['env_steps_per_s']), round(d['ms_per_step'],4))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 200 --warmup 5 --e2e-steps 5 --same-device 2>&1 | tail -2 | cut -c1-600
