#!/bin/bash
# sweep (single-step graphs) for the product build vs a variant: tools/gpu_sweep_ab.sh VARIANT
mkdir -p gpurun_out
export WDG_NO_MULTISTEP=1
timeout 900 python tools/sweep.py --steps 200 --out gpurun_out/swab_main.json > /dev/null 2>&1
WDG_LIB_VARIANT=$1 timeout 900 python tools/sweep.py --steps 200 --out gpurun_out/swab_var.json > /dev/null 2>&1
python - <<PY
import json
a=json.load(open('gpurun_out/swab_main.json')); b=json.load(open('gpurun_out/swab_var.json'))
for r,q in zip(a,b):
    print(r['sweep'], r['agents'], r['envs'], r['obs'], 'main %.2fus' % (r['ms_per_step']*1e3), '$1 %.2fus' % (q['ms_per_step']*1e3))
PY
