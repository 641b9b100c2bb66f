#!/bin/bash
TAG=$1
mkdir -p gpurun_out
for v in 0 1; do
  if [ $v == 1 ]; then export WDG_NO_MULTISTEP=1; fi
  timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep_nm$v.json > /dev/null 2>&1
done
python - <<PY
import json
a=json.load(open('gpurun_out/${TAG}_sweep_nm0.json')); b=json.load(open('gpurun_out/${TAG}_sweep_nm1.json'))
for r,q in zip(a,b):
    print(r['sweep'], r['agents'], r['envs'], r['obs'], 'multi %.2fus' % (r['ms_per_step']*1e3), 'single %.2fus' % (q['ms_per_step']*1e3), r['geometry']['grid_ctas'], r['geometry']['threads_per_cta'], r['geometry']['smem_bytes'])
PY
