#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/variants.py 1000 main main+WDG_NO_MULTISTEP=1 | tee gpurun_out/${TAG}_variants.txt
timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1
python -c "
import json
for r in json.load(open('gpurun_out/${TAG}_sweep.json')):
    print(r['sweep'], r['agents'], r['envs'], r['obs'], '%.2fM' % (r['env_steps_per_s']/1e6), '%.2fus' % (r['ms_per_step']*1e3), '%.3f' % r['hbm_frac'])
"
