#!/bin/bash
# PDL A/B: parity tests (step() launches use PDL), bench with and without, sanitizers
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 0 1; do
  if [ $v == 1 ]; then export WDG_NO_PDL=1; fi
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_pdl=$v', round(d['value']/1e6,3), 'M', round(d['ms_per_step']*1e3,1), 'us', d['roofline']['frac'], d['gpu_launches'])"
done
unset WDG_NO_PDL
bash tools/gpu_sanitize.sh
