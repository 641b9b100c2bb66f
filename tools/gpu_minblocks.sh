#!/bin/bash
# C2 bench per discrete min-blocks build (register cap 64 at 4, 80 at 3)
for mb in 3 4; do
  make -C paper_2108_13976_b200/csrc clean > /dev/null
  make -C paper_2108_13976_b200/csrc -j16 EXTRA="-DWDG_MIN_BLOCKS_DISCRETE=$mb" > /dev/null 2>&1 || { echo "build $mb failed"; continue; }
  r=$(timeout 300 python bench.py --steps 1000 --warmup 20 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step']*1e3,1), round(d['run_multistep']['env_steps_per_s']/1e6,3))")
  echo "min_blocks_discrete=$mb -> $r"
done
