#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1
cat gpurun_out/${TAG}_sweep.log | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()); continue
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items() if k != 'geometry'})"
