for ab in 0 1 2 4 6 7 15; do
  r=$(WDG_ABLATE=$ab timeout 300 python bench.py --steps 1000 --warmup 20 --e2e-steps 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4))" 2>&1)
  echo "ablate=$ab -> $r"
done
timeout 1200 python tools/sweep.py --steps 300 --out gpurun_out/sweep_r01.json 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['sweep'], d['agents'], d['envs'], d['obs'], round(d['env_steps_per_s']), round(d['ms_per_step'],4), 'hbm', round(d['hbm_frac'],3))"
