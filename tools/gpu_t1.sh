mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t1_pytest.log
tail -3 gpurun_out/t1_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t1_bench.json 2> gpurun_out/t1_bench.err; cat gpurun_out/t1_bench.json | head -c 600; echo
timeout 900 python tools/sweep.py --steps 300 --out gpurun_out/t1_sweep.json > gpurun_out/t1_sweep.log 2>&1
python -c "
import json
for r in json.load(open('gpurun_out/t1_sweep.json')):
  print(r['sweep'],r['agents'],r['envs'],r['obs'],'%.2f'%r['single_step']['us_per_step'] if 'single_step' in r else r.get('ms_per_step'), '%.2f'%r.get('run_multistep',{}).get('us_per_step',0))
" 2>&1 | tail -20
timeout 300 ncu --set full --clock-control none --import-source on -s 3 -c 1 -k regex:tag_env -o gpurun_out/a100p -f python tools/profile_cfg.py 5 2000 num_taggers=20 num_runners=80 obs_mode=1 k_nearest=5 > gpurun_out/a100p.log 2>&1; tail -2 gpurun_out/a100p.log
