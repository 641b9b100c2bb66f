nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
for t in 256 512 1024; do WDG_TPE_MAX=$t timeout 300 python bench.py --steps 1000 --warmup 20 --e2e-steps 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TPE', $t, 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']))"; done
cp paper_2108_13976_b200/lib/libwdg_b200.so gpurun_out/libwdg_b200_profiled.so
ncu --set full --clock-control none --import-source on -k regex:tag_env_kernel -s 6 -c 1 -o gpurun_out/prof_c2_v3 python tools/profile_c2.py 8 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
