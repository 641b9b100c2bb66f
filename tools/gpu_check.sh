timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"
cp paper_2108_13976_b200/lib/libwdg_b200.so gpurun_out/libwdg_b200_profiled.so
ncu --set full --clock-control none --import-source on -k regex:tag_env_kernel -s 6 -c 1 -o gpurun_out/prof_c2_v6 python tools/profile_c2.py 8 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
