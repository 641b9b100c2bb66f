nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 300 python bench.py --steps 1000 --warmup 20 --e2e-steps 100 --cpu-steps 200 2>&1 | tail -2
WDG_TPE_MAX=512 timeout 300 python bench.py --steps 1000 --warmup 20 --e2e-steps 20 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:tag_env_kernel -s 6 -c 1 -o gpurun_out/prof_c2_v2 python tools/profile_c2.py 8 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
