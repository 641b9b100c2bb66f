nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r01.json; cat gpurun_out/bench_r01.json
timeout 300 python bench.py --impl reference --steps 300 --warmup 5 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r01_bench.csv python bench.py --steps 20 --warmup 3 --e2e-steps 5 --no-cpu-baseline > /dev/null 2>&1
cp paper_2108_13976_b200/lib/libwdg_b200.so gpurun_out/libwdg_b200_profiled.so
ncu --set full --clock-control none --import-source on -k regex:tag_env_kernel -s 6 -c 1 -o gpurun_out/prof_c2_v4 python tools/profile_c2.py 8 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
