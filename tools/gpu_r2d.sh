mkdir -p gpurun_out
timeout 300 python bench.py --steps 50 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
echo rc=$?; tail -30 gpurun_out/r2d_bench.err; cat gpurun_out/r2d_bench.json
