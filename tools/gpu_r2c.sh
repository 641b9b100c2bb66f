mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu_device.py tests/test_host_path.py -x -q --timeout 600 > gpurun_out/r2c_new.log 2>&1; echo rc=$? >> gpurun_out/r2c_new.log
WDG_LIB_VARIANT=nofix timeout 600 python -m pytest tests/test_host_path.py -q -k "overlap" --timeout 300 > gpurun_out/r2c_nofix.log 2>&1; echo rc=$? >> gpurun_out/r2c_nofix.log
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2c_bench_ref.json 2> gpurun_out/r2c_bench_ref.err
tail -5 gpurun_out/r2c_new.log; tail -8 gpurun_out/r2c_nofix.log; cat gpurun_out/r2c_bench.json; tail -3 gpurun_out/r2c_bench.err; cat gpurun_out/r2c_bench_ref.json
