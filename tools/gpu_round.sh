#!/bin/bash
# One GPU call: parity tests, smoke, default bench (both arms), launch list,
# one ncu --set full capture of the fused kernel at C2, and (optional) the
# C3/C4 sweep. Outputs under gpurun_out/.   usage: tools/gpu_round.sh TAG [sweep]
TAG=${1:-cur}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-sweep > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tag_env_kernel -s 6 -c 1 \
  -o gpurun_out/${TAG}_prof_c2 python tools/profile_c2.py 8 > gpurun_out/${TAG}_ncu_full.log 2>&1
if [ "$2" == "sweep" ]; then
  timeout 1500 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1
fi
tail -1 gpurun_out/${TAG}_ncu_full.log
cat gpurun_out/${TAG}_bench.json
tail -3 gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_pytest.log
cat gpurun_out/${TAG}_smoke.log
