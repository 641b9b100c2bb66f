#!/bin/bash
# Perf iteration call: parity tests, bench, phase ablations, optional sweep.
# usage: tools/gpu_perf.sh TAG [sweep]
TAG=${1:-cur}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 600 python tools/ablate.py 1000 | tee gpurun_out/${TAG}_ablate.txt
if [ "$2" == "sweep" ]; then
  timeout 1500 python tools/sweep.py --steps 300 --out gpurun_out/${TAG}_sweep.json > gpurun_out/${TAG}_sweep.log 2>&1
  tail -20 gpurun_out/${TAG}_sweep.log
fi
