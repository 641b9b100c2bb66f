#!/bin/bash
# usage: tools/gpu_var.sh TAG variant...   (parity tests on the product build, then variant timings)
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python tools/variants.py 1000 main "$@" | tee gpurun_out/${TAG}_variants.txt
timeout 600 python tools/ablate.py 1000 | tee gpurun_out/${TAG}_ablate.txt
