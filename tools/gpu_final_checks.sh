#!/bin/bash
# Final checks: full GPU suite twice, and memcheck / synccheck with every overlap mode forced
for rep in 1 2; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
for m in 0 1 2 3; do
  for tool in memcheck synccheck; do
    r=$(WDG_PDL=$m timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cfgs.py 2>&1 | grep -E "SUMMARY" | tail -1)
    echo "WDG_PDL=$m $tool: $r"
  done
done
