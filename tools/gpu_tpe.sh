#!/bin/bash
for t in 192 160; do
echo "WDG_TPE_MAX=$t"; WDG_TPE_MAX=$t timeout 600 python tools/time_cfgs.py d500 d700 c2 c500 c300
done
