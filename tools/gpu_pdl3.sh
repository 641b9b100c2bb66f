#!/bin/bash
timeout 400 python tools/time_cfgs.py d200 d700 d100f c4 d500f
echo "--- WDG_TPE_MAX=256"; WDG_TPE_MAX=256 timeout 300 python tools/time_cfgs.py d300 d500
echo "--- no pdl"; WDG_NO_PDL=1 timeout 400 python tools/time_cfgs.py d200 d700 d100f c4 d500f
