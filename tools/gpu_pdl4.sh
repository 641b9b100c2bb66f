#!/bin/bash
echo "--- early trigger, forced on"; WDG_PDL=1 timeout 300 python tools/time_cfgs.py d300 d500 c2 c4
echo "--- late trigger, forced on"; WDG_PDL=1 WDG_PDL_LATE=1 timeout 300 python tools/time_cfgs.py d300 d500 c2 c4
echo "--- off"; WDG_PDL=0 timeout 300 python tools/time_cfgs.py d300 d500 c2 c4
