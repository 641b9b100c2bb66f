#!/bin/bash
for d in 2 3 4 5; do echo "WDG_CONT_GC_DIV=$d"; WDG_CONT_GC_DIV=$d timeout 300 python tools/time_cfgs.py c300 c500 c1000; done
