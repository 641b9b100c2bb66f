#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/time_cfgs.py c1000 c300
WDG_NO_SXY=1 timeout 900 python tools/time_cfgs.py c1000 c300
