#!/bin/bash
bash tools/gpu_sweep.sh s6
timeout 300 python tools/time_cfgs.py d200 d300 d500 d700 c2
