#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/time_cfgs.py d200 d300 d500 d700 c2 c300 c500 c1000
