#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 400 python tools/time_cfgs.py c2 d500 d300 d100 c1000 c300
