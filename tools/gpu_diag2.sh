python tools/diag_one.py 8 2>&1 | tail -12
compute-sanitizer --tool memcheck python tools/diag_one.py 8 2>&1 | grep -v "^ dev\|^ ora" | head -40
compute-sanitizer --tool racecheck --racecheck-report hazard python tools/diag_one.py 8 2>&1 | grep -v "^ dev\|^ ora" | head -40
