"""Compare tuning builds (paper_2108_13976_b200/lib/variants/<name>) at C2.
  python tools/variants.py STEPS main name1 name2 ...   ('main' = the product build)"""
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
steps = sys.argv[1]
for rep in range(2):
    for v in sys.argv[2:]:
        env = dict(os.environ, WDG_ABLATE="0")
        env.pop("WDG_LIB_VARIANT", None)
        lib, *kv = v.split("+")  # e.g. main+WDG_NO_BULK=1
        if lib != "main":
            env["WDG_LIB_VARIANT"] = lib
        for item in kv:
            k, val = item.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, os.path.join(here, "ablate.py"), "--one", steps], env=env,
                           capture_output=True, text=True)
        print(f"rep{rep} {v:10s}: {r.stdout.strip() or r.stderr.strip()[-300:]}", flush=True)
