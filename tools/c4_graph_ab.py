"""C4 single-step graph replay µs/step (run() with multi-step windows off), long windows:
  python tools/c4_graph_ab.py [envs ...]   (select the library with WDG_LIB_VARIANT)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.sweep import measure  # noqa: E402
import paper_2108_13976_b200 as W  # noqa: E402

cfg = W.TagConfig(num_taggers=1, num_runners=4)
W.set_tuning("multistep", 0)
out = []
for E in [int(x) for x in sys.argv[1:]] or [1, 2000, 10000]:
    _, ms, _ = measure(cfg, E, 4096, warmup=64)
    out.append(f"E={E} {ms * 1e3:.2f}")
print("  ".join(out), flush=True)
