"""run() and single-step µs/step of a few shapes under tuning keys (A/B of
plan choices on the launch path the sweeps time).
  python tools/run_scan.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.sweep import measure  # noqa: E402
import paper_2108_13976_b200 as W  # noqa: E402

SCANS = [
    ("c4 2000", (W.DISCRETE, 5, 0, 2000), "packed_warps_max", [8, 4, 2, 1]),
    ("c4 10000", (W.DISCRETE, 5, 0, 10000), "packed_warps_max", [8, 4, 2, 1]),
    ("c4 100", (W.DISCRETE, 5, 0, 100), "packed_warps_max", [8, 2, 1]),
    ("disc10 part", (W.DISCRETE, 10, 5, 2000), "packed_warps_max", [8, 4, 2, 1]),
    ("disc10 full", (W.DISCRETE, 10, 0, 2000), "packed_warps_max", [8, 4, 2, 1]),
    ("cont5 full", (W.CONTINUOUS, 5, 0, 2000), "packed_warps_max", [8, 4, 2, 1]),
]
for name, (var, A, K, E), key, vals in SCANS:
    T = 1 if A == 5 else round(A / 5)
    cfg = W.TagConfig(variant=var, num_taggers=T, num_runners=A - T, obs_mode=W.PARTIAL if K else W.FULL,
                      k_nearest=K or 5)
    for v in vals:
        W.set_tuning(key, v)
        W.set_tuning("multistep", 0)
        _, ms1, geo = measure(cfg, E, 200, warmup=5)
        W.set_tuning("multistep", -1)
        _, ms2, _ = measure(cfg, E, 200, warmup=5)
        print(f"{name} {key}={v}: single {ms1 * 1e3:.2f} run {ms2 * 1e3:.2f} us/step  "
              f"threads={geo['threads_per_cta']} envs_per_cta={geo['envs_per_cta']}", flush=True)
        W.set_tuning("reset")
