"""Phase ablation at C2 or (ABLATE_CONT=1) continuous, ABLATE_A agents, 2000 envs (performance analysis only; results are WRONG with
WDG_ABLATE != 0): ms per fused step with phases skipped.
  python tools/ablate.py [steps]   (bits: 1 sampler, 2 cell K-NN, 4 obs rows, 8 grid build)"""
import os
import subprocess
import sys

if len(sys.argv) > 2 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tools.sweep import measure
    import paper_2108_13976_b200 as W
    var = W.CONTINUOUS if os.environ.get("ABLATE_CONT") else W.DISCRETE  # ABLATE_CONT=1: continuous
    A = int(os.environ.get("ABLATE_A", "1000"))  # agents per env (taggers = A / 5)
    cfg = W.TagConfig(variant=var, num_taggers=A // 5, num_runners=A - A // 5, obs_mode=W.PARTIAL, k_nearest=5,
                      seed=0)
    sps, ms, geo = measure(cfg, 2000, int(sys.argv[2]), warmup=10, graphs=False, check=False)
    print(f"{sps:.0f} {ms:.4f}")
    sys.exit(0)
steps = sys.argv[1] if len(sys.argv) > 1 else "1000"
for ab in (0, 1, 2, 4, 8, 1 | 2 | 4 | 8):
    env = dict(os.environ, WDG_ABLATE=str(ab))
    r = subprocess.run([sys.executable, __file__, "--one", steps], env=env, capture_output=True, text=True)
    print(f"ablate={ab:2d}: {r.stdout.strip() or r.stderr.strip()[-300:]}", flush=True)
