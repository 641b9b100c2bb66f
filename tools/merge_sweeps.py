"""Merge a single-step sweep (WDG_NO_MULTISTEP=1) and a run() sweep of
tools/sweep.py into the profiles/sweep_r01.json layout (one row per shape,
`single_step` and `run_multistep` columns).

  python tools/merge_sweeps.py SINGLE.json RUN.json OUT.json"""
import json
import sys


def col(r):
    return dict(env_steps_per_s=r["env_steps_per_s"], us_per_step=r["ms_per_step"] * 1e3, hbm_frac=r["hbm_frac"])


def main():
    single, run = (json.load(open(f)) for f in sys.argv[1:3])
    out = []
    for a, b in zip(single, run):
        assert (a["sweep"], a["agents"], a["envs"], a["obs"]) == (b["sweep"], b["agents"], b["envs"], b["obs"])
        out.append(dict(sweep=a["sweep"], agents=a["agents"], envs=a["envs"], obs=a["obs"],
                        single_step=col(a), run_multistep=col(b), geometry=a["geometry"]))
    json.dump(out, open(sys.argv[3], "w"), indent=1)
    for r in out:
        print(f'{r["sweep"]:10s} A={r["agents"]:5d} E={r["envs"]:6d} {r["obs"]:8s} '
              f'single {r["single_step"]["us_per_step"]:8.2f} us  run {r["run_multistep"]["us_per_step"]:8.2f} us  '
              f'frac {r["single_step"]["hbm_frac"]:.3f}')


if __name__ == "__main__":
    main()
