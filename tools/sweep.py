"""C3 agent sweep and C4 env sweep (BASELINE.json configs[2], configs[3]) on
one GPU: env-steps/s of the fused step, device-timed with CUDA events.

  python tools/sweep.py [--steps K] [--out profiles/sweep_r01.json]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2108_13976_b200 as W  # noqa: E402


def algo_bytes(cfg):
    """SURVEY.md §8(d) algorithmic bytes per env-step (+ continuous speed/dir)."""
    A, C, V, D = cfg.num_agents(), cfg.action_categories(), cfg.action_choices(), cfg.obs_dim()
    cont = 16 if cfg.variant == W.CONTINUOUS else 0
    return A * (8 * C * V + 4 * C + 8 + 8 + cont + 1 + 2 + 4 + 1 + 4 + 4 * D) + 9


def hbm_peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def measure(cfg, envs, steps, warmup=10, graphs=True, check=True):
    stream = torch.cuda.current_stream()
    ws = W.Workspace(cfg, envs, stream=stream)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, cfg.seed)
    drv.set_graphs(graphs)
    drv.run(warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    drv.run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if check:
        drv.check()
    geo = ws.plan.geometry()
    ws.close()
    return envs * steps / (ms / 1e3), ms / steps, geo


def launch_floor(n=2000):
    """The C4 floor: per-launch time of an empty kernel
    (torch.cuda._sleep(0)) launched back to back, and per node of a CUDA graph
    of such nodes (each kernel waits for the previous: the stream order every
    Tag step has)."""
    st = torch.cuda.current_stream()
    for _ in range(50):
        torch.cuda._sleep(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        torch.cuda._sleep(0)
    e1.record(st)
    torch.cuda.synchronize()
    direct = e0.elapsed_time(e1) * 1e3 / n
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            for _ in range(64):
                torch.cuda._sleep(0)
    g.replay()
    torch.cuda.synchronize()
    e0.record(st)
    reps = max(1, n // 64)
    for _ in range(reps):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) * 1e3 / (reps * 64)
    return {"empty_kernel_us": direct, "graph_node_us": graph}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    # C3: agent sweep at 2000 envs, partial K=5, taggers = llround(A/5) (harness.cpp:823-832)
    for A in (10, 100, 500, 1000):
        T = max(1, min(A - 1, round(A / 5)))
        for mode, name in ((W.PARTIAL, "partial"), (W.FULL, "full")):
            cfg = W.TagConfig(num_taggers=T, num_runners=A - T, obs_mode=mode, k_nearest=min(5, A - 1))
            n = args.steps if A <= 500 else max(100, args.steps // 2)
            if mode == W.FULL and A >= 500:
                n = 30  # 8 / 32 GB of observations per step: HBM-bound
            sps, ms, geo = measure(cfg, 2000, n, warmup=3)
            gbs = sps * algo_bytes(cfg) / 1e9
            rows.append(dict(sweep="C3 agents", agents=A, envs=2000, obs=name, env_steps_per_s=sps,
                             ms_per_step=ms, per_env_step_us=1e3 * ms / 2000, algo_GBps=gbs,
                             hbm_frac=gbs / hbm_peak(), geometry=geo))
            print(json.dumps(rows[-1]))
    # C4: env sweep, 5 agents (1 tagger + 4 runners), full obs D=19. The
    # working set fits in L2, so the bound is launch latency: each row also
    # reports the empty-kernel floor and the step's multiple of it.
    floor = launch_floor()
    rows.append(dict(sweep="launch floor", **floor))
    print(json.dumps(rows[-1]))
    for E in (1, 10, 100, 1000, 2000, 5000, 10000):
        cfg = W.TagConfig(num_taggers=1, num_runners=4)
        W.set_tuning("multistep", 0)  # one launch per step (graph replay): the single-step latency
        sps1, ms1, _ = measure(cfg, E, args.steps)
        W.set_tuning("multistep", -1)
        sps, ms, geo = measure(cfg, E, args.steps)
        gbs = sps * algo_bytes(cfg) / 1e9
        rows.append(dict(sweep="C4 envs", agents=5, envs=E, obs="full", env_steps_per_s=sps,
                         ms_per_step=ms, single_step_us=1e3 * ms1, run_step_us=1e3 * ms,
                         floor_graph_node_us=floor["graph_node_us"],
                         single_step_vs_floor=1e3 * ms1 / floor["graph_node_us"],
                         algo_GBps=gbs, hbm_frac=gbs / hbm_peak(), geometry=geo))
        print(json.dumps(rows[-1]))
    # Continuous Tag (paper: 2000 envs x 5 agents) and larger A
    for A, mode, name in ((5, W.FULL, "full"), (100, W.PARTIAL, "partial"), (1000, W.PARTIAL, "partial")):
        T = max(1, min(A - 1, round(A / 5)))
        cfg = W.TagConfig(variant=W.CONTINUOUS, num_taggers=T, num_runners=A - T, obs_mode=mode,
                          k_nearest=min(5, A - 1))
        sps, ms, geo = measure(cfg, 2000, args.steps if A <= 100 else max(100, args.steps // 2))
        gbs = sps * algo_bytes(cfg) / 1e9
        rows.append(dict(sweep="continuous", agents=A, envs=2000, obs=name, env_steps_per_s=sps,
                         ms_per_step=ms, algo_GBps=gbs, hbm_frac=gbs / hbm_peak(), geometry=geo))
        print(json.dumps(rows[-1]))
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
