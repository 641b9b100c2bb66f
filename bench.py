#!/usr/bin/env python
"""bench.py — env-steps/s of the Tag hot path (sample -> step -> reset-on-done)
on B200, BASELINE.json's metric on its headline config.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one RolloutDriver::step (proj/src/harness.cpp:478-490) over every
env of the shard: sample_actions from f64 logits (zeros = the reference
benchmark's uniform policy, harness.cpp:439,446-447), the Tag step, episode
statistics, reset-on-done — on our side ONE fused sm_100a kernel launch.
The `run_multistep` leg reports RolloutDriver::run (harness.cpp:492-494),
which runs up to 64 consecutive steps per launch with each env's state in
shared memory; with the benchmark's fixed logits buffer, the same env's
40 KB of logits are then re-read from L2, so that leg is not the headline.

Workload (N=1): C2 = discrete Tag, partial obs K=5, 2000 envs x 1000 agents
(200 taggers, the bench_agents scaling rule harness.cpp:823-831), D=23.
Multi-GPU (torchrun): weak scaling, 2000 envs per GPU, contiguous env shards
with global env ids in every RNG key (C5 = 16000 envs at N=8); NCCL carries
only the episode-statistics all-reduce every --stats-every steps.

value  = env-steps/s with state resident in HBM, device-timed (CUDA events on
         the store's stream, max over ranks).
e2e    = the same metric through the C-ABI host-buffer entry point
         (wdg_rollout_step_host): each step copies its f64 logits from pinned
         host memory to the device and reads rewards+done back.
--impl reference: the reference's own CPU path (oracle/_ref, compiled from the
reference sources) on all host cores, sharded into race-free single-worker
worlds; rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---- the workload (BASELINE.json configs[1]) ------------------------------------
ENVS_PER_GPU = 2000
C2 = dict(variant=0, obs_mode=1, grid_size=20, num_taggers=200, num_runners=800, k_nearest=5,
          episode_length=500, seed=0)
# Algorithmic bytes per env-step: each store element read
# and/or written once: A*[8CV logits r + 4C actions w + 8 loc r + 8 loc w +
# 1 is_tagger r + 2 active r/w + 4 credits w + 1 was_tagged w + 4 rewards w +
# 4D obs w] + 9 (step_count r/w, done w) = 164,009 B at C2.
def algo_bytes_per_env_step(A=1000, C=1, V=5, D=23):
    return A * (8 * C * V + 4 * C + 8 + 8 + 1 + 2 + 4 + 1 + 4 + 4 * D) + 9


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms; only samples
    taken while `active` (a timed region) count."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.active = False
        self._stop = False
        self._t = threading.Thread(target=self._run, daemon=True)

    def start(self):
        self._t.start()
        return self

    def _run(self):
        while not self._stop:
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out and self.active:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            time.sleep(0.2)

    def stop(self):
        self._stop = True

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 5 + i and s[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(config_key):
    """Per-launch DRAM bytes of the fused kernel from the committed ncu
    capture (profiles/ncu_traffic.json, written from an `ncu --set full` run
    by tools/ncu_summary.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(config_key)
    except Exception:
        return None


# ---- reference arm ----------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle as O  # the reference build lives under oracle/_ref (test/baseline infra)
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libwarpref.so not built"}))
        return 0
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    cfg = O.make_config(**C2)
    envs_per_thread = args.ref_envs_per_thread
    per_step = []
    setup_total = 0.0
    # each "step" of this arm = a bounded sample of the workload: every thread
    # advances its own envs_per_thread-env world by --ref-inner steps.
    sps, setup, run_s = O.bench_reference_sharded(cfg, envs_per_thread, threads, args.warmup,
                                                  args.ref_inner * args.steps)
    setup_total += setup
    value = sps
    ms_per_step = 1e3 * ENVS_PER_GPU / value  # one 2000-env step at this rate
    line = {
        "impl": "reference",
        "metric": "env-steps/sec (Tag, 2000 envs x 1000 agents)",
        "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": "C2: discrete Tag, partial obs K=5, 2000 envs x 1000 agents "
                               "(200 taggers), zero logits", "parallelism": f"cpu x{threads}"},
        "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": threads, "kind": "reference",
                         "sample": f"{threads} threads x {envs_per_thread} envs x 1000 agents, "
                                   f"{args.ref_inner * args.steps} steps after {args.warmup} warm-up "
                                   f"(reference StepEngine worker_count=1 per thread; setup {setup:.1f}s, "
                                   f"run {run_s:.1f}s)"},
        "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---- our arm ---------------------------------------------------------------------
def cpu_baseline_sample(args):
    """The reference (oracle/_ref) timed on this box's host cores on a bounded
    sample of C2 (rank 0, N=1 only)."""
    try:
        import oracle as O
        if not O.ref_available():
            return None
        threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        cfg = O.make_config(**C2)
        sps, setup, run_s = O.bench_reference_sharded(cfg, args.ref_envs_per_thread, threads, 3,
                                                      args.cpu_steps)
        return {"value": sps, "unit": "env-steps/s", "cores": threads, "kind": "reference",
                "sample": f"{threads} threads x {args.ref_envs_per_thread} envs x 1000 agents x "
                          f"{args.cpu_steps} steps (reference sources compiled in oracle/_ref, "
                          f"StepEngine worker_count=1 per shard; run {run_s:.1f}s)"}
    except Exception as e:  # baseline is reported, never required
        return {"value": None, "unit": "env-steps/s", "cores": 0, "kind": "reference",
                "sample": f"failed: {e}"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2108_13976_b200 as W

    torch.cuda.set_device(local_rank)
    W.lib().wdg_set_device(local_rank)
    stream = torch.cuda.current_stream()
    from paper_2108_13976_b200.sharding import weak_shard
    env_offset, E = weak_shard(ENVS_PER_GPU, rank)
    cfg = W.TagConfig(**C2)
    ws = W.Workspace(cfg, E, env_offset=env_offset, stream=stream)
    drv = W.RolloutDriver(ws.store, ws.plan, ws.resets, cfg.seed)
    A, Cc, V, D = cfg.num_agents(), cfg.action_categories(), cfg.action_choices(), cfg.obs_dim()
    geo = ws.plan.geometry()
    stats_t = torch.zeros(8, dtype=torch.float64, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    def stats_allreduce():
        drv.reduce_stats_into(stats_t)
        if world > 1:
            dist.all_reduce(stats_t)

    clocks = ClockSampler(local_rank).start()
    # ---- device-resident timed region ----
    for _ in range(args.warmup):
        drv.step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.active = True
    ev0.record(stream)
    launches0 = drv.launches()
    stats_launches = 0
    # One fused launch per step (RolloutDriver::step): each step's 328 MB
    # working set (80 MB logits read + state + 184 MB observations written)
    # exceeds the 126 MB L2, so no step finds the previous step's inputs there.
    for i in range(args.steps):
        drv.step()
        if world > 1 and (i + 1) % args.stats_every == 0:
            stats_allreduce()
            stats_launches += 2  # tracker reduce + NCCL all-reduce
    ev1.record(stream)
    launches = drv.launches() - launches0 + stats_launches
    torch.cuda.synchronize()
    clocks.active = False
    barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * E * args.steps / (ms_max / 1e3)
    drv.check()
    stats_allreduce()
    stats = stats_t.cpu().tolist()

    # ---- sampler stress: the same fused step on non-uniform logits ----
    # The headline uses the reference benchmark's zero logits, where every
    # exp() of the softmax is exp(0) == 1 and is skipped exactly. This leg
    # reports the step with N(0, 3^2) logits so the general
    # sampler cost is visible next to it; not part of `value`.
    gen = torch.Generator(device="cuda").manual_seed(1234)
    stress_logits = torch.randn(E * A * Cc * V, dtype=torch.float64, device="cuda", generator=gen) * 3.0
    drv.set_logits(stress_logits, stress_logits.numel())
    stress_steps = max(1, min(args.steps, 500))
    for _ in range(3):
        drv.step()
    torch.cuda.synchronize()
    es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es0.record(stream)
    for _ in range(stress_steps):
        drv.step()
    es1.record(stream)
    torch.cuda.synchronize()
    stress_ms = es0.elapsed_time(es1)
    drv.set_logits(None, 0)
    drv.check()
    del stress_logits

    # ---- multi-step residency leg (RolloutDriver::run): informational ----
    ms_steps = max(64, min(args.steps, 2048)) // 64 * 64
    drv.run(64)
    torch.cuda.synchronize()
    es0.record(stream)
    ml0 = drv.launches()
    drv.run(ms_steps)
    es1.record(stream)
    torch.cuda.synchronize()
    ms_ms = es0.elapsed_time(es1)
    multistep_leg = {"steps": ms_steps, "launches": drv.launches() - ml0,
                     "env_steps_per_s": E * ms_steps / (ms_ms / 1e3), "ms_per_step": ms_ms / ms_steps,
                     "note": "64 steps per launch, env state resident in smem; the fixed logits buffer "
                             "is re-read from L2 within an env's 64 steps"}
    drv.check()

    # ---- policy leg: the rollout driven by device policies (SURVEY.md §8f
    # row 1): tagger / runner MLPs (obs -> 64 -> 64 -> logits) on the tcgen05
    # tensor cores, sampling fused into their epilogue, then the fused step.
    # Reported beside `value`, not part of it.
    policy_leg = None
    try:
        pol_t, pol_r = W.Policy.for_tag(cfg, seed=1), W.Policy.for_tag(cfg, seed=2)
        drv.set_policies(pol_t, pol_r, W.POLICY_BF16)
        pol_steps = max(1, min(args.steps, 300))
        for _ in range(3):
            drv.step()
        torch.cuda.synchronize()
        es0.record(stream)
        for _ in range(pol_steps):
            drv.step()
        es1.record(stream)
        torch.cuda.synchronize()
        pol_ms = es0.elapsed_time(es1)
        drv.check()
        policy_leg = {"policy": "2 x MLP obs->64->64->5 (tagger, runner), bf16 tcgen05, f32 accumulate",
                      "steps": pol_steps, "env_steps_per_s": E * pol_steps / (pol_ms / 1e3),
                      "ms_per_step": pol_ms / pol_steps, "gpu_launches_per_step": 3}
    except Exception as exc:  # reported, never required
        policy_leg = {"error": str(exc)}
    finally:
        drv.set_policies(None, None)

    # ---- e2e through the C-ABI host-buffer entry point ----
    n_logits = E * A * Cc * V
    host_logits = torch.zeros(n_logits, dtype=torch.float64).pin_memory()
    host_rewards = torch.empty(E * A, dtype=torch.float32).pin_memory()
    host_done = torch.empty(E, dtype=torch.uint8).pin_memory()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(min(args.warmup, 5)):
        drv.step_host(host_logits, n_logits, host_rewards, host_done)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks.active = True
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        drv.step_host(host_logits, n_logits, host_rewards, host_done)
    ws.store.synchronize()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    clocks.active = False
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * E * e2e_steps / float(te.item())
    clocks.stop()

    if rank == 0:
        peak, peak_kind = measured_peak_hbm()
        b_env = algo_bytes_per_env_step(A, Cc, V, D)
        launch_s = (ms / 1e3) / args.steps  # one fused launch per step
        achieved = E * b_env / launch_s / 1e9
        traffic = ncu_traffic("c2_fused")
        line = {
            "metric": "env-steps/sec (Tag, 2000 envs x 1000 agents)",
            "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (env) / f64 (sampler)",
            "data": "synthetic (episode-0 placement from seed 0, zero logits = uniform policy)",
            "config": {"workload": f"C2: discrete Tag, partial obs K=5, {E} envs x {A} agents "
                                   f"(200 taggers) per GPU, D={D}",
                       "envs_total": world * E, "agents": A, "parallelism": f"env-shard x{world}",
                       "l2": "per-step state 328 MB > 126 MB L2 (no flush needed)",
                       "kernel_geometry": geo},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind,
                         "algorithmic_bytes_per_env_step": b_env,
                         "kernel": "tag_env_kernel<discrete,partial,grid> (fused step)"},
            "e2e": {"value": e2e_value, "unit": "env-steps/s",
                    "h2d_bytes_per_step": n_logits * 8, "d2h_bytes_per_step": E * A * 4 + E,
                    # per-rank PCIe upload rate implied by the e2e value (bound: the link's
                    # pinned H2D rate, 55.3 GB/s measured by tools/h2d_probe.py)
                    "h2d_gbs": (e2e_value / world) / E * n_logits * 8 / 1e9,
                    "path": "wdg_rollout_step_host (pinned host logits -> fused kernel -> rewards+done)"},
            "sampler_stress": {"logits": "N(0, 3^2), seed 1234", "steps": stress_steps,
                               "env_steps_per_s": E * stress_steps / (stress_ms / 1e3),
                               "ms_per_step": stress_ms / stress_steps},
            "policy_rollout": policy_leg,
            "run_multistep": multistep_leg,
            "per_gpu_value": value / world,  # aggregate and per-GPU env-steps/s
            "gpu_launches": launches,
            "episode_stats": {"episodes": stats[0], "tag_events": stats[3], "env_steps": stats[4]},
            "clocks": clocks.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample(args)
        print(json.dumps(line))
    ws.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--stats-every", type=int, default=100)
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--cpu-steps", type=int, default=12000)  # ~10 s of reference CPU work at C2
    ap.add_argument("--ref-envs-per-thread", type=int, default=4)
    ap.add_argument("--ref-inner", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # Test-only: run every rank on cuda:0 over gloo, to exercise the N>1
    # logic (shards, barriers, max-over-ranks, stats all-reduce) on one GPU.
    ap.add_argument("--same-device", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = 0 if args.same_device else env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if args.same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
