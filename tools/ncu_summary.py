"""Summarise an `ncu --set full` report of the fused Tag kernel into profiles/.

  python tools/ncu_summary.py <report.ncu-rep> <tag> [--config c2_fused] [--bytes-per-launch B]

Writes profiles/<tag>.md (speed-of-light, occupancy, stall reasons, DRAM
traffic vs algorithmic bytes) and merges {config: dram bytes per launch} into
profiles/ncu_traffic.json (only with --config NAME, e.g. c2_fused), which
bench.py reports as roofline.traffic."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% peak)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (% peak)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block (B)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe (% active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe (% active)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe (% active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe (% active)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (% active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)"),
]


KERNEL = os.environ.get("NCU_KERNEL", "tag_env_kernel")  # e.g. NCU_KERNEL=tag_small_kernel


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in d and units.get(k) in scale:
                d[k] = str(float(d[k].replace(",", "")) * scale[units[k]])
        if KERNEL in d.get("Kernel Name", ""):
            kernels.append(d)
    return kernels


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    global KERNEL
    rep, tag = sys.argv[1], sys.argv[2]
    if "--kernel" in sys.argv:
        KERNEL = sys.argv[sys.argv.index("--kernel") + 1]
    cfg = None  # roofline.traffic entry to update (e.g. c2_fused); none by default
    if "--config" in sys.argv:
        cfg = sys.argv[sys.argv.index("--config") + 1]
    steps = 1
    if "--steps-per-launch" in sys.argv:  # multi-step residency launches
        steps = int(sys.argv[sys.argv.index("--steps-per-launch") + 1])
    algo = 2000 * 164009 * steps
    if "--bytes-per-launch" in sys.argv:
        algo = float(sys.argv[sys.argv.index("--bytes-per-launch") + 1])
    ks = raw(rep)
    if not ks:
        sys.exit(f"no {KERNEL} in report")
    d = ks[0]
    lines = [f"# ncu summary `{tag}`", "", f"kernel: `{d.get('Kernel Name')}`", "",
             f"report: `{os.path.basename(rep)}` (`ncu --set full --clock-control none`, 1 launch, "
             "cold caches — compare shares, not absolutes)", "", "| metric | value |", "|---|---|"]
    vals = {}
    for k, label in KEYS:
        v = num(d.get(k))
        if v is None:
            continue
        if k.startswith("dram__bytes"):
            vals[k] = v
            v = v / 1e6
            label += ""
        lines.append(f"| {label} | {v:,.3f} |")
    rd = num(d.get("dram__bytes_read.sum"))
    wr = num(d.get("dram__bytes_write.sum"))
    traffic = None
    if rd is not None and wr is not None:
        traffic = rd + wr  # bytes (unit-normalised in raw())
        lines += ["", f"DRAM traffic per launch: {traffic / 1e6:,.1f} MB vs algorithmic "
                      f"{algo / 1e6:,.1f} MB ({traffic / algo:.2f}x)"]
        if steps > 1:
            lines += [f"launch = {steps} env-steps (multi-step residency): per step "
                      f"{traffic / steps / 1e6:,.1f} MB DRAM, {num(d.get('gpu__time_duration.sum')) / steps:,.2f} "
                      "(duration unit) per step"]
            traffic /= steps  # per env-step launch equivalent, as bench.py reports
    stalls = {k: num(v) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    top = sorted(((v, k) for k, v in stalls.items() if v), reverse=True)[:10]
    lines += ["", "warp stall reasons (warps per issue-active cycle):", ""]
    for v, k in top:
        lines.append(f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.2f}")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic is not None and cfg:
        p = os.path.join(PROF, "ncu_traffic.json")
        cur = {}
        if os.path.exists(p):
            cur = json.load(open(p))
        cur[cfg] = traffic
        cur[cfg + "_source"] = f"profiles/{tag}.md"
        json.dump(cur, open(p, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
