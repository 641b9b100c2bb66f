"""Aggregate an ncu report's per-SASS metrics onto CUDA source lines.

  python tools/ncu_lines.py <report.ncu-rep> [kernel-substring] [--top N]

Joins `ncu --page source --print-source sass` (per-address metrics) with the
line table from `nvdisasm -g` of the built library's cubin (compiled with
-lineinfo), and prints the hottest source lines by warp-stall samples and
executed instructions."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.environ.get("WDG_SO", os.path.join(ROOT, "paper_2108_13976_b200", "lib", "libwdg_b200.so"))


def sass_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    kernels = {}
    cur = None
    rows = []
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            if cur:
                kernels[cur] = rows
            cur = next(csv.reader(io.StringIO(line)))[1]
            rows = []
        elif line.startswith('"Address"'):
            header = next(csv.reader(io.StringIO(line)))
        elif cur and line.startswith('"'):
            rows.append(dict(zip(header, next(csv.reader(io.StringIO(line))))))
    if cur:
        kernels[cur] = rows
    return kernels


def line_table():
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(SO)], cwd=d, capture_output=True)
    txt = ""
    for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):
        txt += subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                              text=True).stdout + "\n"
    funcs = {}
    fn, line = None, None
    for ln in txt.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
            funcs[fn] = {}
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and fn:
            funcs[fn][int(m.group(1), 16)] = line
    return funcs


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "tag_env_kernel"
    top = 40
    if "--top" in sys.argv:
        top = int(sys.argv[sys.argv.index("--top") + 1])
    kernels = sass_metrics(rep)
    funcs = line_table()
    for kname, rows in kernels.items():
        if want not in kname:
            continue
        # match function by template args
        targs = re.findall(r"\((bool|int)\)(\w+)", kname)
        base_name = re.findall(r"(\w+)(?:<\(|\()", kname)[0]
        mangled = [f for f in funcs if base_name in f]
        sig = "".join((f"Lb{a}E" if t == "bool" else f"Li{a}E") for t, a in targs)
        cand = [f for f in mangled if sig in f.replace("ILb", "Lb").replace("ILi", "Li")] or mangled
        table = funcs[cand[0]]
        agg = defaultdict(lambda: [0, 0, 0])
        tot = [0, 0]
        base = min(int(r["Address"], 16) for r in rows)
        for r in rows:
            addr = int(r["Address"], 16) - base
            ln = table.get(addr, "?")
            s = int(r.get("Warp Stall Sampling (All Samples)", 0) or 0)
            ins = int(r.get("Instructions Executed", 0) or 0)
            agg[ln][0] += s
            agg[ln][1] += ins
            agg[ln][2] += 1
            tot[0] += s
            tot[1] += ins
        print(f"{kname}\n  samples={tot[0]} warp-instructions={tot[1]}")
        for ln, (s, ins, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
            print(f"  {ln:28s} samples {100 * s / max(1, tot[0]):5.1f}%  instr {100 * ins / max(1, tot[1]):5.1f}%  sass {n}")


if __name__ == "__main__":
    main()
