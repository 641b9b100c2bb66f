"""Live-register pressure per CUDA source line of one kernel (compile-time
analysis, no GPU): joins `nvdisasm -plr -lrm count` (live GPRs per SASS
instruction) with `nvdisasm -g` (line table).

  python tools/reg_pressure.py <obj.o|cubin> <kernel-substring> [--top N]"""
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def cubins(path):
    if path.endswith(".cubin"):
        return [path]
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(path)], cwd=d, capture_output=True)
    return [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")]


def section(text, kern):
    out, on = [], False
    for ln in text.splitlines():
        if ln.startswith(".text.") or ln.startswith("\t.section\t.text."):
            on = kern in ln.split(":")[0] and ln.startswith(".text.")
        if on:
            out.append(ln)
    return out


def main():
    path, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    for cb in cubins(path):
        plr = subprocess.run(["nvdisasm", "-plr", "-lrm", "count", cb], capture_output=True, text=True).stdout
        g = subprocess.run(["nvdisasm", "-g", cb], capture_output=True, text=True).stdout
        sp, sg = section(plr, kern), section(g, kern)
        if not sp:
            continue
        live = {}
        for ln in sp:
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/.*//\s*\|\s*(\d+)", ln)
            if m:
                live[int(m.group(1), 16)] = int(m.group(2))
        cur = "?"
        per_line = defaultdict(int)
        for ln in sg:
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
            if m and int(m.group(1), 16) in live:
                per_line[cur] = max(per_line[cur], live[int(m.group(1), 16)])
        print(f"{os.path.basename(cb)}: max live GPRs {max(live.values())}")
        for k, v in sorted(per_line.items(), key=lambda kv: -kv[1])[:top]:
            print(f"  {v:4d}  {k}")
        return


if __name__ == "__main__":
    main()
