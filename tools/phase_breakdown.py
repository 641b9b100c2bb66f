"""Group ncu_lines.py output into kernel phases by source-line ranges found
from the phase comments in tag_kernels.cu.  python tools/phase_breakdown.py <lines.txt>"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2108_13976_b200", "csrc", "tag_kernels.cu")


def ranges():
    marks = []
    for i, ln in enumerate(open(SRC), 1):
        m = re.match(r"\s*// Phase (\d+)", ln)
        if m:
            marks.append((i, f"P{m.group(1)}"))
            continue
        m = re.match(r"^(?:template <[^>]*>\s*)?__device__.*?\b(\w+)\(", ln)
        if m and "__forceinline__" not in ln or (m and ln.startswith("__device__")):
            marks.append((i, m.group(1)))
        m2 = re.match(r"^__global__.*?\b(\w+)\(", ln)
        if m2:
            marks.append((i, m2.group(1)))
    marks.sort()
    out = []
    for k, (start, name) in enumerate(marks):
        end = marks[k + 1][0] - 1 if k + 1 < len(marks) else 10 ** 9
        out.append((start, end, name))
    return out


def main():
    rs = ranges()
    agg = {}
    for ln in open(sys.argv[1]):
        m = re.match(r"\s+(\S+):(\d+)\s+samples\s+([\d.]+)%\s+instr\s+([\d.]+)%", ln)
        if not m:
            m2 = re.match(r"\s+(\S+)\s+samples\s+([\d.]+)%\s+instr\s+([\d.]+)%", ln)
            if m2:
                a = agg.setdefault("(no line)", [0.0, 0.0])
                a[0] += float(m2.group(2)); a[1] += float(m2.group(3))
            continue
        f, l, s, i = m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4))
        key = f if f != "tag_kernels.cu" else next((n for a, b, n in rs if a <= l <= b), "?")
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += s
        a[1] += i
    for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if s + i >= 0.3:
            print(f"{k:28s} samples {s:5.1f}%  instr {i:5.1f}%")


if __name__ == "__main__":
    main()
