"""Per-kernel counts of the SASS mnemonics that show which hardware paths the
built kernels use (TMA bulk copies, mbarriers, tcgen05 MMA / TMEM, streaming
stores), from `cuobjdump -sass` of the in-tree objects. Writes
profiles/sass_r02.md.   python tools/sass_evidence.py"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2108_13976_b200", "lib", "obj")
KEYS = ["UBLKCP", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "UTCHMMA", "UTCBAR", "LDTM", "MUFU.TANH", "MUFU.EX2",
        "STG.E.EF", "BAR.SYNC", "SHFL", "DFMA", "HMMA"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def main():
    rows = []
    for obj in ("tag_kernels.o", "twin_kernels.o", "policy.o", "batch.o"):
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
        cur, counts = None, collections.OrderedDict()
        for ln in sass.splitlines():
            m = re.match(r"\s+Function : (\S+)", ln)
            if m:
                cur = m.group(1)
                counts[cur] = collections.Counter()
                continue
            if cur and re.search(r"/\*[0-9a-f]{4,}\*/", ln):
                ins = ln.split("*/", 1)[1].strip().split(" ")[0].rstrip(";")
                if ins.startswith("@"):
                    ins = ln.split("*/", 1)[1].strip().split(" ")[1]
                for k in KEYS:
                    if ins.startswith(k):
                        counts[cur][k] += 1
        names = list(counts)
        for n, d in zip(names, demangle(names)):
            if sum(counts[n].values()) == 0:
                continue
            short = re.sub(r"\(.*", "", d.replace("wdg::(anonymous namespace)::", ""))
            rows.append((obj, short, counts[n]))
    lines = ["# SASS evidence (round 2)", "",
             "`cuobjdump -sass` of the in-tree sm_100a objects, by `tools/sass_evidence.py`. Counts are static",
             "instructions per kernel. `UBLKCP` = `cp.async.bulk` global->shared (the Tag kernel's input",
             "staging); `SYNCS.*` = mbarrier arrive / try-wait; `UTCHMMA` / `UTCBAR` / `LDTM` = tcgen05 MMA,",
             "commit and TMEM loads (bf16 policy); `STG.E.EF` = evict-first streaming stores (`__stcs`).", "",
             "| object | kernel | " + " | ".join(KEYS) + " |", "|---|---|" + "---|" * len(KEYS)]
    for obj, k, c in rows:
        lines.append(f"| {obj} | `{k}` | " + " | ".join(str(c.get(x, 0)) for x in KEYS) + " |")
    open(os.path.join(ROOT, "profiles", "sass_r02.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]), f"\n... {len(rows)} kernels")


if __name__ == "__main__":
    main()
