"""SASS evidence for the C2 dataflow kernel: mnemonic counts (bulk copies,
mbarrier, shared loads, spills) and the staged scan loop around its first
warp vote.

    python tools/sass_excerpt.py OBJ.o KERNEL_SUBSTRING > profiles/<tag>_sass.txt
"""
import re
import subprocess
import sys
from collections import Counter

obj, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n")[0]
    if pat not in name:
        continue
    lines = [re.sub(r"\s*/\*[0-9a-fx]+\*/\s*$", "", l.strip()) for l in f.split("\n")
             if re.match(r"\s+/\*[0-9a-f]{4,5}\*/", l)]
    ops = Counter(l.split()[1].split(".")[0] if l.split()[1].startswith("@") is False else
                  l.split()[2].split(".")[0] for l in lines if len(l.split()) > 1)
    print(f"kernel {name}")
    print(f"instructions {len(lines)}")
    for k in ("UBLKCP", "SYNCS", "LDS", "LDG", "LD", "STS", "LDL", "STL", "BAR", "VOTE", "ATOMS",
              "RED", "ATOM", "MEMBAR", "CCTL", "LOP3", "VIMNMX", "VIMNMX3"):
        print(f"  {k:8s} {ops.get(k, 0)}")
    print("\n-- bulk-copy staging (cp.async.bulk -> UBLKCP, mbarrier -> SYNCS):")
    for i, l in enumerate(lines):
        if "UBLKCP" in l or "SYNCS" in l:
            print("  " + l)
    # the staged subset test: LDS.128 source rows against the target words
    # (LOP3), then the warp vote on 'any lane nested'
    hot = None
    for i, l in enumerate(lines):
        if "LDS.128" in l:
            v = next((j for j in range(i, min(len(lines), i + 40)) if "VOTE" in lines[j]), None)
            if v is not None:
                hot = (i, v)
                break
    if hot is None:
        hot = (next(i for i, l in enumerate(lines) if "VOTE.ANY" in l),) * 2
    print("\n-- staged scan loop (subset test on LDS.128 rows, warp vote):")
    for l in lines[max(0, hot[0] - 12):hot[1] + 8]:
        print("  " + l)
    break
