"""Per-CUDA-source-line instruction and stall totals from an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep [N]

Parses `ncu --page source --print-source cuda,sass --csv` (needs -lineinfo)
and prints the N hottest lines by warp-stall samples, with executed warp
instructions, across every source file of the kernel.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
file = "?"
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:  # a source line row
        cur = (file, int(r[0]), r[1].strip()[:80])
        continue
    if cur is None:
        continue
    try:
        samples = float(r[4] or 0)
        execd = float(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += samples
    a[1] += execd
tot_s = sum(v[0] for v in agg.values()) or 1
tot_e = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_e:.3e}")
for (f, ln, src), (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{s / tot_s * 100:5.1f}% stall {e / tot_e * 100:5.1f}% instr  {f}:{ln:<4} {src}")
