"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = idx["Warp Stall Sampling (All Samples)"]
E = idx["Instructions Executed"]
tot = sum(float(r[S] or 0) for r in data)
tot_e = sum(float(r[E] or 0) for r in data)
print(f"total samples {tot:.0f}, warp instrs {tot_e:.3e}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for r in sorted(data, key=lambda r: -float(r[S] or 0))[:n]:
    print(f"{float(r[S] or 0)/tot*100:5.1f}%  {r[idx['Address']]:>6}  {float(r[E] or 0):10.3e}  {r[idx['Source']][:90]}")
