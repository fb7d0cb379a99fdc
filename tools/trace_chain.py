"""Chain analysis of a DSG_TRACE_FILE dump (narrow-level lattices, e.g. C4):
for every level, the old chunk that ended last before the level's finisher
could proceed, how long after its source level was done it became ready and
how long it ran, and the finisher's own time.

    python tools/trace_chain.py TRACE.bin [first_level last_level]
"""
import sys

import numpy as np

buf = open(sys.argv[1], "rb").read()
hdr = np.frombuffer(buf[:32], dtype=np.int64)
n_levels, total = int(hdr[0]), int(hdr[1])
off = 32
level_off = np.frombuffer(buf[off:off + 8 * (n_levels + 1)], dtype=np.int64)
off += 8 * (n_levels + 1) * 2
items = np.frombuffer(buf[off:off + 16 * total], dtype=np.int32).reshape(total, 4)
off += 16 * total
nch = np.frombuffer(buf[off:off + 8 * n_levels], dtype=np.int64)
off += 8 * n_levels
mode = np.frombuffer(buf[off:off + 8 * n_levels], dtype=np.int64)
off += 8 * n_levels
tr = np.frombuffer(buf[off:off + 32 * total], dtype=np.uint64).reshape(total, 4).astype(np.int64)
tr[:, 3] &= (1 << 63) - 1
t0 = tr[tr[:, 0] > 0, 0].min()
tr = np.where(tr > 0, (tr - t0) / 1e3, np.nan)
lv, ch, dep = items[:, 0], items[:, 2], items[:, 3]
fin = ch == nch[lv] - 1
done = np.full(n_levels, np.nan)
for s in range(1, n_levels):
    f = np.nonzero((lv == s) & fin)[0]
    if len(f):
        done[s] = np.nanmax(tr[f, 3])
args = [x for x in sys.argv[2:] if x != "-q"]
a = int(args[0]) if args else 1
b = int(args[1]) if len(args) > 1 else n_levels - 1
rows = []
for s in range(max(a, 2), b):
    o = np.nonzero((lv == s) & ~fin)[0]
    f = np.nonzero((lv == s) & fin)[0]
    if not len(o) or not len(f):
        continue
    g = o[np.nanargmax(tr[o, 3])]
    d = dep[g]
    rows.append((s, level_off[s + 1] - level_off[s], mode[s], done[s] - done[s - 1], d - s,
                 tr[g, 0] - done[d] if d > 0 else np.nan, tr[g, 1] - done[d] if d > 0 else np.nan,
                 tr[g, 3] - tr[g, 1], np.nanmax(tr[f, 1]) - tr[g, 3], done[s] - np.nanmax(tr[f, 1]),
                 np.nanmax(tr[f, 2]) - done[s - 1], done[s] - np.nanmax(tr[f, 2])))
r = np.array(rows, dtype=float)
print("cols: level T mode dt gate_dep-s claim-after-dep ready-after-dep gate_run fin_ready-gate_end fin_run fold_end-prev_done done-fold_end")
print("mean:", " ".join(f"{x:.2f}" for x in np.nanmean(r, axis=0)))
print("median:", " ".join(f"{x:.2f}" for x in np.nanmedian(r, axis=0)))
for x in r[:: max(1, len(r) // 25)] if "-q" not in sys.argv else []:
    print(" ".join(f"{v:.2f}" for v in x))
