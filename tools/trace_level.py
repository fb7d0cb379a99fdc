"""Per-level item timelines of a DSG_TRACE_FILE dump: for each listed level,
its items grouped by dependency (cover = dep s-1, semi = dep s-2, old = the
rest) with claim / ready / end times relative to the completion of level s-2.

    python tools/trace_level.py TRACE.bin LEVEL [LEVEL ...]
"""
import sys

import numpy as np

buf = open(sys.argv[1], "rb").read()
hdr = np.frombuffer(buf[:32], dtype=np.int64)
n_levels, total_items, blocks = int(hdr[0]), int(hdr[1]), int(hdr[2])
off = 32
level_off = np.frombuffer(buf[off:off + 8 * (n_levels + 1)], dtype=np.int64)
off += 8 * (n_levels + 1) * 2
items = np.frombuffer(buf[off:off + 16 * total_items], dtype=np.int32).reshape(total_items, 4)
off += 16 * total_items + 8 * n_levels * 2
tr = np.frombuffer(buf[off:off + 32 * total_items], dtype=np.uint64).reshape(total_items, 4)
last = (tr[:, 3] >> np.uint64(63)).astype(bool)
tr = tr.astype(np.int64)
tr[:, 3] &= (1 << 63) - 1
t0 = tr[tr[:, 0] > 0, 0].min()
rel = (tr - t0) / 1e3
done = {}
for s in range(1, n_levels):
    sel = np.nonzero((items[:, 0] == s) & last)[0]
    if len(sel):
        done[s] = rel[sel, 3].max()
for s in map(int, sys.argv[2:]):
    base = done.get(s - 2, 0.0)
    T = level_off[s + 1] - level_off[s]
    print(f"level {s}: T={T}  done(s-2)=0  done(s-1)={done.get(s - 1, 0) - base:.1f}  "
          f"done(s)={done.get(s, 0) - base:.1f} us")
    for name, cond in (("cover", items[:, 3] == s - 1), ("semi", items[:, 3] == s - 2),
                       ("old", items[:, 3] < s - 2)):
        sel = np.nonzero((items[:, 0] == s) & cond)[0]
        if not len(sel):
            continue
        r = rel[sel] - base
        print(f"  {name:5s} n={len(sel):5d} claim [{r[:, 0].min():7.1f},{r[:, 0].max():7.1f}] "
              f"ready [{r[:, 1].min():7.1f},{r[:, 1].max():7.1f}] end [{r[:, 3].min():7.1f},"
              f"{r[:, 3].max():7.1f}]  scan mean {np.mean(r[:, 2] - r[:, 1]):6.1f} us")
