"""Per-level completion times of a DSG_TRACE_FILE dump, for diffing runs.

    python tools/trace_gaps.py TRACE.bin > gaps.txt     # level T mode done_us
"""
import sys

import numpy as np

buf = open(sys.argv[1], "rb").read()
hdr = np.frombuffer(buf[:32], dtype=np.int64)
n_levels, total_items = int(hdr[0]), int(hdr[1])
off = 32
level_off = np.frombuffer(buf[off:off + 8 * (n_levels + 1)], dtype=np.int64)
off += 8 * (n_levels + 1) * 2
items = np.frombuffer(buf[off:off + 16 * total_items], dtype=np.int32).reshape(total_items, 4)
off += 16 * total_items
off += 8 * n_levels
mode = np.frombuffer(buf[off:off + 8 * n_levels], dtype=np.int64)
off += 8 * n_levels
tr = np.frombuffer(buf[off:off + 32 * total_items], dtype=np.uint64).reshape(total_items, 4)
last = (tr[:, 3] >> np.uint64(63)).astype(bool)
tr = tr.astype(np.int64)
tr[:, 3] &= (1 << 63) - 1
t0 = tr[tr[:, 0] > 0, 0].min()
for s in range(1, n_levels):
    sel = np.nonzero((items[:, 0] == s) & last)[0]
    done = (tr[sel, 3].max() - t0) / 1e3 if len(sel) else float("nan")
    print(s, level_off[s + 1] - level_off[s], mode[s], f"{done:.1f}")
