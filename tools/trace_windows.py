"""Wait / scan CTA-time per time window of a DSG_TRACE_FILE dump.

    python tools/trace_windows.py TRACE.bin [window_us]
"""
import sys

import numpy as np

buf = open(sys.argv[1], "rb").read()
win = float(sys.argv[2]) if len(sys.argv) > 2 else 500.0
hdr = np.frombuffer(buf[:32], dtype=np.int64)
n_levels, total_items, blocks = int(hdr[0]), int(hdr[1]), int(hdr[2])
off = 32 + 8 * (n_levels + 1) * 2
items = np.frombuffer(buf[off:off + 16 * total_items], dtype=np.int32).reshape(total_items, 4)
off += 16 * total_items + 8 * n_levels * 2
tr = np.frombuffer(buf[off:off + 32 * total_items], dtype=np.uint64).reshape(total_items, 4)
tr = tr.astype(np.int64)
tr[:, 3] &= (1 << 63) - 1
t0 = tr[tr[:, 0] > 0, 0].min()
rel = (tr - t0) / 1e3
span = rel[:, 3].max()
edges = np.arange(0, span + win, win)


def spread(a, b):
    # CTA-time of intervals [a, b) falling in each window
    out = np.zeros(len(edges) - 1)
    for i in range(len(edges) - 1):
        lo, hi = edges[i], edges[i + 1]
        out[i] = np.clip(np.minimum(b, hi) - np.maximum(a, lo), 0, None).sum()
    return out


w = spread(rel[:, 0], rel[:, 1])
s = spread(rel[:, 1], rel[:, 2])
f = spread(rel[:, 2], rel[:, 3])
print(f"span {span:.0f} us, {blocks} CTAs; per window: busy fraction of CTA-time")
print("   t_us     wait%   scan%   fin%   idle%  max_level_started")
for i in range(len(edges) - 1):
    cap = blocks * win
    started = items[(rel[:, 0] >= edges[i]) & (rel[:, 0] < edges[i + 1]), 0]
    ml = started.max() if len(started) else -1
    print(f"{edges[i]:7.0f} {100*w[i]/cap:7.1f} {100*s[i]/cap:7.1f} {100*f[i]/cap:6.1f} "
          f"{100*(1-(w[i]+s[i]+f[i])/cap):7.1f}  {ml}")
