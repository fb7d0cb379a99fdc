"""Dump every traced item (debug): level, unit, chunk, dep, claim/ready/end us."""
import sys
import numpy as np
buf = open(sys.argv[1], "rb").read()
hdr = np.frombuffer(buf[:32], dtype=np.int64)
n_levels, total = int(hdr[0]), int(hdr[1])
off = 32 + 8 * (n_levels + 1) * 2
items = np.frombuffer(buf[off:off + 16 * total], dtype=np.int32).reshape(total, 4)
off += 16 * total + 16 * n_levels
tr = np.frombuffer(buf[off:off + 32 * total], dtype=np.uint64).reshape(total, 4).astype(np.int64)
t0 = tr[tr[:, 0] > 0, 0].min() if (tr[:, 0] > 0).any() else 0
for i in range(total):
    r = tr[i]
    f = lambda x: f"{(x - t0) / 1e3:9.1f}" if x > 0 else "        -"
    print(i, tuple(items[i]), f(r[0]), f(r[1]), f(r[2]), f(r[3] & ((1 << 63) - 1)))
