"""Summarise a DSG_TRACE_FILE dump of the dataflow level kernel.

Per level: when its first item started / finished waiting, when the level
completed (last finalize), item wait and scan times.  Usage:
    DSG_TRACE_FILE=/tmp/t.bin python tools/profile_one.py C2 1
    python tools/trace_view.py /tmp/t.bin
"""
import sys

import numpy as np

buf = open(sys.argv[1], "rb").read()
hdr = np.frombuffer(buf[:32], dtype=np.int64)
n_levels, total_items, blocks = int(hdr[0]), int(hdr[1]), int(hdr[2])
off = 32


def take(n, dt=np.int64):
    global off
    a = np.frombuffer(buf[off:off + 8 * n], dtype=dt)
    off += 8 * n
    return a


level_off = take(n_levels + 1)
item_base = take(n_levels + 1)
items = np.frombuffer(buf[off:off + 16 * total_items], dtype=np.int32).reshape(total_items, 4)
off += 16 * total_items
n_chunks = take(n_levels)
mode = take(n_levels)
tr = take(total_items * 4, np.uint64).reshape(total_items, 4)
last = (tr[:, 3] >> np.uint64(63)).astype(bool)
tr = tr.astype(np.int64)
tr[:, 3] &= (1 << 63) - 1
t0 = tr[tr[:, 0] > 0, 0].min()
rel = (tr - t0) / 1e3  # us
print(f"levels {n_levels}, items {total_items}, blocks {blocks}, span {rel[:, 3].max():.1f} us")
wait = rel[:, 1] - rel[:, 0]
scan = rel[:, 2] - rel[:, 1]
fin = rel[:, 3] - rel[:, 2]
print(f"item wait  mean {wait.mean():.2f} us  p99 {np.percentile(wait, 99):.2f}  total {wait.sum()/1e3:.1f} ms")
print(f"item scan  mean {scan.mean():.2f} us  p99 {np.percentile(scan, 99):.2f}  total {scan.sum()/1e3:.1f} ms")
print(f"item fin   mean {fin.mean():.2f} us  (finalizers {last.sum()}, mean {fin[last].mean():.2f} us)")
rows = []
for s in range(1, n_levels):
    sel = np.nonzero(items[:, 0] == s)[0]
    if len(sel) == 0:
        continue
    r = rel[sel]
    done = r[last[sel], 3].max() if last[sel].any() else float("nan")
    rows.append((s, level_off[s + 1] - level_off[s], len(sel), n_chunks[s], mode[s], r[:, 0].min(),
                 done, scan[sel].max()))
rows = np.array(rows)
lat = np.diff(np.concatenate([[0], rows[:, 6]]))
print("per-level completion gaps (us): mean %.2f  p50 %.2f  p90 %.2f  max %.2f" %
      (lat.mean(), np.median(lat), np.percentile(lat, 90), lat.max()))
step = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, len(rows) // 25)
lim = int(sys.argv[3]) if len(sys.argv) > 3 else len(rows)
print(" level   T  items chunks mode   start_us    done_us  gap_us  max_scan_us")
for i in range(0, min(lim, len(rows)), step):
    s, T, it, ch, md, st, dn, ms = rows[i]
    print(f"{int(s):6d} {int(T):4d} {int(it):6d} {int(ch):6d} {int(md):4d} {st:10.1f} {dn:10.1f} {lat[i]:7.2f} {ms:10.2f}")

# critical path per level: previous level done -> critical items (dep = s-1)
# claimed / scanning / done -> this level done
print("\ncritical path (us): level T prev_done crit_claim crit_scan0 crit_end done | n_crit")
done_at = {}
for s in range(1, n_levels):
    sel = np.nonzero(items[:, 0] == s)[0]
    if len(sel) and last[sel].any():
        done_at[s] = rel[sel][last[sel], 3].max()
for s in range(2, min(n_levels, lim + 1)):
    sel = np.nonzero((items[:, 0] == s) & (items[:, 3] == s - 1))[0]
    if not len(sel) or s not in done_at or (s - 1) not in done_at:
        continue
    r = rel[sel]
    print(f"{s:5d} {level_off[s + 1] - level_off[s]:4d} {done_at[s - 1]:9.1f} {r[:, 0].min() - done_at[s - 1]:7.1f} "
          f"{r[:, 1].min() - done_at[s - 1]:7.1f} {r[:, 3].max() - done_at[s - 1]:7.1f} "
          f"{done_at[s] - done_at[s - 1]:7.1f} | {len(sel)}")
