"""Device vs oracle-port lattice, level by level (debug): which levels differ
and whether as sets (content) or only in order.

    python tools/lattice_diff.py WORKLOAD [FLAGS]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402  (checker)
from paper_2006_16423_b200 import solver, workloads as wl  # noqa: E402

w = wl.by_name(sys.argv[1])
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
d = solver.enumerate_ideals(w.graph, flags=flags)
r = ob.enumerate_ideals("port", w.graph)
rb = np.array([[int(x) for x in row] for row in r.bits], dtype=np.uint64)
print("counts", d.bits.shape, rb.shape, "levels equal", np.array_equal(d.level_offsets, r.level_offsets))
lo = [int(x) for x in r.level_offsets]
bad = 0
for s in range(len(lo) - 1):
    a, b = d.bits[lo[s]:lo[s + 1]], rb[lo[s]:lo[s + 1]]
    if not np.array_equal(a, b):
        same_set = set(map(tuple, a.tolist())) == set(map(tuple, b.tolist()))
        first = int(np.nonzero(~np.all(a == b, axis=1))[0][0])
        print(f"level {s} T={lo[s + 1] - lo[s]} differs: same set {same_set}, first bad row {first}")
        bad += 1
print("bad levels", bad)
