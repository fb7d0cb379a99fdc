"""Golden ideal lists of large lattices as digests: the UNMODIFIED reference's
enumerate_ideals (oracle/_ref, ideals.cpp:14-86) in ordinal order, hashed
(SHA-256 of the little-endian uint64 bitset rows, and of the level offsets),
so the device lattice can be compared ordinal by ordinal without a
multi-megabyte fixture.  Writes tests/golden/ideal_digests.json.

    python tests/golden/make_ideal_digests.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_bind as ob  # noqa: E402
from paper_2006_16423_b200 import workloads as wl  # noqa: E402

CASES = ["C4", "C5:16,1,1,300", "C2", "C5:8,2,7,600", "C5:4,3,40,1400", "C5:12,1,8,1000"]


def digest(bits, level_offsets):
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint64))
    lo = np.asarray(level_offsets, dtype=np.int64)
    return hashlib.sha256(b.tobytes()).hexdigest(), hashlib.sha256(lo.tobytes()).hexdigest()


def main():
    rows = []
    for name in CASES:
        w = wl.by_name(name)
        ix = ob.enumerate_ideals("ref", w.graph)
        bits = np.array([[int(x) for x in r] for r in ix.bits], dtype=np.uint64)
        hb, hl = digest(bits, ix.level_offsets)
        rows.append({"workload": name, "count": int(bits.shape[0]), "words": int(bits.shape[1]),
                     "levels": len(ix.level_offsets) - 1,
                     "max_level": int(np.max(np.diff(np.asarray(ix.level_offsets)))),
                     "bits_sha256": hb, "level_offsets_sha256": hl})
        print(rows[-1], flush=True)
    with open(os.path.join(HERE, "ideal_digests.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
