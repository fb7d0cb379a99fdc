"""Large lattices ordinal by ordinal: the device enumeration (both dedup
modes) against the UNMODIFIED reference's enumerate_ideals (ideals.cpp:14-86),
held as SHA-256 digests of the ordinal-ordered bitset rows and of the level
offsets (tests/golden/make_ideal_digests.py).  Covers W = 24 (C4), the
3 %-dense sweep point whose widest level (12,870 ideals) takes the merge-pass
ordering, W = 31 and the C5 top point."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_bind as ob
from golden_io import GOLDEN
from paper_2006_16423_b200 import _abi, solver
from paper_2006_16423_b200 import workloads as wl

ROWS = json.load(open(os.path.join(GOLDEN, "ideal_digests.json")))


def digests(ix):
    b = np.ascontiguousarray(np.asarray(ix.bits, dtype=np.uint64))
    lo = np.asarray(ix.level_offsets, dtype=np.int64)
    return hashlib.sha256(b.tobytes()).hexdigest(), hashlib.sha256(lo.tobytes()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("hash_mode", [False, True], ids=["canonical", "hashset"])
@pytest.mark.parametrize("row", ROWS, ids=[r["workload"] for r in ROWS])
def test_device_lattice_matches_reference(gpu, row, hash_mode):
    w = wl.by_name(row["workload"])
    ix = solver.enumerate_ideals(w.graph, flags=_abi.DSG_FLAG_HASH_ENUM if hash_mode else 0)
    assert ix.bits.shape == (row["count"], row["words"])
    assert digests(ix) == (row["bits_sha256"], row["level_offsets_sha256"])


@pytest.mark.parametrize("name", ["C4", "C5:16,1,1,300"])
def test_oracle_port_lattice_matches_reference(name):
    """The C restatement's enumeration is pinned to the same digests."""
    row = next(r for r in ROWS if r["workload"] == name)
    w = wl.by_name(name)
    ix = ob.enumerate_ideals("port", w.graph)
    bits = np.array([[int(x) for x in r] for r in ix.bits], dtype=np.uint64)
    b = hashlib.sha256(np.ascontiguousarray(bits).tobytes()).hexdigest()
    lo = hashlib.sha256(np.asarray(ix.level_offsets, dtype=np.int64).tobytes()).hexdigest()
    assert (b, lo) == (row["bits_sha256"], row["level_offsets_sha256"])
