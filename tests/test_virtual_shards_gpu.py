"""Virtual shards: the multi-GPU wavefront emulated on one GPU.

dsg_options.shard_count = G runs G ranks inside ONE cooperative launch
(CTA b is rank b % G).  Each rank has its own dp replica, merge keys, arrival
counters, level counters and readiness-ordered item list holding only its
target units (unit % G == rank) — what a rank owns on its own GPU — and its
finalizers store every finished row into all G replicas and bump all G level
counters (system scope), exactly the world >= 2 code a multi-GPU solve runs.
The library compares every replica with rank 0's after the solve (DSG_LOGIC on
any difference); here rank 0's table is compared byte for byte with the
unsharded solve, which mirrors the ordinal loop of dp_solver.cpp:327-330.
"""
import numpy as np
import pytest

import oracle_bind as ob
from golden_io import config_from_case, graph_from_json, load, rat_from_json
from paper_2006_16423_b200 import _abi, solver
from paper_2006_16423_b200 import workloads as wl
from paper_2006_16423_b200.errors import DeadlineExceeded, InfeasibleError, Unsupported
from paper_2006_16423_b200.graph import INF, verify_split

pytestmark = pytest.mark.gpu

CORPUS = load("dp_corpus.json")
KEEP = _abi.DSG_FLAG_KEEP_TABLES


def tables(mode, g, cfg, shards=0, flags=0, max_blocks=0):
    lib = solver.load_library()
    opt = solver.SolveOptions(flags=KEEP | flags, shard_count=shards, max_blocks=max_blocks)
    return solver.run_dp(lib, "dsg", mode, g, cfg, opt)


def check_same(mode, g, cfg, shards, flags=0, max_blocks=0):
    try:
        base = tables(mode, g, cfg, 0, flags)
    except InfeasibleError:
        with pytest.raises(InfeasibleError):
            tables(mode, g, cfg, shards, flags, max_blocks)
        return None
    got = tables(mode, g, cfg, shards, flags, max_blocks)
    assert got.objective == base.objective
    assert got.n_pairs == base.n_pairs
    assert got.n_ideals == base.n_ideals
    assert np.array_equal(got.dp_values, base.dp_values)
    assert np.array_equal(got.ideal_bits, base.ideal_bits)
    split = solver.make_canonical_split(g, cfg, got.blocks, got.objective)
    assert not verify_split(g, cfg, split, training=(mode == 1 and g.has_backward_nodes()))
    return got


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_corpus_tables_identical(gpu, shards):
    """AC-1 (inference) and AC-2 (mirrored training) corpora."""
    for case in CORPUS[::2]:
        g = graph_from_json(case["graph"])
        cfg = config_from_case(case)
        got = check_same(case["mode"], g, cfg, shards)
        want = rat_from_json(case["objective"])
        assert (got.objective if got else INF) == want, case["name"]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
@pytest.mark.parametrize("shards", [2, 3, 8])
def test_standin_tables_identical(gpu, name, shards):
    w = wl.standin(name)
    check_same(1 if w.training else 0, w.graph, w.config, shards)


@pytest.mark.parametrize("shards", [2, 5])
def test_int64_and_generic_cells(gpu, shards):
    """64-bit values, the generic shared-memory cells (K=12, L=3) and the
    unpruned path, sharded."""
    w = wl.standin("C3")
    check_same(1, w.graph, w.config, shards, _abi.DSG_FLAG_FORCE_INT64)
    w = wl.sweep(2, 8, 20, 100, k=12, l=3)
    check_same(0, w.graph, w.config, shards)


@pytest.mark.parametrize("shards,max_blocks", [(2, 2), (3, 3), (4, 9), (8, 8)])
def test_few_ctas_per_rank(gpu, shards, max_blocks):
    """One or two CTAs per rank: every rank's claims, waits and arrivals
    interleave with the other ranks' at fine grain."""
    for name in ("C1", "C3"):
        w = wl.standin(name)
        check_same(1, w.graph, w.config, shards, max_blocks=max_blocks)
    for case in CORPUS[1::9]:
        g = graph_from_json(case["graph"])
        check_same(case["mode"], g, config_from_case(case), shards, max_blocks=max_blocks)


def test_replication_sharded(gpu):
    from fractions import Fraction
    from paper_2006_16423_b200.graph import ReplicationCombine
    for seed in range(6):
        inst = wl.random_instance(seed)
        cfg = inst.config
        cfg.accelerators = 3
        cfg.bandwidth = Fraction(3, 2)
        cfg.replication_combine = ReplicationCombine(seed % 2)
        want = ob.objective_or_inf("port", 2, inst.graph, cfg)
        lib = solver.load_library()
        try:
            got = solver.run_dp(lib, "dsg", 2, inst.graph, cfg,
                                solver.SolveOptions(shard_count=4)).objective
        except InfeasibleError:
            got = INF
        assert got == want


def test_deadline_reaches_every_rank(gpu):
    """The deadline stops every rank (the stop word is raised on all of
    them), so no rank waits out its watchdog."""
    w = wl.standin("C2")
    lib = solver.load_library()
    with pytest.raises(DeadlineExceeded):
        solver.run_dp(lib, "dsg", 0, w.graph, w.config,
                      solver.SolveOptions(shard_count=4, deadline_seconds=1e-4))


def test_shards_need_the_persistent_kernel(gpu):
    w = wl.standin("C1")
    lib = solver.load_library()
    with pytest.raises(Unsupported):
        solver.run_dp(lib, "dsg", 1, w.graph, w.config,
                      solver.SolveOptions(shard_count=2, flags=_abi.DSG_FLAG_LEVEL_LAUNCH))
