"""Device parity: the sm_100a path against the golden vectors dumped from the
unmodified reference and against the C restatement of the reference
algorithm.  Objectives must be bit-identical (exact rationals), ideal lists
identical ordinal by ordinal, and every returned split is verified feasible
with equal cost."""
import json
import os

import pytest

import oracle_bind as ob
from dag_gen import random_dag
from golden_io import GOLDEN, config_from_case, graph_from_json, load, rat_from_json
from paper_2006_16423_b200 import _abi, solver
from paper_2006_16423_b200 import workloads as wl
from paper_2006_16423_b200.errors import (DeadlineExceeded, IdealBudgetExceeded, InfeasibleError,
                                          Unsupported)
from paper_2006_16423_b200.graph import INF, DeviceConfig, Interleaving, verify_split

pytestmark = pytest.mark.gpu

CORPUS = load("dp_corpus.json")
IDEALS = load("ideals.json")


def device_solve(mode, g, cfg, flags=0, **kw):
    opt = solver.SolveOptions(flags=flags, **kw)
    f = solver.solve_maxload_training if mode == 1 else solver.solve_maxload_inference
    return f(g, cfg, opt)


def device_obj(mode, g, cfg, flags=0):
    try:
        split = device_solve(mode, g, cfg, flags)
    except InfeasibleError:
        return INF, None
    problems = verify_split(g, cfg, split, training=(mode == 1 and g.has_backward_nodes()))
    assert not problems, problems
    return split.objective_value, split


@pytest.mark.parametrize("case", CORPUS, ids=[c["name"] for c in CORPUS])
def test_golden_objective(gpu, case):
    g = graph_from_json(case["graph"])
    cfg = config_from_case(case)
    obj, split = device_obj(case["mode"], g, cfg)
    assert obj == rat_from_json(case["objective"])


@pytest.mark.parametrize("flags", [_abi.DSG_FLAG_FORCE_INT64, _abi.DSG_FLAG_NO_FASTGATE])
def test_golden_objective_alternate_paths(gpu, flags):
    """64-bit value path and the general backward-contiguity gate agree too."""
    for case in CORPUS[::3]:
        g = graph_from_json(case["graph"])
        cfg = config_from_case(case)
        obj, _ = device_obj(case["mode"], g, cfg, flags)
        assert obj == rat_from_json(case["objective"]), case["name"]


@pytest.mark.parametrize("flags,max_blocks", [(_abi.DSG_FLAG_LEVEL_LAUNCH, 0), (0, 1), (0, 3),
                                               (_abi.DSG_FLAG_FORCE_INT64, 2)],
                         ids=["level-launch", "persistent-1cta", "persistent-3cta", "int64-2cta"])
def test_driver_variants_match_golden(gpu, flags, max_blocks):
    """Per-level launches and tiny persistent grids (every CTA owns many work
    items, exercising the tile counters and the grid barrier) agree."""
    for case in CORPUS[::5]:
        g = graph_from_json(case["graph"])
        cfg = config_from_case(case)
        f = solver.solve_maxload_training if case["mode"] == 1 else solver.solve_maxload_inference
        try:
            got = f(g, cfg, solver.SolveOptions(flags=flags, max_blocks=max_blocks)).objective_value
        except InfeasibleError:
            got = INF
        assert got == rat_from_json(case["objective"]), case["name"]


def test_standin_driver_variants_agree(gpu):
    w = wl.standin("C3")
    base = device_solve(1, w.graph, w.config)
    for flags, mb in [(_abi.DSG_FLAG_LEVEL_LAUNCH, 0), (0, 5), (_abi.DSG_FLAG_FORCE_INT64, 0)]:
        s = solver.solve_maxload_training(w.graph, w.config,
                                          solver.SolveOptions(flags=flags, max_blocks=mb))
        assert s.objective_value == base.objective_value
        assert s.stats["n_pairs"] == base.stats["n_pairs"]


@pytest.mark.parametrize("hash_mode", [False, True], ids=["canonical", "hashset"])
@pytest.mark.parametrize("case", IDEALS, ids=[c["name"] for c in IDEALS])
def test_golden_ideal_lists(gpu, case, hash_mode):
    g = graph_from_json(case["graph"])
    flags = _abi.DSG_FLAG_HASH_ENUM if hash_mode else 0
    run = (lambda: solver.enumerate_ideals_within(g, case["within"], case["budget"], flags)) \
        if case["within"] is not None else (lambda: solver.enumerate_ideals(g, case["budget"], flags))
    if "error" in case:
        with pytest.raises(IdealBudgetExceeded):
            run()
        return
    ix = run()
    assert [[int(x) for x in r] for r in ix.bits] == case["ideals"]
    assert [int(x) for x in ix.level_offsets] == case["level_offsets"]


@pytest.mark.parametrize("seed", range(60))
def test_random_dags_match_oracle(gpu, seed):
    g, cfg = random_dag(seed)
    want = ob.objective_or_inf("port", 0, g, cfg)
    got, _ = device_obj(0, g, cfg)
    assert got == want


@pytest.mark.parametrize("seed", range(40))
def test_random_training_dags_match_oracle(gpu, seed):
    g, cfg = random_dag(1000 + seed, n_lo=4, n_hi=11, training=True)
    want = ob.objective_or_inf("port", 1, g, cfg)
    got, _ = device_obj(1, g, cfg)
    assert got == want
    got2, _ = device_obj(1, g, cfg, _abi.DSG_FLAG_NO_FASTGATE)
    assert got2 == want


@pytest.mark.parametrize("k,l", [(0, 2), (3, 0), (16, 0), (12, 1), (2, 6), (5, 3), (8, 4), (9, 5)])
def test_cell_shapes_match_oracle(gpu, k, l):
    """Every (K+1)x(L+1) specialisation and the generic shared-memory path."""
    for seed in range(6):
        g, cfg = random_dag(500 + seed, n_lo=8, n_hi=16)
        cfg.accelerators, cfg.cpus = k, l
        want = ob.objective_or_inf("port", 0, g, cfg)
        got, _ = device_obj(0, g, cfg)
        assert got == want, (seed, k, l)


def test_fine_and_coarse_denominators(gpu):
    for seed in range(10):
        g, cfg = random_dag(3000 + seed, den=1000)
        assert device_obj(0, g, cfg)[0] == ob.objective_or_inf("port", 0, g, cfg)
    # weights large enough to force the 64-bit value path
    g, cfg = random_dag(4000, den=7)
    for nd in g.nodes():
        if nd.cpu_time != INF:
            nd.cpu_time = nd.cpu_time * 10 ** 9
    g = wl.Graph(g.nodes(), g.edges(), g.artificial_edges())
    split = None
    got, split = device_obj(0, g, cfg)
    assert got == ob.objective_or_inf("port", 0, g, cfg)


def test_known_answers(gpu):
    d4 = wl.diamond4()
    assert device_solve(0, d4, DeviceConfig(2, 0, 4)).objective_value == 6
    split = device_solve(0, d4, DeviceConfig(2, 0, 4))
    blocks = {frozenset(i for i, p in split.assignment.items() if p == pl)
              for pl in split.assignment.values()}
    assert blocks in ({frozenset({1, 2}), frozenset({3, 4})}, {frozenset({1, 3}), frozenset({2, 4})})
    tr = wl.mirror_training(d4)
    split = device_solve(1, tr, DeviceConfig(2, 0, 8))
    assert split.objective_value == 12
    for n in tr.nodes():
        if n.is_backward:
            assert split.assignment[n.id] == split.assignment[n.forward_pair]
    with pytest.raises(InfeasibleError):
        device_solve(0, wl.Graph([wl.make_node(1, 1, 1, 0, 10)]), DeviceConfig(1, 0, 4))


def test_error_semantics(gpu):
    d4 = wl.diamond4()
    with pytest.raises(ValueError, match="at least one device"):
        device_solve(0, d4, DeviceConfig(0, 0, 4))
    unpaired = wl.Graph([wl.Node(id=1), wl.Node(id=2, is_backward=True)])
    with pytest.raises(ValueError, match="paired"):
        device_solve(1, unpaired, DeviceConfig(1, 0, 4))
    dangling = wl.Graph([wl.Node(id=1), wl.Node(id=2, is_backward=True, forward_pair=7)])
    with pytest.raises(ValueError, match="missing node"):
        device_solve(1, dangling, DeviceConfig(1, 0, 4))
    with pytest.raises(IdealBudgetExceeded) as ei:
        device_solve(0, wl.edgeless(20), DeviceConfig(2, 0, 100), ideal_budget=1000)
    assert ei.value.limit == 1000
    with pytest.raises(ValueError, match="infinity"):
        device_solve(0, wl.Graph([wl.make_node(1, INF, 1, 0, 1)]), DeviceConfig(1, 1, 4))
    from paper_2006_16423_b200.errors import MissingBandwidth
    with pytest.raises(MissingBandwidth):
        solver.solve_maxload_replicated(d4, DeviceConfig(2, 0, 4))
    with pytest.raises(ValueError, match="inference graph"):
        solver.solve_maxload_replicated(wl.mirror_training(d4), DeviceConfig(2, 0, 4, bandwidth=1))


def test_replication_known_answers(gpu):
    """test_dp_solver.cpp:145-164: one block of base 10, weight 4."""
    from paper_2006_16423_b200.graph import ReplicationCombine
    g = wl.Graph([wl.make_node(1, 10, 10, 0, 4)])
    s = solver.solve_maxload_replicated(g, DeviceConfig(2, 0, 4, bandwidth=1))
    assert s.objective_value == 7 and s.replication == {"acc1": 2}
    s = solver.solve_maxload_replicated(
        g, DeviceConfig(2, 0, 4, bandwidth=1, replication_combine=ReplicationCombine.Max))
    assert s.objective_value == 5
    assert solver.solve_maxload_replicated(g, DeviceConfig(1, 0, 4, bandwidth=1)).objective_value == 10


@pytest.mark.parametrize("seed", range(40))
def test_replication_matches_oracle(gpu, seed):
    from fractions import Fraction
    from paper_2006_16423_b200.graph import ReplicationCombine
    g, cfg = random_dag(7000 + seed, n_lo=4, n_hi=12)
    cfg.accelerators = 1 + seed % 5
    cfg.bandwidth = [Fraction(1), Fraction(3, 2), Fraction(1000000), Fraction(1, 7)][seed % 4]
    cfg.replication_combine = ReplicationCombine(seed % 2)
    try:
        want = ob.dp("port", 2, g, cfg).objective
    except InfeasibleError:
        want = INF
    try:
        split = solver.solve_maxload_replicated(g, cfg)
        got = split.objective_value
        assert not verify_split(g, cfg, split, training=False)
    except InfeasibleError:
        got = INF
    assert got == want


def test_deadline(gpu):
    w = wl.standin("C2")
    with pytest.raises(DeadlineExceeded):
        device_solve(0, w.graph, w.config, deadline_seconds=1e-4)


def test_ideal_count_and_order_properties(gpu):
    """subset-before-superset and brute-force count (test_graph_core.cpp:123-139)."""
    for seed in range(15):
        g = wl.random_instance(seed).graph
        ix = solver.enumerate_ideals(g)
        ideals = ix.ideals
        n = g.size()
        naive = sum(1 for m in range(1 << n)
                    if all((m >> u) & 1 for v in range(n) if (m >> v) & 1 for u in g.in_all(v)))
        assert len(ideals) == naive
        for i in range(len(ideals)):
            for j in range(i + 1, len(ideals)):
                assert not ideals[j] <= ideals[i]


STANDINS = os.path.join(GOLDEN, "standins.json")


@pytest.mark.skipif(not os.path.exists(STANDINS), reason="standins.json not generated")
def test_standins_match_reference(gpu):
    for row in json.load(open(STANDINS)):
        if row["name"].startswith("sweep"):
            w = wl.sweep(*row["point"])
        else:
            w = wl.standin(row["name"])
        split = device_solve(1 if w.training else 0, w.graph, w.config)
        assert split.objective_value == rat_from_json(row["objective"]), row["name"]
        assert split.stats["n_ideals"] == row["ideals"]
        assert split.stats["n_pairs"] == row["pairs"]
        assert not verify_split(w.graph, w.config, split, training=w.training)


@pytest.mark.parametrize("pt", [(2, 8, 20, 100), (4, 4, 20, 300), (16, 1, 1, 300)])
def test_sweep_pair_counts(gpu, pt):
    """Size-independent check at sweep sizes: transitions == closed form."""
    w = wl.sweep(*pt)
    split = device_solve(0, w.graph, w.config)
    nv, ni, npairs = wl.chain_counts(w.spec)
    assert split.stats["n_ideals"] == ni
    assert split.stats["n_pairs"] == npairs
    assert not verify_split(w.graph, w.config, split, training=False)


def test_repeat_solves_are_deterministic(gpu):
    w = wl.standin("C3")
    a = device_solve(1, w.graph, w.config)
    b = device_solve(1, w.graph, w.config)
    assert a.assignment == b.assignment and a.objective_value == b.objective_value


def test_sharded_protocol_single_rank(gpu):
    """dsg_session_shard_{prepare,attach,reset} + run at world 1: the same
    phase split, reset/run protocol and peer-table indirection as N GPUs."""
    from paper_2006_16423_b200.solver import ShardComm, ShardedSession
    comm = ShardComm(0, 1, lambda b: [b], lambda: None)
    for name in ("C3", "C1"):
        w = wl.standin(name)
        ref = device_solve(1 if w.training else 0, w.graph, w.config)
        s = ShardedSession(1 if w.training else 0, w.graph, w.config, comm)
        for _ in range(2):
            raw = s.run()
            assert raw.objective == ref.objective_value
            assert raw.n_pairs == ref.stats["n_pairs"]
        s.close()
    g, cfg = random_dag(42)
    s = ShardedSession(0, g, cfg, comm)
    try:
        got = s.run().objective
    except InfeasibleError:
        got = INF
    assert got == ob.objective_or_inf("port", 0, g, cfg)


def test_replication_sync_term_no_overflow(gpu):
    """the sync term (r-1)/r * mem / B formed (mem*(r-1)) before
    dividing and wrapped the 32-bit path at K >= 8.  One node, cpu = acc = 1,
    mem = 300, K = 16, bandwidth 1: the reference answer is 1."""
    from fractions import Fraction
    g = wl.Graph([wl.make_node(1, 1, 1, 0, 300)])
    for k in (8, 12, 16):
        cfg = DeviceConfig(k, 0, INF, bandwidth=Fraction(1))
        want = ob.dp("port", 2, g, cfg).objective
        assert want == 1
        s = solver.solve_maxload_replicated(g, cfg)
        assert s.objective_value == want, k
    for seed in range(8):
        gr, cfg = random_dag(7100 + seed, n_lo=4, n_hi=9)
        cfg.accelerators = 9 + seed % 8
        cfg.bandwidth = [Fraction(1), Fraction(3, 2), Fraction(1, 7)][seed % 3]
        for nd in gr.nodes():
            nd.mem_size = nd.mem_size * 50
        gr = wl.Graph(gr.nodes(), gr.edges(), gr.artificial_edges())
        cfg.memory_limit = INF
        try:
            got = solver.solve_maxload_replicated(gr, cfg).objective_value
        except InfeasibleError:
            got = INF
        assert got == ob.objective_or_inf("port", 2, gr, cfg), seed


def test_negative_comm_under_sum(gpu):
    """the exact pruning assumes acc(B) >= proc(B); negative comm
    weights under Interleaving::Sum break that, so those solves run unpruned
    and still equal the oracle."""
    from fractions import Fraction
    for seed in range(12):
        g, cfg = random_dag(7300 + seed, n_lo=5, n_hi=12)
        for i, nd in enumerate(g.nodes()):
            if nd.comm_time != INF and i % 2 == 0:
                nd.comm_time = -nd.comm_time - Fraction(1, 2)
        g = wl.Graph(g.nodes(), g.edges(), g.artificial_edges())
        for mode in (Interleaving.Sum, Interleaving.HalfDuplexMax):
            cfg.interleaving = mode
            want = ob.objective_or_inf("port", 0, g, cfg)
            try:
                got = device_solve(0, g, cfg).objective_value
            except InfeasibleError:
                got = INF
            assert got == want, (seed, mode)


def test_large_cell_grid_falls_back(gpu):
    """replicated K=16, L=8 (153 cells) with 64-bit values needs
    more shared memory than a persistent CTA has; the solve must fall back to
    the per-level driver instead of failing the launch."""
    from fractions import Fraction
    g, cfg = random_dag(7400, n_lo=6, n_hi=10)
    cfg.accelerators, cfg.cpus = 16, 8
    cfg.bandwidth = Fraction(3, 2)
    want = ob.objective_or_inf("port", 2, g, cfg)
    try:
        got = solver.solve_maxload_replicated(
            g, cfg, solver.SolveOptions(flags=_abi.DSG_FLAG_FORCE_INT64)).objective_value
    except InfeasibleError:
        got = INF
    assert got == want


HOST_REF = os.path.join(GOLDEN, "host_reference.json")


@pytest.mark.skipif(not os.path.exists(HOST_REF), reason="host_reference.json not generated")
def test_full_size_objectives_match_reference(gpu):
    """Objectives of the unmodified reference on full workloads, solved on the
    bench host (tools/cpu_ref_host.sh): the C5 top point (943.5M transitions),
    the 3 %-dense sweep point (16,1,1,300), a second weight seed and D = 1000
    weights for C2, C1-C4, and a wide-bitset sweep point (16,1,1,1300: W = 21,
    66,838 ideals; solved by the reference in the build container)."""
    for row in json.load(open(HOST_REF)):
        w = wl.by_name(row["workload"])
        split = device_solve(1 if w.training else 0, w.graph, w.config)
        assert str(split.objective_value) == row["objective"], row["workload"]
        assert split.stats["n_ideals"] == row["ideals"]
        assert split.stats["n_pairs"] == row["pairs_closed_form"]
        assert not verify_split(w.graph, w.config, split, training=w.training)


@pytest.mark.parametrize("name", ["C2", "C5:16,1,1,300", "C5:4,4,8,1400"])
def test_int64_exact_variants(gpu, name):
    """The 64-bit exact-word kernels (K = 8, L = 0, AW = 6 / 6 / 26->generic):
    the same objective and transition count as the 32-bit path, which the
    host-reference objectives pin for the first two."""
    w = wl.by_name(name)
    base = solver.solve_maxload_inference(w.graph, w.config)
    s = solver.solve_maxload_inference(w.graph, w.config,
                                       solver.SolveOptions(flags=_abi.DSG_FLAG_FORCE_INT64))
    assert s.stats["value_bits"] == 64 and base.stats["value_bits"] == 32
    assert s.objective_value == base.objective_value
    assert s.stats["n_pairs"] == base.stats["n_pairs"]
    assert not verify_split(w.graph, w.config, s, training=False)
