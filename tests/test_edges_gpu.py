"""Edge cases at the size limits: the empty graph, one node, ragged word
counts (|V| = 63, 64, 65, 127, 128, 129) against the oracle port, the
4,096-node maximum (64 words) against an independent path checker, and the
unsupported size above it."""
import pytest

import oracle_bind as ob
from chain_check import path_maxload, random_path
from paper_2006_16423_b200 import solver
from paper_2006_16423_b200 import workloads as wl
from paper_2006_16423_b200.errors import InfeasibleError, Unsupported
from paper_2006_16423_b200.graph import INF, DeviceConfig, Graph, verify_split


def test_path_checker_matches_oracle():
    """Pin the path checker against the oracle port on small paths."""
    for seed in range(12):
        n = 5 + seed * 3
        g, acc, comm, mem = random_path(n, seed)
        K, M = 1 + seed % 5, int(mem.sum()) // 2 + 3
        want = path_maxload(acc, comm, mem, K, M)
        try:
            got = ob.dp("port", 0, g, DeviceConfig(K, 0, M)).objective
        except InfeasibleError:
            got = INF
        assert (got == INF) if want >= 2 ** 60 else (got == want)



@pytest.mark.gpu
def test_empty_graph(gpu):
    split = solver.solve_maxload_inference(Graph([]), DeviceConfig(1, 0, 4))
    ref = ob.dp("port", 0, Graph([]), DeviceConfig(1, 0, 4))
    assert split.objective_value == ref.objective == 0
    assert split.assignment == {}
    assert solver.enumerate_ideals(Graph([])).count() == 1


@pytest.mark.gpu
def test_single_node(gpu):
    g = Graph([wl.make_node(7, 3, 2, 5, 1)])
    for K, L in ((1, 0), (0, 1), (2, 1)):
        cfg = DeviceConfig(K, L, 4)
        split = solver.solve_maxload_inference(g, cfg)
        assert split.objective_value == ob.dp("port", 0, g, cfg).objective
        assert not verify_split(g, cfg, split, training=False)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [63, 64, 65, 127, 128, 129])
def test_ragged_word_counts(gpu, n):
    stem = n - 9  # one module [3, 2]: split + 5 branch nodes + join + 2 tail
    g = wl.module_chain(wl.ChainSpec(stem, [[3, 2]], 2))
    assert g.size() == n
    cfg = DeviceConfig(4, 1, 10 ** 6)
    split = solver.solve_maxload_inference(g, cfg)
    assert split.objective_value == ob.dp("port", 0, g, cfg).objective
    assert not verify_split(g, cfg, split, training=False)
    tr = wl.mirror_training(g)
    cfg = DeviceConfig(3, 1, 10 ** 6)
    split = solver.solve_maxload_training(tr, cfg)
    assert split.objective_value == ob.dp("port", 1, tr, cfg).objective
    assert not verify_split(tr, cfg, split, training=True)


@pytest.mark.gpu
@pytest.mark.parametrize("n,K", [(4096, 8), (3000, 5)])
def test_maximum_size_path(gpu, n, K):
    g, acc, comm, mem = random_path(n, n)
    M = int(mem.sum()) // K + 40
    split = solver.solve_maxload_inference(g, DeviceConfig(K, 0, M))
    assert split.objective_value == path_maxload(acc, comm, mem, K, M)
    assert split.stats["n_ideals"] == n + 1
    assert split.stats["n_pairs"] == (n + 1) * n // 2
    assert not verify_split(g, DeviceConfig(K, 0, M), split, training=False)


@pytest.mark.gpu
def test_above_maximum_size_is_unsupported(gpu):
    g, *_ = random_path(4097, 1)
    with pytest.raises(Unsupported):
        solver.solve_maxload_inference(g, DeviceConfig(2, 0, 10 ** 6))


def _coprime_chain(dens):
    from fractions import Fraction as F
    from paper_2006_16423_b200.graph import Edge, Node
    nodes = [Node(i + 1, F(1, d), F(1, d), F(1, d), F(1, d)) for i, d in enumerate(dens)]
    return Graph(nodes, [Edge(i + 1, i + 2) for i in range(len(dens) - 1)])


@pytest.mark.gpu
@pytest.mark.parametrize("dens", [[2097143, 2097091], [2 ** 20, 3 ** 12, 5 ** 8]])
def test_large_denominators_match_oracle(gpu, dens):
    """Weights whose common denominator is large but <= 2^62: exact and equal
    to the reference (rational.cpp arithmetic)."""
    from fractions import Fraction as F
    g = _coprime_chain(dens)
    cfg = DeviceConfig(accelerators=2, memory_limit=F(10))
    split = solver.solve_maxload_inference(g, cfg)
    assert split.objective_value == ob.dp("port", 0, g, cfg).objective
    assert not verify_split(g, cfg, split, training=False)


@pytest.mark.gpu
def test_common_denominator_above_2_62_is_overflow(gpu):
    """The documented boundary of the fixed-point design: three
    ~2^21 primes as weight denominators give a common denominator ~2^63.  The
    reference still solves this instance (its Rat reduces pairwise sums), the
    B200 path reports std::overflow_error (DSG_OVERFLOW) instead of a wrong
    value."""
    from fractions import Fraction as F
    g = _coprime_chain([2097143, 2097091, 2097083])
    cfg = DeviceConfig(accelerators=2, memory_limit=F(10))
    assert ob.dp("port", 0, g, cfg).objective == F(6291377, 4397899711013)
    with pytest.raises(OverflowError):
        solver.solve_maxload_inference(g, cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [600, 700, 1000, 1500, 2000])
def test_exact_word_variants_wide(gpu, n):
    """K = 8, L = 0 inference on 600 to 2,000 nodes: the exact-word
    kernels for AW = 10, 12, 16, 24 and 32 (persistent_x_i32_inf.cu) against the
    oracle port; one module keeps the lattice small."""
    stem = n - 9
    g = wl.module_chain(wl.ChainSpec(stem, [[3, 2]], 2))
    assert g.size() == n
    cfg = DeviceConfig(8, 0, 10 ** 6)
    split = solver.solve_maxload_inference(g, cfg)
    assert split.objective_value == ob.dp("port", 0, g, cfg).objective
    assert not verify_split(g, cfg, split, training=False)
