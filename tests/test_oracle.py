"""Pin the checker before trusting it: the C restatement (oracle/_build) must
reproduce every golden vector dumped from the unmodified reference, and, where
the compiled reference (oracle/_ref) is present, agree with it directly."""
import pytest

import oracle_bind as ob
from golden_io import config_from_case, graph_from_json, load, rat_from_json
from paper_2006_16423_b200.errors import IdealBudgetExceeded, InfeasibleError
from paper_2006_16423_b200.graph import INF, DeviceConfig, recompute_maxload
from paper_2006_16423_b200 import workloads as wl

pytestmark = pytest.mark.skipif(not ob.available("port"), reason="oracle not built (make -C oracle)")

CORPUS = load("dp_corpus.json")
IDEALS = load("ideals.json")


def _obj(kind, case):
    g = graph_from_json(case["graph"])
    cfg = config_from_case(case)
    try:
        return ob.dp(kind, case["mode"], g, cfg).objective
    except InfeasibleError:
        return INF


@pytest.mark.parametrize("case", CORPUS, ids=[c["name"] for c in CORPUS])
def test_port_matches_golden_objective(case):
    assert _obj("port", case) == rat_from_json(case["objective"])
    if "expect" in case:
        assert case["objective"] == case["expect"]


@pytest.mark.parametrize("case", IDEALS, ids=[c["name"] for c in IDEALS])
def test_port_ideal_list_matches_golden(case):
    g = graph_from_json(case["graph"])
    if "error" in case:
        with pytest.raises(IdealBudgetExceeded):
            ob.enumerate_ideals("port", g, case["within"], case["budget"])
        return
    ix = ob.enumerate_ideals("port", g, case["within"], case["budget"])
    assert [[int(x) for x in r] for r in ix.bits] == case["ideals"]
    assert [int(x) for x in ix.level_offsets] == case["level_offsets"]


def test_port_split_reproduces_objective():
    """reported loads reproduce the objective (test_dp_solver.cpp:340-357)."""
    for seed in range(700, 720):
        inst = wl.random_instance(seed)
        try:
            split, _ = ob.solve("port", 0, inst.graph, inst.config)
        except InfeasibleError:
            continue
        _, worst = recompute_maxload(inst.graph, inst.config, split)
        assert worst == split.objective_value


@pytest.mark.skipif(not ob.available("ref"), reason="oracle/_ref not built")
def test_port_and_reference_choose_identical_splits():
    """Same visit order => same tie-breaking => identical assignments."""
    for seed in range(60):
        inst = wl.random_instance(seed)
        try:
            a, _ = ob.solve("port", 0, inst.graph, inst.config)
        except InfeasibleError:
            continue
        b, _ = ob.solve("ref", 0, inst.graph, inst.config)
        assert a.assignment == b.assignment
        assert a.objective_value == b.objective_value


def test_port_error_semantics():
    d4 = wl.diamond4()
    with pytest.raises(ValueError):
        ob.dp("port", 0, d4, DeviceConfig(0, 0, 4))  # need at least one device
    bad = wl.mirror_training(d4)
    bad.nodes()[5].forward_pair = None
    bad = wl.Graph(bad.nodes(), bad.edges())
    with pytest.raises(ValueError):
        ob.dp("port", 1, bad, DeviceConfig(2, 0, 8))
    with pytest.raises(IdealBudgetExceeded):
        ob.dp("port", 0, wl.edgeless(12), DeviceConfig(2, 0, 100), ob.SolveOptions(ideal_budget=100))
