"""DPL row of SURVEY 8(f): seeded_topo_order / linearize / solve_dpl
(dp_solver.hpp:39-52) pinned to tests/golden/dpl.json, which
make_dpl_golden.py dumped from the unmodified reference."""
import pytest

import oracle_bind as ob
from golden_io import config_from_case, graph_from_json, load, rat_from_json
from paper_2006_16423_b200 import solver
from paper_2006_16423_b200 import workloads as wl
from paper_2006_16423_b200.errors import InfeasibleError
from paper_2006_16423_b200.graph import INF, verify_split

DPL = load("dpl.json")
IDS = [c["name"] for c in DPL]


@pytest.mark.parametrize("case", DPL, ids=IDS)
def test_topo_order_matches_reference(case):
    g = graph_from_json(case["graph"])
    assert solver.seeded_topo_order(g, case["seed"]) == case["order"]


def test_linearize_collapses_lattice_to_prefixes():
    g = wl.random_instance(3).graph
    lin = solver.linearize(g, 5)
    assert ob.available("port")
    ix = ob.enumerate_ideals("port", lin)
    assert ix.count() == g.size() + 1
    # artificial only: real edges (and so every comm term) are unchanged
    assert [(e.src, e.dst) for e in lin.edges()] == [(e.src, e.dst) for e in g.edges()]


@pytest.mark.skipif(not ob.available("port"), reason="oracle not built")
@pytest.mark.parametrize("case", DPL, ids=IDS)
def test_port_on_chained_graph_matches_reference_dpl(case):
    """The checker for the GPU test below: oracle port DP over the chain."""
    g = graph_from_json(case["graph"])
    cfg = config_from_case(case)
    training = g.has_backward_nodes()
    order = [v for v in case["order"] if not (training and g.node(v).is_backward)]
    chained = solver._chain_along(g, order)
    try:
        obj = ob.dp("port", int(training), chained, cfg).objective
    except InfeasibleError:
        obj = INF
    assert obj == rat_from_json(case["objective"])


@pytest.mark.skipif(not ob.available("ref"), reason="oracle/_ref not built")
def test_topo_order_random_seeds_vs_reference():
    for i in range(30):
        g = wl.random_instance(300 + i).graph
        for seed in (0, 2**63 + 11, i):
            assert solver.seeded_topo_order(g, seed) == ob.ref_topo_order(g, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("case", DPL, ids=IDS)
def test_device_dpl_matches_reference(gpu, case):
    g = graph_from_json(case["graph"])
    cfg = config_from_case(case)
    want = rat_from_json(case["objective"])
    try:
        split = solver.solve_dpl(g, cfg, case["seed"])
    except InfeasibleError:
        assert want == INF
        return
    assert split.objective_value == want
    problems = verify_split(g, cfg, split, training=g.has_backward_nodes())
    assert not problems, problems
