"""Workload generators: the builder port is bit-exact against the compiled
reference builders, and the stand-ins hit the paper's node/ideal counts."""
from fractions import Fraction

import pytest

import oracle_bind as ob
from golden_io import load, rat_from_json
from paper_2006_16423_b200 import workloads as wl

DUMP = load("random_instances.json")


@pytest.mark.parametrize("key,allow", [("allow_unsupported", True), ("supported_only", False)])
def test_random_instance_port_is_bit_exact(key, allow):
    for row in DUMP[key]:
        inst = wl.random_instance(row["seed"], allow_unsupported=allow)
        g = inst.graph
        assert inst.config.accelerators == row["k"]
        assert inst.config.cpus == row["l"]
        assert inst.config.memory_limit == Fraction(row["M"][0], row["M"][1])
        nodes = [[n.id] + [[v.numerator, v.denominator] if v != wl.INF else [1, 0]
                           for v in (n.cpu_time, n.acc_time, n.comm_time, n.mem_size)]
                 for n in g.nodes()]
        assert nodes == row["nodes"], row["seed"]
        assert [[e.src, e.dst] for e in g.edges()] == row["edges"]


def test_splitmix64_known_values():
    r = wl.SplitMix64(0)
    # reference constants (rng.hpp:62-67)
    assert r.next() == 0xE220A8397B1DCDAF
    assert r.next() == 0x6E789E6AA1B965F4


@pytest.mark.parametrize("name,nodes,ideals,pairs", [
    ("C1", 177, 242, 28_729),
    ("C2", 326, 36_596, 563_731_351),
    ("C3", 96, 17_914, 45_900_843),
    ("C4", 1_516, 4_013, None),
])
def test_standin_closed_forms(name, nodes, ideals, pairs):
    nv, ni, npairs = wl.chain_counts(wl.SPECS[name])
    assert (nv, ni) == (nodes, ideals)
    if pairs is not None:
        assert npairs == pairs
    g = wl.module_chain(wl.SPECS[name])
    assert g.size() == nodes


def test_c2_matches_survey_recipe():
    g = wl.module_chain(wl.SPECS["C2"])
    assert len(g.edges()) == 356


@pytest.mark.parametrize("pt,expect", [((2, 8, 20, 100), (441, 1_722, 1_460_000)),
                                       ((8, 2, 7, 600), (720, 46_529, 944_000_000))])
def test_sweep_closed_forms(pt, expect):
    nv, ni, npairs = wl.chain_counts(wl.sweep_spec(*pt))
    assert (nv, ni) == expect[:2]
    assert abs(npairs - expect[2]) / expect[2] < 0.01


@pytest.mark.skipif(not ob.available("port"), reason="oracle not built")
def test_closed_form_pairs_match_oracle_walk():
    """The oracle's apply_candidate count equals the closed-form pair count."""
    spec = wl.ChainSpec(3, [[2, 1], [3, 0, 2]], 2)
    g = wl.module_chain(spec)
    raw = ob.dp("port", 0, g, wl.DeviceConfig(3, 1, 1000))
    nv, ni, npairs = wl.chain_counts(spec)
    assert raw.n_ideals == ni
    assert raw.n_pairs == npairs
