"""(De)serialisation of graphs and exact values for the golden fixtures."""
from __future__ import annotations

import json
import os
from fractions import Fraction

from paper_2006_16423_b200.graph import INF, DeviceConfig, Edge, Graph, Interleaving, Node, is_inf

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rat_to_json(x) -> str:
    if is_inf(x):
        return "inf"
    f = Fraction(x)
    return str(f.numerator) if f.denominator == 1 else f"{f.numerator}/{f.denominator}"


def rat_from_json(s):
    if s == "inf":
        return INF
    return Fraction(s)


def graph_to_json(g: Graph) -> dict:
    nodes = []
    for n in g.nodes():
        row = [n.id, rat_to_json(n.cpu_time), rat_to_json(n.acc_time), rat_to_json(n.comm_time),
               rat_to_json(n.mem_size)]
        if n.is_backward:
            row += [1, n.forward_pair]
        nodes.append(row)
    return dict(nodes=nodes, edges=[[e.src, e.dst] for e in g.edges()],
                art=[[e.src, e.dst] for e in g.artificial_edges()])


def graph_from_json(d: dict) -> Graph:
    nodes = []
    for row in d["nodes"]:
        n = Node(id=row[0], cpu_time=rat_from_json(row[1]), acc_time=rat_from_json(row[2]),
                 comm_time=rat_from_json(row[3]), mem_size=rat_from_json(row[4]))
        if len(row) > 5:
            n.is_backward = bool(row[5])
            n.forward_pair = row[6]
        nodes.append(n)
    return Graph(nodes, [Edge(a, b) for a, b in d["edges"]], [Edge(a, b) for a, b in d.get("art", [])])


def config_from_case(c: dict) -> DeviceConfig:
    return DeviceConfig(accelerators=c["k"], cpus=c["l"], memory_limit=rat_from_json(c["M"]),
                        interleaving=Interleaving(c.get("interleaving", 0)))


def load(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)
