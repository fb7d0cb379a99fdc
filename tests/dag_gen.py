"""Test-only random DAG generator for oracle-vs-device parity beyond the
reference corpus: skip edges, artificial edges, infinite-comm sentinels,
unsupported nodes, several weight denominators, training twins with extra
backward edges (so the general contiguity gate is exercised)."""
from __future__ import annotations

from fractions import Fraction

from paper_2006_16423_b200.graph import INF, DeviceConfig, Edge, Graph, Interleaving, Node
from paper_2006_16423_b200.workloads import SplitMix64


def random_dag(seed: int, n_lo: int = 6, n_hi: int = 22, training: bool = False,
               den: int = 2, inf_comm: bool = True) -> tuple:
    rng = SplitMix64(seed * 7919 + 17)
    n = n_lo + rng.below(n_hi - n_lo + 1)
    nodes = []
    for i in range(1, n + 1):
        cpu = Fraction(rng.below(20 * den), den)
        acc = Fraction(rng.below(10 * den), den)
        comm = Fraction(rng.below(6 * den), den)
        mem = Fraction(1 + rng.below(5))
        nd = Node(id=i, cpu_time=cpu, acc_time=acc, comm_time=comm, mem_size=mem)
        if rng.below(12) == 0:
            nd.acc_time = INF
        if inf_comm and rng.below(15) == 0:
            nd.comm_time = INF
        nodes.append(nd)
    edges, art = [], []
    seen = set()
    width = 1 + rng.below(4)
    for v in range(2, n + 1):
        # a few predecessors among the previous `width*2` nodes (layered-ish)
        for _ in range(1 + rng.below(2)):
            u = max(1, v - 1 - rng.below(width * 2))
            if u < v and (u, v) not in seen:
                seen.add((u, v))
                (art if rng.below(8) == 0 else edges).append(Edge(u, v))
    for _ in range(rng.below(4)):  # long skip edges
        u = 1 + rng.below(n)
        v = 1 + rng.below(n)
        if u < v and (u, v) not in seen:
            seen.add((u, v))
            edges.append(Edge(u, v))
    g = Graph(nodes, edges, art)
    total_mem = sum((nd.mem_size for nd in nodes), Fraction(0))
    k = rng.below(5)
    l = rng.below(4) if k else 1 + rng.below(3)
    cfg = DeviceConfig(accelerators=k, cpus=l,
                       memory_limit=total_mem * Fraction(3 + rng.below(10), 10),
                       interleaving=Interleaving(rng.below(3)))
    if training:
        off = n
        bnodes = []
        for nd in nodes:
            b = Node(**vars(nd))
            b.id = nd.id + off
            b.is_backward = True
            b.forward_pair = nd.id
            bnodes.append(b)
        bedges = [Edge(e.dst + off, e.src + off) for e in edges]
        bedges += [Edge(e.dst + off, e.src + off) for e in art]
        if rng.below(3) == 0:  # an extra backward edge that breaks the mirror symmetry
            a = 1 + rng.below(n)
            b = 1 + rng.below(n)
            if a != b:  # reversed-topological like the mirror, so still acyclic
                bedges.append(Edge(max(a, b) + off, min(a, b) + off))
        fwbw = [Edge(n, 2 * n)] if n > 1 else []
        g = Graph(nodes + bnodes, edges + bedges + fwbw, art)
        cfg.memory_limit = cfg.memory_limit * 2
    return g, cfg
