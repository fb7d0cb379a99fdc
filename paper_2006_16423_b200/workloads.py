"""Synthetic workloads: reference test fixtures and the BASELINE config stand-ins.

* ``SplitMix64``           include/dagsplit/rng.hpp:55-75 (bit-exact)
* ``diamond4`` / ``mirror_training`` / ``path_graph`` / ``edgeless`` /
  ``random_instance``      tests/support/builders.cpp:80-158 (bit-exact; the
                           corpus behind AC-1/AC-2 and test_dp_solver.cpp)
* ``module_chain`` and the C1..C5 stand-ins of SURVEY.md §8(d): the named
  workload graphs (ResNet-50, InceptionV3, GNMT, BERT-24) are absent from the
  reference (proj/workloads holds only diamond*.json), so these chains
  reproduce the paper's node and ideal counts exactly.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

from .graph import INF, DeviceConfig, Edge, Graph, Node, make_node

MASK64 = (1 << 64) - 1


class SplitMix64:
    """rng.hpp:55-75."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        return 0 if n == 0 else self.next() % n

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.below(i)
            v[i - 1], v[j] = v[j], v[i - 1]


# ------------------------------------------------------------ builders.cpp

def diamond4() -> Graph:
    """builders.cpp:80-87 — the D4 fixture of SPEC.md:150."""
    nodes = [make_node(i, 10, 2, 1, 1) for i in range(1, 5)]
    return Graph(nodes, [Edge(1, 2), Edge(1, 3), Edge(2, 4), Edge(3, 4)])


def mirror_training(g: Graph) -> Graph:
    """builders.cpp:89-104: backward twin per node, mirrored edges, paired."""
    offset = g.max_id()
    nodes = [Node(**vars(n)) for n in g.nodes()]
    for n in g.nodes():
        b = Node(**vars(n))
        b.id = n.id + offset
        b.is_backward = True
        b.forward_pair = n.id
        nodes.append(b)
    edges = list(g.edges()) + [Edge(e.dst + offset, e.src + offset) for e in g.edges()]
    return Graph(nodes, edges, g.artificial_edges())


def path_graph(n: int, cpu, acc, comm, mem) -> Graph:
    """builders.cpp:106-114."""
    nodes = [make_node(i, cpu, acc, comm, mem) for i in range(1, n + 1)]
    edges = [Edge(i - 1, i) for i in range(2, n + 1)]
    return Graph(nodes, edges)


def edgeless(n: int) -> Graph:
    """builders.cpp:116-120."""
    return Graph([make_node(i, 1, 1, 0, 1) for i in range(1, n + 1)], [])


@dataclass
class RandomInstance:
    graph: Graph
    config: DeviceConfig


def random_instance(seed: int, allow_unsupported: bool = True) -> RandomInstance:
    """builders.cpp:122-158.

    `make_node(i, half(), half(), half(), Rat(1 + below(6)))` evaluates its
    arguments in g++'s order for this call (right to left), so the draws go
    mem, comm, acc, cpu; tests/golden/random_instances.json (dumped from the
    compiled reference builders) pins this."""
    rng = SplitMix64((seed * 0x100000001B3 + 0x9E3779B97F4A7C15) & MASK64)
    n = 2 + rng.below(9)

    def half(lo, hi):
        return Fraction(lo + rng.below(hi - lo + 1), 2)

    nodes = []
    total_mem = Fraction(0)
    for i in range(1, n + 1):
        mem = Fraction(1 + rng.below(6))
        comm = half(0, 20)
        acc = half(0, 20)
        cpu = half(0, 20)
        node = make_node(i, cpu, acc, comm, mem)
        if allow_unsupported and rng.below(10) == 0:
            node.acc_time = INF
        total_mem += node.mem_size
        nodes.append(node)
    edges = []
    seen = set()
    want = rng.below(21)
    t = 0
    while t < want * 3 and len(edges) < want:
        a = 1 + rng.below(n)
        b = 1 + rng.below(n)
        t += 1
        if a == b:
            continue
        if a > b:
            a, b = b, a
        if (a, b) not in seen:
            seen.add((a, b))
            edges.append(Edge(a, b))
    cfg = DeviceConfig()
    cfg.accelerators = 1 + rng.below(3)
    cfg.cpus = rng.below(3)
    scale = Fraction(4 + rng.below(11), 10)
    cfg.memory_limit = scale * total_mem
    return RandomInstance(Graph(nodes, edges), cfg)


def make_corpus(count: int) -> List[RandomInstance]:
    """acceptance.cpp:40-47."""
    return [random_instance(seed) for seed in range(count)]


# ---------------------------------------------------------- module chains

@dataclass
class ChainSpec:
    stem: int
    modules: List[Sequence[int]]  # branch chain lengths per module
    tail: int = 0


def module_chain(spec: ChainSpec, seed: int = 1, decimals: int = 1) -> Graph:
    """SURVEY §8(d) generator: stem chain -> modules (split -> branch chains ->
    join; the join is the next split) -> tail chain.  Ids from 1 in creation
    order; each node draws cpu, acc, comm, mem from one SplitMix64(seed)."""
    rng = SplitMix64(seed)
    scale = 10 ** decimals
    nodes: List[Node] = []
    edges: List[Edge] = []

    def new_node() -> int:
        i = len(nodes) + 1
        if decimals == 1:
            cpu = Fraction(10 + rng.below(90), 10)
            acc = Fraction(1 + rng.below(20), 10)
            comm = Fraction(rng.below(10), 10)
        else:  # D = 10**decimals variant with finer weights
            cpu = Fraction(scale + rng.below(9 * scale), scale)
            acc = Fraction(1 + rng.below(2 * scale), scale)
            comm = Fraction(rng.below(scale), scale)
        mem = Fraction(1 + rng.below(4))
        nodes.append(make_node(i, cpu, acc, comm, mem))
        return i

    prev = None
    for _ in range(spec.stem):
        v = new_node()
        if prev is not None:
            edges.append(Edge(prev, v))
        prev = v
    split = new_node()
    if prev is not None:
        edges.append(Edge(prev, split))
    for branches in spec.modules:
        ends = []
        for c in branches:
            last = split
            for _ in range(c):
                v = new_node()
                edges.append(Edge(last, v))
                last = v
            ends.append(last)
        join = new_node()
        for last in ends:
            edges.append(Edge(last, join))
        split = join
    prev = split
    for _ in range(spec.tail):
        v = new_node()
        edges.append(Edge(prev, v))
        prev = v
    return Graph(nodes, edges)


def chain_counts(spec: ChainSpec) -> Tuple[int, int, int]:
    """Closed forms: (|V|, #ideals, #nested pairs I' < I)."""
    nv = spec.stem + 1 + sum(sum(b) + 1 for b in spec.modules) + spec.tail
    blocks = [1] + [1] * spec.stem
    within = 0
    for b in spec.modules:
        pi = 1
        tri = 1
        for c in b:
            pi *= c + 1
            tri *= (c + 1) * (c + 2) // 2
        blocks.append(pi)
        within += tri - pi
    blocks += [1] + [1] * spec.tail
    ideals = sum(blocks)
    pairs = within
    acc = 0
    for size in blocks:
        pairs += acc * size
        acc += size
    return nv, ideals, pairs


def _mem_limit(g: Graph, k: int) -> Fraction:
    total = sum((n.mem_size for n in g.nodes()), Fraction(0))
    return Fraction(3, 2) * total / k + 1


@dataclass
class Workload:
    name: str
    graph: Graph
    config: DeviceConfig
    training: bool
    spec: ChainSpec
    description: str
    flags: int = 0  # extra dsg_options flags (the @int64 tag: DSG_FLAG_FORCE_INT64)

    @property
    def counts(self):
        return chain_counts(self.spec)


SPECS = {
    # C1: ResNet-50 layer graph, 177 nodes / 242 ideals
    "C1": ChainSpec(12, [[8, 2] if i in (1, 4, 8, 14) else [8, 0] for i in range(1, 17)], 12),
    # C2: InceptionV3 layer graph, 326 nodes / 36,596 ideals
    "C2": ChainSpec(12, [[3, 6, 9, 2]] * 3 + [[3, 9, 1]] + [[3, 9, 15, 4]] * 4
                    + [[6, 12, 1]] + [[4, 6, 14, 19]] * 2, 0),
    # C3: GNMT layer graph, 96 nodes / 17,914 ideals
    "C3": ChainSpec(0, [[12, 31, 42], [3, 5]], 0),
    # C4: BERT-24 operator graph stand-in, 1,516 nodes / 4,013 ideals
    "C4": ChainSpec(51, [[1, 1, 1], [10, 10], [35]] * 24, 0),
}

CONFIGS = {
    "C1": dict(k=4, l=1, training=True,
               desc="ResNet-50-like layer graph (177 fw / 354 nodes), pipelined-training DP, 4 acc + 1 CPU"),
    "C2": dict(k=8, l=0, training=False,
               desc="InceptionV3-like layer graph (326 nodes, 36,596 ideals), inference DP, 8 acc"),
    "C3": dict(k=6, l=2, training=True,
               desc="GNMT-like layer graph (96 fw / 192 nodes), training DP, 6 acc + 2 CPUs, memory-bound"),
    "C4": dict(k=8, l=4, training=False,
               desc="BERT-24-operator-like graph (1,516 nodes), inference DP, 8 acc + 4 CPUs"),
}


def sweep_spec(width: int, chain: int, modules: int, stem: int) -> ChainSpec:
    """C5 sweep point (w, c, M, stem): M modules of w branches of length c."""
    return ChainSpec(stem, [[chain] * width] * modules, 0)


SWEEP_POINTS = [
    (2, 8, 20, 100), (2, 24, 8, 200), (4, 4, 20, 300), (4, 6, 10, 400), (8, 2, 6, 600),
    (12, 1, 8, 1000), (16, 1, 1, 300), (4, 3, 40, 1400), (6, 2, 30, 1500), (8, 2, 7, 600),
]


def standin(name: str, seed: int = 1, decimals: int = 1) -> Workload:
    """The BASELINE.json config stand-ins C1..C4.  seed /
    decimals select the weight draw (decimals=3: D = 1000 weights)."""
    spec = SPECS[name]
    c = CONFIGS[name]
    g = module_chain(spec, seed=seed, decimals=decimals)
    if c["training"]:
        g = mirror_training(g)
    cfg = DeviceConfig(accelerators=c["k"], cpus=c["l"], memory_limit=_mem_limit(g, c["k"]))
    tag = name + (f"@seed{seed}" if seed != 1 else "") + (f"@D{10 ** decimals}" if decimals != 1 else "")
    return Workload(tag, g, cfg, c["training"], spec, c["desc"])


def by_name(name: str) -> Workload:
    """Workload names used by bench.py and the tools: C1..C4, optionally
    suffixed @seedN / @D1000 (weight draw) / @int64 (64-bit values forced),
    or C5:w,c,M,stem (sweep point)."""
    if name.startswith("C5"):
        pt = tuple(int(x) for x in name[3:].split(","))
        return sweep(*pt)
    base, *tags = name.split("@")
    seed, decimals, flags = 1, 1, 0
    for t in tags:
        if t == "int64":
            from . import _abi
            flags |= _abi.DSG_FLAG_FORCE_INT64
        elif t.startswith("seed"):
            seed = int(t[4:])
        elif t.startswith("D"):
            d = int(t[1:])
            decimals = len(str(d)) - 1
            if 10 ** decimals != d:
                raise ValueError(f"weight denominator must be a power of 10: {name}")
        else:
            raise ValueError(f"unknown workload tag {t!r} in {name!r}")
    w = standin(base, seed=seed, decimals=decimals)
    if flags:
        w = dataclasses.replace(w, name=name, flags=flags)
    return w


def sweep(width: int, chain: int, modules: int, stem: int, k: int = 8, l: int = 0,
          seed: int = 1) -> Workload:
    spec = sweep_spec(width, chain, modules, stem)
    g = module_chain(spec, seed=seed)
    cfg = DeviceConfig(accelerators=k, cpus=l, memory_limit=_mem_limit(g, k))
    return Workload(f"C5(w={width},c={chain},M={modules},stem={stem})", g, cfg, False, spec,
                    f"synthetic layered sweep point w={width} c={chain} M={modules} stem={stem}")
