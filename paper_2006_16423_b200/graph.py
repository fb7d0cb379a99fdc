"""Host-side mirror of the reference data model and its exact cost functions.

Mirrors /root/reference/proj/include/dagsplit/graph.hpp so callers (and the
parity tests) read like the reference's own code:

  Node / Edge / Graph            graph.hpp:19-39, 152-186; graph.cpp:132-158
  DeviceConfig / Placement       graph.hpp:98-132
  Split                          graph.hpp:134-141
  acc_cost_parts / acc_cost /    graph.cpp:397-479
  cpu_cost / combine_interleaving
  make_canonical_split           graph.cpp:573-621
  recompute_maxload              graph.cpp:623-659
  reachability / is_contiguous   graph.cpp:291-367

Weights are exact: ``fractions.Fraction`` for finite values and ``INF``
(float +inf) for the reference's ``Rat::infinity()``.  Nothing here is on the
device hot path: the DP runs in libdsg_b200.so (CUDA); this module only
builds the POD input and turns the device's blocks into a ``Split``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum
from fractions import Fraction
from typing import Dict, Iterable, List, Optional, Sequence, Tuple, Union

INF = math.inf
Num = Union[Fraction, float]


def rat(x) -> Num:
    """Exact rational from int / Fraction / str / INF (the reference Rat)."""
    if isinstance(x, float):
        if x == INF:
            return INF
        raise TypeError("use Fraction or str for finite non-integer weights "
                        f"(got float {x!r}); JSON ingest snaps via Rat.from_double")
    if isinstance(x, Fraction):
        return x
    return Fraction(x)


def is_inf(x: Num) -> bool:
    return isinstance(x, float) and x == INF


class Interleaving(IntEnum):
    Sum = 0
    HalfDuplexMax = 1
    FullDuplexMax = 2


class ReplicationCombine(IntEnum):
    Sum = 0
    Max = 1


@dataclass
class Node:
    id: int
    cpu_time: Num = Fraction(0)
    acc_time: Num = Fraction(0)
    comm_time: Num = Fraction(0)
    mem_size: Num = Fraction(0)
    name: str = ""
    color_class: Optional[int] = None
    is_backward: bool = False
    forward_pair: Optional[int] = None
    colocate_with: Optional[int] = None
    artificial: bool = False

    def __post_init__(self):
        self.cpu_time = rat(self.cpu_time)
        self.acc_time = rat(self.acc_time)
        self.comm_time = rat(self.comm_time)
        self.mem_size = rat(self.mem_size)

    def acc_supported(self) -> bool:
        return not is_inf(self.acc_time)


@dataclass
class Edge:
    src: int
    dst: int
    comm_override: Optional[Num] = None


def make_node(id: int, cpu, acc, comm, mem) -> Node:
    return Node(id=id, cpu_time=cpu, acc_time=acc, comm_time=comm, mem_size=mem)


class Graph:
    """Dense-index DAG with real (comm-carrying) and artificial edges."""

    def __init__(self, nodes: Sequence[Node], edges: Sequence[Edge] = (),
                 artificial_edges: Sequence[Edge] = ()):
        self._nodes: List[Node] = list(nodes)
        self._edges: List[Edge] = [e if isinstance(e, Edge) else Edge(*e) for e in edges]
        self._art: List[Edge] = [e if isinstance(e, Edge) else Edge(*e) for e in artificial_edges]
        self._index: Dict[int, int] = {}
        for i, n in enumerate(self._nodes):
            self._index.setdefault(n.id, i)  # first occurrence wins (graph.cpp:139)
        n = len(self._nodes)
        self._out = [[] for _ in range(n)]
        self._in = [[] for _ in range(n)]
        self._out_all = [[] for _ in range(n)]
        self._in_all = [[] for _ in range(n)]
        for real, lst in ((True, self._edges), (False, self._art)):
            for e in lst:
                f = self._index.get(e.src)
                t = self._index.get(e.dst)
                if f is None or t is None:
                    continue
                if real:
                    self._out[f].append(t)
                    self._in[t].append(f)
                self._out_all[f].append(t)
                self._in_all[t].append(f)
        self._pod_cache = None
        self._ids: List[int] = [nd.id for nd in self._nodes]

    def ids(self) -> List[int]:
        """External id of every dense index (the Graph is immutable)."""
        return self._ids

    # --- reference accessors (graph.hpp:157-185) ---
    def size(self) -> int:
        return len(self._nodes)

    def nodes(self) -> List[Node]:
        return self._nodes

    def node(self, idx: int) -> Node:
        return self._nodes[idx]

    def edges(self) -> List[Edge]:
        return self._edges

    def artificial_edges(self) -> List[Edge]:
        return self._art

    def index_of(self, id: int) -> Optional[int]:
        return self._index.get(id)

    def id_of(self, idx: int) -> int:
        return self._nodes[idx].id

    def out(self, idx):
        return self._out[idx]

    def in_(self, idx):
        return self._in[idx]

    def out_all(self, idx):
        return self._out_all[idx]

    def in_all(self, idx):
        return self._in_all[idx]

    def has_backward_nodes(self) -> bool:
        return any(n.is_backward for n in self._nodes)

    def forward_set(self) -> frozenset:
        return frozenset(i for i, n in enumerate(self._nodes) if not n.is_backward)

    def backward_set(self) -> frozenset:
        return frozenset(i for i, n in enumerate(self._nodes) if n.is_backward)

    def max_id(self) -> int:
        return max((n.id for n in self._nodes), default=-1)


@dataclass
class DeviceConfig:
    accelerators: int = 0
    cpus: int = 0
    memory_limit: Num = INF
    q: int = 1
    interleaving: Interleaving = Interleaving.Sum
    bandwidth: Optional[Num] = None
    replication_combine: ReplicationCombine = ReplicationCombine.Sum

    def __post_init__(self):
        self.memory_limit = rat(self.memory_limit)
        if self.bandwidth is not None:
            self.bandwidth = rat(self.bandwidth)


@dataclass(frozen=True)
class Placement:
    """graph.hpp:108-132."""
    is_cpu_: bool
    index: int
    slot: int = 1

    @staticmethod
    def cpu(index: int = 0) -> "Placement":
        return Placement(True, index, 1)

    @staticmethod
    def acc(index: int, slot: int = 1) -> "Placement":
        return Placement(False, index, slot)

    def is_cpu(self) -> bool:
        return self.is_cpu_

    def label(self) -> str:
        if self.is_cpu_:
            return "cpu" if self.index == 0 else f"cpu{self.index}"
        s = f"acc{self.index}"
        if self.slot > 1:
            s += f".{self.slot}"
        return s


@dataclass
class Split:
    assignment: Dict[int, Placement] = field(default_factory=dict)
    objective_value: Num = Fraction(0)
    per_device_loads: List[Tuple[str, Num]] = field(default_factory=list)
    replication: Dict[str, int] = field(default_factory=dict)
    # not in the reference Split: how the solve went (for benches / tests)
    stats: Dict[str, float] = field(default_factory=dict)

    def placement_of(self, node_id: int) -> Optional[Placement]:
        return self.assignment.get(node_id)


@dataclass
class SplitBlock:
    cpu: bool
    members: List[int]
    repl: int = 1
    load: Optional[Num] = None  # per-device load recomputed by the device, if reported


# ---------------------------------------------------------------- costs

@dataclass
class AccParts:
    comm_in: Num = Fraction(0)
    proc: Num = Fraction(0)
    comm_out: Num = Fraction(0)
    mem: Num = Fraction(0)
    unsupported: bool = False


def _fsum(vals: Iterable[Num]) -> Num:
    """Exact sum of rationals (INF absorbing): numerators summed per
    denominator with Python ints, one Fraction per distinct denominator —
    the same value as a Rat accumulation in any order, without a gcd per
    addition."""
    acc: Dict[int, int] = {}
    for x in vals:
        if isinstance(x, float):
            if x == INF:
                return INF
            x = Fraction(x)
        d = x.denominator
        acc[d] = acc.get(d, 0) + x.numerator
    total = Fraction(0)
    for d, n in acc.items():
        total += Fraction(n, d)
    return total


def acc_cost_parts(g: Graph, s: Iterable[int]) -> AccParts:
    """graph.cpp:397-428: comm_in charges each outside producer once."""
    s = set(s)
    p = AccParts()
    nodes = [g.node(v) for v in s]
    p.unsupported = any(not n.acc_supported() for n in nodes)
    p.proc = _fsum(n.acc_time for n in nodes if n.acc_supported())
    p.mem = _fsum(n.mem_size for n in nodes)
    p.comm_out = _fsum(g.node(v).comm_time for v in s if any(w not in s for w in g.out(v)))
    producers = {u for v in s for u in g.in_(v) if u not in s}
    p.comm_in = _fsum(g.node(u).comm_time for u in producers)
    return p


def combine_interleaving(p: AccParts, mode: Interleaving) -> Num:
    """graph.cpp:457-467."""
    if mode == Interleaving.Sum:
        return p.comm_in + p.proc + p.comm_out
    if mode == Interleaving.HalfDuplexMax:
        return max(p.proc, p.comm_in + p.comm_out)
    return max(p.proc, p.comm_in, p.comm_out)


def acc_cost(g: Graph, s: Iterable[int], config: DeviceConfig) -> Num:
    """graph.cpp:469-473 (strict memory test, unsupported -> inf)."""
    p = acc_cost_parts(g, s)
    if p.unsupported or p.mem > config.memory_limit:
        return INF
    return combine_interleaving(p, config.interleaving)


def cpu_cost(g: Graph, s: Iterable[int]) -> Num:
    return _fsum(g.node(v).cpu_time for v in s)


def _replicated(load: Num, mem: Num, r: int, config: DeviceConfig) -> Num:
    if r <= 1 or is_inf(load):
        return load
    divided = load / r
    sync = (r - 1) * mem / (r * config.bandwidth) if config.bandwidth is not None else Fraction(0)
    if config.replication_combine == ReplicationCombine.Sum:
        return divided + sync
    return max(divided, sync)


def make_canonical_split(g: Graph, config: DeviceConfig, blocks: List[SplitBlock],
                         objective: Num) -> Split:
    """graph.cpp:573-621: accelerators first, each kind by smallest external id."""
    ids = g.ids()

    def smallest_id(b: SplitBlock) -> int:
        return min(map(ids.__getitem__, b.members), default=2 ** 31 - 1)

    blocks = sorted(blocks, key=lambda b: (b.cpu, smallest_id(b)))  # stable
    split = Split(objective_value=objective)
    next_acc, next_cpu = 1, 1
    for b in blocks:
        if not b.members:
            continue
        pl = Placement.cpu(next_cpu) if b.cpu else Placement.acc(next_acc)
        split.assignment.update(dict.fromkeys(map(ids.__getitem__, b.members), pl))
        if b.load is not None:
            load = b.load  # recomputed on the device (dsg_block::load_num)
        else:
            load = cpu_cost(g, b.members) if b.cpu else acc_cost(g, b.members, config)
            if not b.cpu and b.repl > 1:
                mem = _fsum(g.node(v).mem_size for v in b.members)
                load = _replicated(load, mem, b.repl, config)
        if not b.cpu and b.repl > 1:
            split.replication[pl.label()] = b.repl
            for r in range(b.repl):
                split.per_device_loads.append((Placement.acc(next_acc + r).label(), load))
            next_acc += b.repl
            continue
        split.per_device_loads.append((pl.label(), load))
        if b.cpu:
            next_cpu += 1
        else:
            next_acc += 1
    return split


def recompute_maxload(g: Graph, config: DeviceConfig, split: Split):
    """graph.cpp:623-659: per-device loads recomputed from scratch."""
    device_sets: Dict[str, set] = {}
    device_is_cpu: Dict[str, bool] = {}
    for nid, pl in split.assignment.items():
        idx = g.index_of(nid)
        if idx is None:
            continue
        dev = Placement(pl.is_cpu_, pl.index, 1)
        device_sets.setdefault(dev.label(), set()).add(idx)
        device_is_cpu[dev.label()] = pl.is_cpu()
    loads = []
    worst: Num = Fraction(0)
    for label in sorted(device_sets):
        s = device_sets[label]
        load = cpu_cost(g, s) if device_is_cpu[label] else acc_cost(g, s, config)
        r = split.replication.get(label, 1)
        if r > 1 and not is_inf(load):
            mem = sum((g.node(v).mem_size for v in s), Fraction(0))
            load = _replicated(load, mem, r, config)
        loads.append((label, load))
        worst = max(worst, load)
    return loads, worst


# ------------------------------------------------------ reachability

def reach_within(g: Graph, within: Optional[Iterable[int]] = None) -> List[set]:
    """Nodes reachable from each node over real+artificial edges inside `within`."""
    inside = set(range(g.size())) if within is None else set(within)
    reach: List[set] = [set() for _ in range(g.size())]
    for s in inside:
        seen = {s}
        stack = [s]
        while stack:
            v = stack.pop()
            for w in g.out_all(v):
                if w in inside and w not in seen:
                    seen.add(w)
                    stack.append(w)
        reach[s] = seen
    return reach


def is_contiguous(g: Graph, s: Iterable[int], within: Optional[Iterable[int]] = None,
                  reach: Optional[List[set]] = None) -> bool:
    """No node outside s is both reachable from s and reaching s (graph.cpp:349-363)."""
    s = set(s)
    inside = set(range(g.size())) if within is None else set(within)
    reach = reach if reach is not None else reach_within(g, inside)
    from_s = set().union(*(reach[u] for u in s)) if s else set()
    for v in from_s - s:
        if v in inside and reach[v] & s:
            return False
    return True


def is_ideal(g: Graph, s: Iterable[int]) -> bool:
    s = set(s)
    return all(u in s for v in s for u in g.in_all(v))


def verify_split(g: Graph, config: DeviceConfig, split: Split, training: bool) -> List[str]:
    """Feasible-with-equal-cost check from SURVEY §8(a) a15.

    Returns a list of violations (empty = verified): recomputed max-load equals
    the objective; accelerator memory within the limit; every device set is
    contiguous; training: forward/backward twins colocated and each device's
    forward and backward parts contiguous within their halves."""
    problems: List[str] = []
    loads, worst = recompute_maxload(g, config, split)
    if worst != split.objective_value:
        problems.append(f"recomputed max-load {worst} != objective {split.objective_value}")
    reported = max((l for _, l in split.per_device_loads), default=Fraction(0))
    if reported != split.objective_value:
        problems.append(f"reported max load {reported} != objective")
    if len(split.assignment) != g.size():
        problems.append("not every node is placed")
    by_dev: Dict[str, set] = {}
    for nid, pl in split.assignment.items():
        by_dev.setdefault(pl.label(), set()).add(g.index_of(nid))
    fw, bw = g.forward_set(), g.backward_set()
    reach_all = reach_within(g)
    reach_fw = reach_within(g, fw) if training else None
    reach_bw = reach_within(g, bw) if training else None
    for label, s in by_dev.items():
        if label.startswith("acc"):
            mem = sum((g.node(v).mem_size for v in s), Fraction(0))
            if mem > config.memory_limit:
                problems.append(f"{label}: memory {mem} > {config.memory_limit}")
        if training and bw:
            if not is_contiguous(g, s & fw, fw, reach_fw):
                problems.append(f"{label}: forward part not contiguous")
            if not is_contiguous(g, s & bw, bw, reach_bw):
                problems.append(f"{label}: backward part not contiguous")
        elif not is_contiguous(g, s, None, reach_all):
            problems.append(f"{label}: not contiguous")
    if training:
        for n in g.nodes():
            if n.is_backward and n.forward_pair is not None:
                if split.assignment.get(n.id) != split.assignment.get(n.forward_pair):
                    problems.append(f"node {n.id} not colocated with its forward pair")
    return problems
