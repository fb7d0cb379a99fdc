"""The reference's solver API (include/dagsplit/dp_solver.hpp:21-37,
graph.hpp:253-258) backed by the sm_100a kernels in libdsg_b200.so.

There is no CPU fallback: if the CUDA library is missing or no B200 is
visible, every call raises DeviceError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Iterable, List, Optional

import numpy as np

from . import _abi
from .errors import DeviceError, raise_for_status
from fractions import Fraction

from .graph import INF, DeviceConfig, Graph, SplitBlock, make_canonical_split

_I64_MAX = (1 << 63) - 1

_HERE = os.path.dirname(os.path.abspath(__file__))
# DSG_B200_LIB: an alternative build of the same library (kernel variants
# under test); the default is the in-tree build.
LIB_PATH = os.environ.get("DSG_B200_LIB") or os.path.join(_HERE, "libdsg_b200.so")
_lib: Optional[C.CDLL] = None


def load_library() -> C.CDLL:
    """Load the in-tree CUDA library (fails loudly when it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    _abi.bind(lib, "dsg")
    lib.dsg_device_count.restype = C.c_int
    lib.dsg_version.restype = C.c_char_p
    lib.dsg_kernel_launch_count.restype = C.c_int64
    lib.dsg_default_options.argtypes = [C.POINTER(_abi.dsg_options)]
    lib.dsg_session_create.restype = C.c_void_p
    lib.dsg_session_create.argtypes = [C.c_int32, C.POINTER(_abi.dsg_graph),
                                       C.POINTER(_abi.dsg_config), C.POINTER(_abi.dsg_options),
                                       C.POINTER(_abi.dsg_result)]
    lib.dsg_session_run.argtypes = [C.c_void_p, C.POINTER(_abi.dsg_result)]
    lib.dsg_session_run.restype = C.c_int
    lib.dsg_session_destroy.argtypes = [C.c_void_p]
    lib.dsg_session_destroy.restype = None
    lib.dsg_session_shard_prepare.argtypes = [C.c_void_p, C.c_int32, C.c_int32,
                                              C.POINTER(_abi.dsg_shard_handle),
                                              C.POINTER(_abi.dsg_result)]
    lib.dsg_session_shard_attach.argtypes = [C.c_void_p, C.POINTER(_abi.dsg_shard_handle),
                                             C.POINTER(_abi.dsg_result)]
    lib.dsg_session_shard_reset.argtypes = [C.c_void_p, C.POINTER(_abi.dsg_result)]
    lib.dsg_session_reload.argtypes = [C.c_void_p, C.POINTER(_abi.dsg_graph),
                                       C.POINTER(_abi.dsg_config), C.POINTER(_abi.dsg_result)]
    _lib = lib
    return lib


def kernel_launch_count() -> int:
    return int(load_library().dsg_kernel_launch_count())


@dataclass
class SolveOptions:
    """dp_solver.hpp:11-14 plus device knobs."""
    deadline_seconds: Optional[float] = None
    ideal_budget: int = _abi.DSG_DEFAULT_IDEAL_BUDGET
    device: int = -1
    flags: int = 0
    shard_count: int = 0
    max_blocks: int = 0  # > 0 caps the persistent kernel's grid (testing)


@dataclass
class RawResult:
    objective: object
    blocks: List[SplitBlock]
    best_k: int
    best_l: int
    n_ideals: int
    n_pairs: int
    n_levels: int
    value_bits: int
    denominator: int
    stats: dict = field(default_factory=dict)
    ideal_bits: Optional[np.ndarray] = None
    dp_values: Optional[np.ndarray] = None


STAT_FIELDS = ("t_prepare_ms", "t_enumerate_ms", "t_describe_ms", "t_dp_ms", "t_traceback_ms",
               "t_total_ms", "t_transition_kernel_ms", "t_device_ms", "kernel_launches",
               "h2d_bytes", "d2h_bytes")


def _raw_from(res, config: DeviceConfig) -> RawResult:
    blocks = []
    n_mem = 0
    for b in range(res.n_blocks):
        n_mem = max(n_mem, res.blocks[b].offset + res.blocks[b].n_members)
    # one view of the member array (per-element ctypes indexing costs ~0.1 us each)
    mem = np.ctypeslib.as_array(res.members, shape=(n_mem,)).tolist() if n_mem else []
    for b in range(res.n_blocks):
        blk = res.blocks[b]
        members = mem[blk.offset:blk.offset + blk.n_members]
        load = None
        if res.block_loads:
            load = INF if blk.load_num == _I64_MAX else Fraction(blk.load_num, res.denominator)
        blocks.append(SplitBlock(cpu=bool(blk.cpu), members=members, repl=blk.repl, load=load))
    stats = {k: getattr(res, k) for k in STAT_FIELDS}
    return RawResult(_abi.from_dsg_rat(res.objective), blocks, res.best_k, res.best_l,
                     res.n_ideals, res.n_pairs, res.n_levels, res.value_bits, res.denominator,
                     stats)


class Session:
    """A solve whose flattened graph stays resident in HBM (dsg_session_*):
    ``run()`` repeats the whole device pipeline without re-uploading inputs."""

    def __init__(self, mode: int, g: Graph, config: DeviceConfig,
                 opt: Optional[SolveOptions] = None):
        lib = load_library()
        opt = opt or SolveOptions()
        self._lib = lib
        self.config = config
        self._pg = _abi.pod_graph(g)
        self._cfg = _abi.pod_config(config)
        self._po = _abi.pod_options(opt.ideal_budget, opt.deadline_seconds, opt.device,
                                    opt.shard_count, opt.flags, opt.max_blocks)
        st = _abi.dsg_result()
        self._h = lib.dsg_session_create(mode, C.byref(self._pg.struct), C.byref(self._cfg),
                                         C.byref(self._po), C.byref(st))
        raise_for_status(st.status, st.message, st.budget_limit)
        self.prepare_ms = st.t_prepare_ms

    def reload(self, g: Graph, config: DeviceConfig) -> dict:
        """Re-flatten + re-upload a same-shaped graph (the H2D leg of e2e)."""
        self._pg = _abi.PodGraph(g)
        self._cfg = _abi.pod_config(config)
        self.config = config
        st = _abi.dsg_result()
        self._lib.dsg_session_reload(self._h, C.byref(self._pg.struct), C.byref(self._cfg),
                                     C.byref(st))
        raise_for_status(st.status, st.message, st.budget_limit)
        return {"h2d_bytes": st.h2d_bytes, "t_prepare_ms": st.t_prepare_ms}

    def run(self) -> RawResult:
        res = _abi.dsg_result()
        self._lib.dsg_session_run(self._h, C.byref(res))
        try:
            raise_for_status(res.status, res.message, res.budget_limit)
            return _raw_from(res, self.config)
        finally:
            self._lib.dsg_result_free(C.byref(res))

    def close(self) -> None:
        if self._h:
            self._lib.dsg_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardComm:
    """What a sharded session needs from the process group: an all-gather of
    small byte strings and a barrier.  `from_torch()` uses torch.distributed
    (NCCL or gloo); tests can pass any object with the same two methods."""

    def __init__(self, rank: int, world: int, all_gather_bytes, barrier):
        self.rank, self.world = rank, world
        self.all_gather_bytes = all_gather_bytes
        self.barrier = barrier

    @staticmethod
    def from_torch(group=None) -> "ShardComm":
        import torch.distributed as dist

        def gather(b: bytes):
            out = [None] * dist.get_world_size(group)
            dist.all_gather_object(out, b, group=group)
            return out

        return ShardComm(dist.get_rank(group), dist.get_world_size(group), gather,
                         lambda: dist.barrier(group=group))


class ShardedSession(Session):
    """One rank of the multi-GPU wavefront (dsg_session_shard_*, SURVEY
    §8(e)): target units of every level are split across ranks; finished dp
    rows travel GPU->GPU over NVLink inside the persistent kernel."""

    def __init__(self, mode: int, g: Graph, config: DeviceConfig, comm: ShardComm,
                 opt: Optional[SolveOptions] = None):
        super().__init__(mode, g, config, opt)
        self.comm = comm
        mine = _abi.dsg_shard_handle()
        st = _abi.dsg_result()
        self._lib.dsg_session_shard_prepare(self._h, comm.rank, comm.world, C.byref(mine),
                                            C.byref(st))
        raise_for_status(st.status, st.message, st.budget_limit)
        blobs = comm.all_gather_bytes(bytes(mine))
        handles = (_abi.dsg_shard_handle * comm.world)()
        for r, b in enumerate(blobs):
            C.memmove(C.byref(handles[r]), b, C.sizeof(_abi.dsg_shard_handle))
        self._lib.dsg_session_shard_attach(self._h, handles, C.byref(st))
        raise_for_status(st.status, st.message, st.budget_limit)
        comm.barrier()

    def run(self) -> RawResult:
        st = _abi.dsg_result()
        self._lib.dsg_session_shard_reset(self._h, C.byref(st))
        raise_for_status(st.status, st.message, st.budget_limit)
        self.comm.barrier()  # every rank reset before any rank writes into it
        res = _abi.dsg_result()
        self._lib.dsg_session_run(self._h, C.byref(res))
        try:
            self.comm.barrier()  # every peer finished writing into this rank
            raise_for_status(res.status, res.message, res.budget_limit)
            raw = _raw_from(res, self.config)
            # phase 1 (lattice + descriptors) ran inside the reset call
            raw.stats["t_reset_device_ms"] = st.t_device_ms
            raw.stats["t_enumerate_ms"] = st.t_enumerate_ms
            raw.stats["t_describe_ms"] = st.t_describe_ms
            raw.stats["t_device_ms"] = st.t_device_ms + res.t_device_ms
            return raw
        finally:
            self._lib.dsg_result_free(C.byref(res))


def run_dp(lib: C.CDLL, prefix: str, mode: int, g: Graph, config: DeviceConfig,
           opt: Optional[SolveOptions] = None) -> RawResult:
    """Call <prefix>_dp_solve on the POD form of (g, config); raise on error.

    Shared by the product path (prefix "dsg") and, in tests only, the oracle
    libraries (prefixes "dsgo", "dsgref")."""
    opt = opt or SolveOptions()
    pg = _abi.pod_graph(g)
    cfg = _abi.pod_config(config)
    po = _abi.pod_options(opt.ideal_budget, opt.deadline_seconds, opt.device, opt.shard_count,
                          opt.flags, opt.max_blocks)
    res = _abi.dsg_result()
    getattr(lib, f"{prefix}_dp_solve")(mode, C.byref(pg.struct), C.byref(cfg), C.byref(po),
                                       C.byref(res))
    try:
        raise_for_status(res.status, res.message, res.budget_limit)
        out = _raw_from(res, config)
        if res.ideal_bits:
            n = res.n_ideals * res.words
            out.ideal_bits = np.ctypeslib.as_array(res.ideal_bits, shape=(n,)).copy().reshape(
                res.n_ideals, res.words)
        if res.dp_values:
            cells = (config.accelerators + 1) * (config.cpus + 1)
            out.dp_values = np.ctypeslib.as_array(res.dp_values, shape=(res.n_ideals * cells,)).copy(
            ).reshape(res.n_ideals, cells)
        return out
    finally:
        getattr(lib, f"{prefix}_result_free")(C.byref(res))


def _solve(mode: int, g: Graph, config: DeviceConfig, opt: Optional[SolveOptions]):
    raw = run_dp(load_library(), "dsg", mode, g, config, opt)
    split = make_canonical_split(g, config, raw.blocks, raw.objective)
    split.stats = dict(raw.stats, n_ideals=raw.n_ideals, n_pairs=raw.n_pairs,
                       n_levels=raw.n_levels, value_bits=raw.value_bits,
                       best_k=raw.best_k, best_l=raw.best_l)
    return split


def solve_maxload_inference(g: Graph, config: DeviceConfig, opt: Optional[SolveOptions] = None):
    """dp_solver.hpp:21-22 on the B200."""
    return _solve(_abi.DSG_MODE_INFERENCE, g, config, opt)


def solve_maxload_training(g: Graph, config: DeviceConfig, opt: Optional[SolveOptions] = None):
    """dp_solver.hpp:28-29 on the B200."""
    return _solve(_abi.DSG_MODE_TRAINING, g, config, opt)


def solve_maxload_replicated(g: Graph, config: DeviceConfig, opt: Optional[SolveOptions] = None):
    """dp_solver.hpp:36-37 on the B200."""
    return _solve(_abi.DSG_MODE_REPLICATED, g, config, opt)


def seeded_topo_order(g: Graph, seed: int) -> List[int]:
    """dp_solver.hpp:39-41 (dp_solver.cpp:407-438): DFS topological order,
    roots and every out_all list shuffled by one SplitMix64 stream keyed on
    `seed`, reversed post-order.  Host-side ordering, not on the hot path."""
    from .workloads import MASK64, SplitMix64
    rng = SplitMix64((seed * 0x9E3779B97F4A7C15 + 0x2545F4914F6CDD1D) & MASK64)
    n = g.size()
    roots = list(range(n))
    rng.shuffle(roots)
    succ = []
    for v in range(n):
        lst = list(g.out_all(v))
        rng.shuffle(lst)
        succ.append(lst)
    seen = [False] * n
    post: List[int] = []
    for r in roots:
        if seen[r]:
            continue
        seen[r] = True
        stack = [[r, 0]]
        while stack:
            top = stack[-1]
            if top[1] < len(succ[top[0]]):
                w = succ[top[0]][top[1]]
                top[1] += 1
                if not seen[w]:
                    seen[w] = True
                    stack.append([w, 0])
            else:
                post.append(top[0])
                stack.pop()
    post.reverse()
    return post


def _chain_along(g: Graph, order: List[int]) -> Graph:
    """Artificial precedence edges between consecutive nodes of `order`
    (dp_solver.cpp:443-454); existing real/artificial pairs are not repeated."""
    from .graph import Edge
    have = {(e.src, e.dst) for e in g.edges()} | {(e.src, e.dst) for e in g.artificial_edges()}
    art = list(g.artificial_edges())
    for a, b in zip(order, order[1:]):
        pair = (g.id_of(a), g.id_of(b))
        if pair not in have:
            have.add(pair)
            art.append(Edge(*pair))
    return Graph(g.nodes(), g.edges(), art)


def linearize(g: Graph, seed: int) -> Graph:
    """dp_solver.hpp:43-46: the |V|+1-prefix chain along seeded_topo_order."""
    return _chain_along(g, seeded_topo_order(g, seed))


def solve_dpl(g: Graph, config: DeviceConfig, seed: int, opt: Optional[SolveOptions] = None):
    """dp_solver.hpp:48-52 (dp_solver.cpp:462-477): linearize (forward part
    only for training graphs), then the exact device DP on the chained graph."""
    training = g.has_backward_nodes()
    order = seeded_topo_order(g, seed)
    if training:
        order = [v for v in order if not g.node(v).is_backward]
    chained = _chain_along(g, order)
    return (solve_maxload_training if training else solve_maxload_inference)(chained, config, opt)


@dataclass
class IdealIndex:
    """graph.hpp:243-249: ideals in size-major, lexicographic order."""
    bits: np.ndarray          # [count, words] uint64
    level_offsets: np.ndarray
    universe: int

    def count(self) -> int:
        return int(self.bits.shape[0])

    def ideal(self, ordinal: int) -> frozenset:
        row = self.bits[ordinal]
        return frozenset(w * 64 + b for w in range(row.shape[0]) for b in range(64)
                         if (int(row[w]) >> b) & 1)

    @property
    def ideals(self) -> List[frozenset]:
        return [self.ideal(i) for i in range(self.count())]


def run_enumerate(lib: C.CDLL, prefix: str, g: Graph, within: Optional[Iterable[int]],
                  budget: int, flags: int = 0, device: int = -1) -> IdealIndex:
    pg = _abi.pod_graph(g)
    w_arr = None
    w_ptr = None
    if within is not None:
        w_arr = np.zeros(max(g.size(), 1), dtype=np.uint8)
        for v in within:
            w_arr[v] = 1
        w_ptr = w_arr.ctypes.data_as(C.POINTER(C.c_uint8))
    po = _abi.pod_options(budget, None, device, 0, flags)
    out = _abi.dsg_ideals()
    getattr(lib, f"{prefix}_enumerate_ideals")(C.byref(pg.struct), w_ptr, int(budget), C.byref(po),
                                               C.byref(out))
    try:
        raise_for_status(out.status, out.message, out.budget_limit)
        words = out.words
        bits = np.ctypeslib.as_array(out.bits, shape=(out.count * words,)).copy().reshape(
            out.count, words) if out.count else np.zeros((0, words), np.uint64)
        offs = np.ctypeslib.as_array(out.level_offsets, shape=(out.n_levels + 1,)).copy()
        return IdealIndex(bits, offs, g.size())
    finally:
        getattr(lib, f"{prefix}_ideals_free")(C.byref(out))


def enumerate_ideals(g: Graph, budget: int = _abi.DSG_DEFAULT_IDEAL_BUDGET, flags: int = 0):
    """graph.hpp:253 on the B200."""
    return run_enumerate(load_library(), "dsg", g, None, budget, flags)


def enumerate_ideals_within(g: Graph, within: Iterable[int],
                            budget: int = _abi.DSG_DEFAULT_IDEAL_BUDGET, flags: int = 0):
    """graph.hpp:256-258 on the B200."""
    return run_enumerate(load_library(), "dsg", g, within, budget, flags)
