"""ctypes mirror of include/dsg_b200.h and Graph -> POD flattening.

The same structs are used to call the product library (libdsg_b200.so, dsg_*)
and, from tests only, the oracle libraries (dsgo_*, dsgref_*).
"""
from __future__ import annotations

import ctypes as C
from fractions import Fraction
from typing import Optional

import numpy as np

from .graph import INF, DeviceConfig, Graph, is_inf

DSG_NO_PAIR = -(2 ** 31)
DSG_DEFAULT_IDEAL_BUDGET = 5_000_000

DSG_MODE_INFERENCE, DSG_MODE_TRAINING, DSG_MODE_REPLICATED = 0, 1, 2

DSG_FLAG_FORCE_INT64 = 1
DSG_FLAG_NO_FASTGATE = 2
DSG_FLAG_HASH_ENUM = 4
DSG_FLAG_KEEP_TABLES = 8
DSG_FLAG_TIME_KERNELS = 16
DSG_FLAG_LEVEL_LAUNCH = 32

(DSG_OK, DSG_INFEASIBLE, DSG_BUDGET, DSG_DEADLINE, DSG_INVALID, DSG_OVERFLOW,
 DSG_MISSING_BANDWIDTH, DSG_CUDA_ERROR, DSG_LOGIC, DSG_UNSUPPORTED) = range(10)

STATUS_NAMES = {
    DSG_OK: "OK", DSG_INFEASIBLE: "INFEASIBLE", DSG_BUDGET: "BUDGET",
    DSG_DEADLINE: "DEADLINE", DSG_INVALID: "INVALID", DSG_OVERFLOW: "OVERFLOW",
    DSG_MISSING_BANDWIDTH: "MISSING_BANDWIDTH", DSG_CUDA_ERROR: "CUDA_ERROR",
    DSG_LOGIC: "LOGIC", DSG_UNSUPPORTED: "UNSUPPORTED",
}


class dsg_rat(C.Structure):
    _fields_ = [("num", C.c_int64), ("den", C.c_int64)]


class dsg_graph(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32),
        ("ids", C.POINTER(C.c_int32)),
        ("cpu_time", C.POINTER(dsg_rat)),
        ("acc_time", C.POINTER(dsg_rat)),
        ("comm_time", C.POINTER(dsg_rat)),
        ("mem_size", C.POINTER(dsg_rat)),
        ("is_backward", C.POINTER(C.c_uint8)),
        ("forward_pair", C.POINTER(C.c_int32)),
        ("n_edges", C.c_int32),
        ("edge_from", C.POINTER(C.c_int32)),
        ("edge_to", C.POINTER(C.c_int32)),
        ("n_artificial", C.c_int32),
        ("art_from", C.POINTER(C.c_int32)),
        ("art_to", C.POINTER(C.c_int32)),
    ]


class dsg_config(C.Structure):
    _fields_ = [
        ("accelerators", C.c_int32),
        ("cpus", C.c_int32),
        ("memory_limit", dsg_rat),
        ("q", C.c_int32),
        ("interleaving", C.c_int32),
        ("has_bandwidth", C.c_int32),
        ("bandwidth", dsg_rat),
        ("replication_combine", C.c_int32),
    ]


class dsg_options(C.Structure):
    _fields_ = [
        ("ideal_budget", C.c_int64),
        ("deadline_seconds", C.c_double),
        ("device", C.c_int32),
        ("shard_count", C.c_int32),
        ("flags", C.c_int32),
        ("reserved", C.c_int32),
    ]


class dsg_block(C.Structure):
    _fields_ = [("cpu", C.c_int32), ("repl", C.c_int32), ("n_members", C.c_int32),
                ("offset", C.c_int32), ("load_num", C.c_int64)]


class dsg_result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("message", C.c_char * 256),
        ("budget_limit", C.c_int64),
        ("objective", dsg_rat),
        ("best_k", C.c_int32),
        ("best_l", C.c_int32),
        ("n_blocks", C.c_int32),
        ("blocks", C.POINTER(dsg_block)),
        ("members", C.POINTER(C.c_int32)),
        ("n_ideals", C.c_int64),
        ("n_pairs", C.c_int64),
        ("n_levels", C.c_int32),
        ("value_bits", C.c_int32),
        ("denominator", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("t_prepare_ms", C.c_double),
        ("t_enumerate_ms", C.c_double),
        ("t_describe_ms", C.c_double),
        ("t_dp_ms", C.c_double),
        ("t_traceback_ms", C.c_double),
        ("t_total_ms", C.c_double),
        ("t_transition_kernel_ms", C.c_double),
        ("t_device_ms", C.c_double),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("persistent_blocks", C.c_int32),
        ("block_loads", C.c_int32),
        ("words", C.c_int32),
        ("ideal_bits", C.POINTER(C.c_uint64)),
        ("dp_values", C.POINTER(C.c_int64)),
    ]


class dsg_ideals(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("message", C.c_char * 256),
        ("budget_limit", C.c_int64),
        ("count", C.c_int64),
        ("words", C.c_int32),
        ("bits", C.POINTER(C.c_uint64)),
        ("n_levels", C.c_int32),
        ("level_offsets", C.POINTER(C.c_int64)),
        ("t_ms", C.c_double),
    ]


class dsg_shard_handle(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("device", C.c_int32),
        ("n_ideals", C.c_int64),
        ("dp", C.c_uint8 * 64),
        ("bp", C.c_uint8 * 64),
        ("ctl", C.c_uint8 * 64),
    ]


def bind(lib: C.CDLL, prefix: str) -> None:
    """Declare argtypes for the <prefix>_dp_solve / _enumerate_ideals family."""
    solve = getattr(lib, f"{prefix}_dp_solve")
    solve.argtypes = [C.c_int32, C.POINTER(dsg_graph), C.POINTER(dsg_config),
                      C.POINTER(dsg_options), C.POINTER(dsg_result)]
    solve.restype = C.c_int
    rfree = getattr(lib, f"{prefix}_result_free")
    rfree.argtypes = [C.POINTER(dsg_result)]
    rfree.restype = None
    enum = getattr(lib, f"{prefix}_enumerate_ideals")
    enum.argtypes = [C.POINTER(dsg_graph), C.POINTER(C.c_uint8), C.c_int64,
                     C.POINTER(dsg_options), C.POINTER(dsg_ideals)]
    enum.restype = C.c_int
    ifree = getattr(lib, f"{prefix}_ideals_free")
    ifree.argtypes = [C.POINTER(dsg_ideals)]
    ifree.restype = None


def to_dsg_rat(x) -> tuple:
    if is_inf(x):
        return (1, 0)
    f = Fraction(x)
    return (f.numerator, f.denominator)


def from_dsg_rat(r) -> object:
    if r.den == 0:
        return INF
    return Fraction(r.num, r.den)


class PodGraph:
    """Owns the numpy buffers behind one dsg_graph (keep alive during calls)."""

    def __init__(self, g: Graph):
        nodes = g.nodes()
        n = len(nodes)
        self.n = n
        self.ids = np.array([nd.id for nd in nodes] or [0], dtype=np.int32)
        rt = np.dtype([("num", np.int64), ("den", np.int64)])

        def rats(attr):
            # one pass per column over Fraction's slots into an (n, 2) int64
            # buffer viewed as dsg_rat (properties and per-element structured
            # assignment dominate otherwise)
            a = np.zeros((max(n, 1), 2), dtype=np.int64)
            try:
                a[:n, 0] = [getattr(nd, attr)._numerator for nd in nodes]
                a[:n, 1] = [getattr(nd, attr)._denominator for nd in nodes]
            except AttributeError:  # int / float / INF weights
                pairs = [to_dsg_rat(getattr(nd, attr)) for nd in nodes]
                a[:n, 0] = [q for q, _ in pairs]
                a[:n, 1] = [d for _, d in pairs]
            return a.view(rt).reshape(-1)

        self.cpu = rats("cpu_time")
        self.acc = rats("acc_time")
        self.comm = rats("comm_time")
        self.mem = rats("mem_size")
        self.bw = np.array([1 if nd.is_backward else 0 for nd in nodes] or [0], dtype=np.uint8)
        self.pair = np.array([nd.forward_pair if nd.forward_pair is not None else DSG_NO_PAIR
                              for nd in nodes] or [0], dtype=np.int32)
        self.ef = np.array([e.src for e in g.edges()] or [0], dtype=np.int32)
        self.et = np.array([e.dst for e in g.edges()] or [0], dtype=np.int32)
        self.af = np.array([e.src for e in g.artificial_edges()] or [0], dtype=np.int32)
        self.at = np.array([e.dst for e in g.artificial_edges()] or [0], dtype=np.int32)
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        self.struct = dsg_graph(
            n, P(self.ids, C.c_int32), P(self.cpu, dsg_rat), P(self.acc, dsg_rat),
            P(self.comm, dsg_rat), P(self.mem, dsg_rat), P(self.bw, C.c_uint8),
            P(self.pair, C.c_int32), len(g.edges()), P(self.ef, C.c_int32),
            P(self.et, C.c_int32), len(g.artificial_edges()), P(self.af, C.c_int32),
            P(self.at, C.c_int32))


def pod_graph(g: Graph) -> PodGraph:
    if g._pod_cache is None:
        g._pod_cache = PodGraph(g)
    return g._pod_cache


def pod_config(cfg: DeviceConfig) -> dsg_config:
    return dsg_config(
        int(cfg.accelerators), int(cfg.cpus), dsg_rat(*to_dsg_rat(cfg.memory_limit)),
        int(cfg.q), int(cfg.interleaving), 1 if cfg.bandwidth is not None else 0,
        dsg_rat(*to_dsg_rat(cfg.bandwidth if cfg.bandwidth is not None else 0)),
        int(cfg.replication_combine))


def pod_options(budget: int = DSG_DEFAULT_IDEAL_BUDGET, deadline_seconds: Optional[float] = None,
                device: int = -1, shard_count: int = 0, flags: int = 0,
                max_blocks: int = 0) -> dsg_options:
    return dsg_options(int(budget), float(deadline_seconds or 0.0), int(device),
                       int(shard_count), int(flags), int(max_blocks))
