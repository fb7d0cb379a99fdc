"""TEST INFRASTRUCTURE: ctypes bindings for the checkers under oracle/.

  port  -> oracle/_build/libdsg_oracle.so  (C restatement, dsgo_*)
  ref   -> oracle/_ref/libdsg_ref.so       (unmodified reference, dsgref_*)

Only tests/, bench.py's cpu_baseline / --impl reference leg and
__graft_entry__.smoke() use these, as checkers.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

from paper_2006_16423_b200 import _abi
from paper_2006_16423_b200.graph import DeviceConfig, Graph, make_canonical_split
from paper_2006_16423_b200.solver import SolveOptions, run_dp, run_enumerate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT_PATH = os.path.join(ROOT, "oracle", "_build", "libdsg_oracle.so")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libdsg_ref.so")

_libs = {}


def _load(kind: str) -> Optional[C.CDLL]:
    if kind in _libs:
        return _libs[kind]
    path, prefix = (PORT_PATH, "dsgo") if kind == "port" else (REF_PATH, "dsgref")
    lib = None
    if os.path.exists(path):
        lib = C.CDLL(path)
        _abi.bind(lib, prefix)
    _libs[kind] = lib
    return lib


def available(kind: str) -> bool:
    return _load(kind) is not None


def prefix(kind: str) -> str:
    return "dsgo" if kind == "port" else "dsgref"


def dp(kind: str, mode: int, g: Graph, cfg: DeviceConfig, opt: Optional[SolveOptions] = None):
    lib = _load(kind)
    if lib is None:
        raise FileNotFoundError(f"oracle library '{kind}' not built")
    return run_dp(lib, prefix(kind), mode, g, cfg, opt)


def solve(kind: str, mode: int, g: Graph, cfg: DeviceConfig, opt: Optional[SolveOptions] = None):
    raw = dp(kind, mode, g, cfg, opt)
    return make_canonical_split(g, cfg, raw.blocks, raw.objective), raw


def enumerate_ideals(kind: str, g: Graph, within=None, budget: int = _abi.DSG_DEFAULT_IDEAL_BUDGET):
    lib = _load(kind)
    if lib is None:
        raise FileNotFoundError(f"oracle library '{kind}' not built")
    return run_enumerate(lib, prefix(kind), g, within, budget)


def objective_or_inf(kind: str, mode: int, g: Graph, cfg: DeviceConfig):
    from paper_2006_16423_b200.errors import InfeasibleError
    from paper_2006_16423_b200.graph import INF
    try:
        return dp(kind, mode, g, cfg).objective
    except InfeasibleError:
        return INF


def ref_topo_order(g: Graph, seed: int):
    """seeded_topo_order of the unmodified reference (dp_solver.cpp:407-438)."""
    lib = _load("ref")
    if lib is None:
        raise FileNotFoundError("oracle/_ref not built")
    fn = lib.dsgref_topo_order
    fn.argtypes = [C.POINTER(_abi.dsg_graph), C.c_uint64, C.POINTER(C.c_int32)]
    fn.restype = C.c_int
    pg = _abi.pod_graph(g)
    out = (C.c_int32 * max(1, g.size()))()
    n = fn(C.byref(pg.struct), seed, out)
    return [int(out[i]) for i in range(n)]


def ref_dpl(g: Graph, cfg: DeviceConfig, seed: int):
    """solve_dpl of the unmodified reference (dp_solver.cpp:462-477)."""
    from paper_2006_16423_b200.errors import raise_for_status
    from paper_2006_16423_b200.solver import _raw_from
    lib = _load("ref")
    if lib is None:
        raise FileNotFoundError("oracle/_ref not built")
    fn = lib.dsgref_dpl_solve
    fn.argtypes = [C.POINTER(_abi.dsg_graph), C.POINTER(_abi.dsg_config), C.c_uint64,
                   C.POINTER(_abi.dsg_options), C.POINTER(_abi.dsg_result)]
    fn.restype = C.c_int
    pg = _abi.pod_graph(g)
    pc = _abi.pod_config(cfg)
    po = _abi.pod_options(_abi.DSG_DEFAULT_IDEAL_BUDGET, 0.0, -1, 1, 0, 0)
    res = _abi.dsg_result()
    fn(C.byref(pg.struct), C.byref(pc), seed, C.byref(po), C.byref(res))
    try:
        raise_for_status(res.status, res.message, res.budget_limit)
        return _raw_from(res, cfg)
    finally:
        lib.dsgref_result_free(C.byref(res))
