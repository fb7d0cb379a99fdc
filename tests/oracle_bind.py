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
