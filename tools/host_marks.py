"""Host step timestamps of a few dsg_dp_solve calls (DSG_PREP_TRACE=1):
    DSG_PREP_TRACE=1 python tools/host_marks.py C1 [calls]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import _abi, solver, workloads as wl

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 5
lib = solver.load_library()
w = wl.by_name(name)
pg = _abi.pod_graph(w.graph)
cfg = _abi.pod_config(w.config)
po = _abi.pod_options(10**7, 0, 0, 0, 0, 0)
res = _abi.dsg_result()
for i in range(calls):
    print(f"--- call {i}", file=sys.stderr, flush=True)
    lib.dsg_dp_solve(1 if w.training else 0, C.byref(pg.struct), C.byref(cfg), C.byref(po), C.byref(res))
    print(f"device {res.t_device_ms:.3f} ms total {res.t_total_ms:.3f} ms", file=sys.stderr, flush=True)
    lib.dsg_result_free(C.byref(res))
