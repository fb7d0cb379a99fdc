"""Where the e2e solve time goes: host flatten, dsg_dp_solve phases, canonical split."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import _abi, solver, workloads as wl
from paper_2006_16423_b200.graph import make_canonical_split
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = wl.standin(name)
mode = 1 if w.training else 0
lib = solver.load_library()
solver.run_dp(lib, "dsg", mode, w.graph, w.config, solver.SolveOptions())
for _ in range(5):
    w.graph._pod_cache = None
    t0 = time.perf_counter()
    pg = _abi.pod_graph(w.graph)
    t1 = time.perf_counter()
    w.graph._pod_cache = None
    raw = solver.run_dp(lib, "dsg", mode, w.graph, w.config, solver.SolveOptions(flags=_abi.DSG_FLAG_TIME_KERNELS))
    t2 = time.perf_counter()
    split = make_canonical_split(w.graph, w.config, raw.blocks, raw.objective)
    t3 = time.perf_counter()
    st = {k: round(v, 3) for k, v in raw.stats.items() if k.startswith("t_")}
    print(f"pod_graph {1e3*(t1-t0):.3f} ms  run_dp {1e3*(t2-t1):.3f} ms  split {1e3*(t3-t2):.3f} ms  {st}")
