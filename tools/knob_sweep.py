"""Sweep max_blocks for a workload (env knobs are set by the caller).

    python tools/knob_sweep.py C4 0,148,296,592
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import solver, workloads as wl
name = sys.argv[1]
w = wl.standin(name) if not name.startswith("C5") else wl.sweep(*map(int, name[3:].split(",")))
for mb in map(int, sys.argv[2].split(",")):
    s = solver.Session(1 if w.training else 0, w.graph, w.config, solver.SolveOptions(max_blocks=mb))
    ts = []
    for _ in range(6):
        r = s.run()
        ts.append(r.stats["t_dp_ms"])
    s.close()
    print(name, os.environ.get("DSG_POLL_NS", "-"), os.environ.get("DSG_CRIT_CTAS", "-"), "max_blocks", mb,
          "t_dp_ms", round(sorted(ts[1:])[len(ts[1:]) // 2], 3), "obj", r.objective)
