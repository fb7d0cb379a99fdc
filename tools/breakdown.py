"""Per-phase timing of one resident solve (dsg_session_run) per workload."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import solver, _abi, workloads as wl
names = sys.argv[1:] or ["C2", "C3", "C4", "C1"]
for name in names:
    w = wl.standin(name)
    s = solver.Session(1 if w.training else 0, w.graph, w.config,
                       solver.SolveOptions(flags=_abi.DSG_FLAG_TIME_KERNELS))
    for _ in range(3):
        r = s.run()
    out = {k: round(v, 3) if isinstance(v, float) else v for k, v in r.stats.items()}
    out.update(name=name, levels=r.n_levels, ideals=r.n_ideals, pairs=r.n_pairs)
    print(json.dumps(out), flush=True)
    s.close()
