"""t_dp_ms vs persistent grid size (and the per-level-launch path)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import solver, _abi, workloads as wl
for name in sys.argv[1:] or ["C1", "C4", "C2"]:
    w = wl.standin(name)
    row = {"name": name}
    for mb in [1, 16, 148, 296, 592, 1184, -1]:
        flags = _abi.DSG_FLAG_LEVEL_LAUNCH if mb == -1 else 0
        s = solver.Session(1 if w.training else 0, w.graph, w.config,
                           solver.SolveOptions(flags=flags, max_blocks=max(mb, 0)))
        ts = []
        for _ in range(3):
            ts.append(s.run().stats["t_dp_ms"])
        row[str(mb)] = round(min(ts), 3)
        s.close()
    print(json.dumps(row), flush=True)
