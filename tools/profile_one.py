"""One warm resident solve of a workload (for ncu: profile the last launch)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import solver, _abi, workloads as wl
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = wl.by_name(name)
s = solver.Session(1 if w.training else 0, w.graph, w.config, solver.SolveOptions(flags=flags))
for _ in range(reps):
    r = s.run()
print(name, r.objective, r.n_pairs, {k: round(v, 3) for k, v in r.stats.items() if k.startswith("t_")})
