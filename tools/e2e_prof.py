"""cProfile of the e2e call path (flatten + dsg_dp_solve + canonical split)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import solver, workloads as wl
from paper_2006_16423_b200.graph import make_canonical_split
w = wl.standin(sys.argv[1] if len(sys.argv) > 1 else "C2")
mode = 1 if w.training else 0
lib = solver.load_library()
def step():
    w.graph._pod_cache = None
    raw = solver.run_dp(lib, "dsg", mode, w.graph, w.config, solver.SolveOptions())
    make_canonical_split(w.graph, w.config, raw.blocks, raw.objective)
    return raw
for _ in range(3):
    step()
t = time.perf_counter()
for _ in range(20):
    raw = step()
print("e2e ms", (time.perf_counter() - t) / 20 * 1e3, {k: round(v, 3) for k, v in raw.stats.items() if k.startswith("t_")})
cProfile.run("for _ in range(20): step()", "/tmp/e2e.prof")
pstats.Stats("/tmp/e2e.prof").sort_stats("tottime").print_stats(14)
