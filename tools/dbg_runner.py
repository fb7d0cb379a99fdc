import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from golden_io import config_from_case, graph_from_json, load
from paper_2006_16423_b200 import solver
CORPUS = load("dp_corpus.json")
case = [c for c in CORPUS if c["name"] == "ac1/2"][0]
g = graph_from_json(case["graph"]); cfg = config_from_case(case)
print("mode", case["mode"], "n", g.size(), "k,l", cfg.accelerators, cfg.cpus)
lib = solver.load_library()
try:
    r = solver.run_dp(lib, "dsg", case["mode"], g, cfg, solver.SolveOptions(flags=0))
    print("ok", r.objective, r.stats)
except Exception as e:
    print("ERR", e)
