"""Debug: dp tables with chain blocks on vs off (DSG_CHAIN_F) for a golden
corpus case or a workload; prints the first differing ordinal and its level.
    python tools/dbg_chain.py ac1/13     |   python tools/dbg_chain.py C1"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

name = sys.argv[1]
if len(sys.argv) > 2 and sys.argv[2] == "child":
    from paper_2006_16423_b200 import _abi, solver, workloads as wl
    if "/" in name:
        from golden_io import config_from_case, graph_from_json, load
        case = [c for c in load("dp_corpus.json") if c["name"] == name][0]
        g = graph_from_json(case["graph"])
        cfg = config_from_case(case)
        mode = case.get("mode", 0)
    else:
        w = wl.by_name(name)
        g, cfg, mode = w.graph, w.config, (1 if w.training else 0)
    raw = solver.run_dp(solver.load_library(), "dsg", mode, g, cfg,
                        solver.SolveOptions(flags=_abi.DSG_FLAG_KEEP_TABLES))
    np.save(sys.argv[3], raw.dp_values)
    lo = np.zeros(1)
    print("obj", raw.objective, "levels", raw.n_levels, "ideals", raw.n_ideals)
    sys.exit(0)

env_on = dict(os.environ)
env_off = dict(os.environ, DSG_CHAIN_F="0")
for tag, env in (("on", env_on), ("off", env_off)):
    r = subprocess.run([sys.executable, __file__, name, "child", f"/tmp/dp_{tag}.npy"], env=env,
                       capture_output=True, text=True)
    print(tag, r.stdout.strip(), r.stderr.strip()[-300:])
a, b = np.load("/tmp/dp_on.npy"), np.load("/tmp/dp_off.npy")
diff = np.nonzero((a != b).any(axis=1))[0]
print("rows differing:", len(diff), "first:", diff[:10])
for o in diff[:3]:
    print(o, "on", a[o], "\n   off", b[o])
