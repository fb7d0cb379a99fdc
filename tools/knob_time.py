"""Median DP-kernel / device ms of warm resident solves (knob sweeps).

    python tools/knob_time.py WORKLOAD [REPS]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import solver, workloads as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
w = wl.by_name(name)
s = solver.Session(1 if w.training else 0, w.graph, w.config,
                   solver.SolveOptions(max_blocks=int(os.environ.get("DSG_KNOB_BLOCKS", "0")), flags=w.flags))
dp, dev = [], []
for i in range(reps + 3):
    r = s.run()
    if i >= 3:
        dp.append(r.stats["t_dp_ms"])
        dev.append(r.stats["t_device_ms"])
print(f"{name} obj {r.objective} pairs {r.n_pairs} dp_ms {statistics.median(dp):.3f} "
      f"dev_ms {statistics.median(dev):.3f} enum_ms {r.stats['t_enumerate_ms']:.3f}")
