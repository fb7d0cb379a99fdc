#!/usr/bin/env python3
"""Time the UNMODIFIED reference solver (oracle/_ref/libdsg_ref.so, compiled
from /root/reference/proj/src by oracle/Makefile) on full workloads, on the
host cores of whatever box this runs on (SURVEY §8(d) "CPU baseline timing").

    python tools/cpu_ref_host.py OUT.json C2 [C4 C5:16,1,1,300 ...]

One solve per workload, 1 thread each (the reference is sequential by
contract); the workloads listed on one command line run one
after the other in this process.  tools/cpu_ref_host.sh starts several such
processes side by side and records lscpu.  Test/bench infrastructure: the
product never loads oracle/.
"""
from __future__ import annotations

import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_bind as ob  # noqa: E402  (checker / baseline only)
from paper_2006_16423_b200 import workloads as wl  # noqa: E402


def main():
    out = sys.argv[1]
    rows = []
    for name in sys.argv[2:]:
        w = wl.by_name(name)
        nv, ideals, pairs = w.counts
        mode = 1 if w.training else 0
        t = time.perf_counter()
        c0 = time.process_time()
        raw = ob.dp("ref", mode, w.graph, w.config)
        wall = time.perf_counter() - t
        cpu = time.process_time() - c0
        rows.append({
            "workload": name, "name": w.name, "nodes": w.graph.size(), "ideals": ideals,
            "pairs_closed_form": pairs, "k": w.config.accelerators, "l": w.config.cpus,
            "objective": str(raw.objective), "ref_wall_s": wall, "ref_cpu_s": cpu,
            "us_per_pair": 1e6 * wall / pairs, "transitions_per_s": pairs / wall,
            "maxrss_mb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024.0,
            "pid": os.getpid(), "host": os.uname().nodename,
        })
        with open(out, "w") as f:
            json.dump(rows, f, indent=1)
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
