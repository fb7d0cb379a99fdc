"""Writers for the reference's workload JSON (ingest.cpp:42-229) and runners
for the reference command line (tools/dagsplit_main.cpp) built twice by
integration/Makefile: on the B200 drop-in (dagsplit_b200) and on the
unmodified CPU reference (dagsplit_ref, the checker)."""
from __future__ import annotations

import json
import os
import subprocess
from fractions import Fraction

from paper_2006_16423_b200.graph import is_inf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
CLI_B200 = os.path.join(BUILD, "dagsplit_b200")
CLI_REF = os.path.join(BUILD, "dagsplit_ref")
INTERLEAVING = ["sum", "halfDuplexMax", "fullDuplexMax"]


def _num(x):
    f = Fraction(x)
    return int(f) if f.denominator == 1 else float(f)


def workload_json(g, cfg) -> str:
    dev = {"accelerators": cfg.accelerators, "cpus": cfg.cpus,
           "interleaving": INTERLEAVING[int(cfg.interleaving)]}
    if not is_inf(cfg.memory_limit):
        dev["memoryLimit"] = _num(cfg.memory_limit)
    else:
        dev["memoryLimit"] = 1e15
    nodes = []
    for n in g.nodes():
        row = {"id": n.id, "cpuTime": _num(n.cpu_time),
               "accTime": None if is_inf(n.acc_time) else _num(n.acc_time),
               "commTime": _num(n.comm_time), "memory": _num(n.mem_size)}
        if n.is_backward:
            row["isBackward"] = True
            row["forwardPair"] = n.forward_pair
        nodes.append(row)
    edges = [{"from": e.src, "to": e.dst} for e in g.edges()]
    return json.dumps({"devices": dev, "nodes": nodes, "edges": edges})


def run_cli(binary, *args, timeout=600):
    return subprocess.run([binary, *map(str, args)], capture_output=True, text=True,
                          timeout=timeout)


def strip_wall(text: str) -> str:
    return "\n".join(l for l in text.splitlines() if "wallTimeSeconds" not in l)
