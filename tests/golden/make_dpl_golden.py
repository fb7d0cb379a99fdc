"""Generate tests/golden/dpl.json from the UNMODIFIED reference (oracle/_ref):
seeded_topo_order (dp_solver.cpp:407-438) and solve_dpl objectives
(dp_solver.cpp:462-477) on the AC-1 random instances, their mirrored training
forms and D4, for several seeds.

    make -C oracle ref && python tests/golden/make_dpl_golden.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import oracle_bind as ob  # noqa: E402
from golden_io import graph_to_json, rat_to_json  # noqa: E402
from paper_2006_16423_b200 import workloads as wl  # noqa: E402
from paper_2006_16423_b200.errors import InfeasibleError  # noqa: E402
from paper_2006_16423_b200.graph import DeviceConfig  # noqa: E402


def case(name, g, cfg, seed):
    try:
        obj = rat_to_json(ob.ref_dpl(g, cfg, seed).objective)
    except InfeasibleError:
        obj = "inf"
    return dict(name=name, graph=graph_to_json(g), k=cfg.accelerators, l=cfg.cpus,
                M=rat_to_json(cfg.memory_limit), interleaving=int(cfg.interleaving), seed=seed,
                order=ob.ref_topo_order(g, seed), objective=obj)


def main():
    out = []
    for seed in (0, 1, 7, 12345):
        out.append(case(f"d4/s{seed}", wl.diamond4(), DeviceConfig(2, 0, 4), seed))
    for i in range(40):
        inst = wl.random_instance(i)
        out.append(case(f"ac1/{i}/s{i % 5}", inst.graph, inst.config, i % 5))
    for i in range(20):
        inst = wl.random_instance(100 + i)
        g = wl.mirror_training(inst.graph)
        cfg = DeviceConfig(inst.config.accelerators, inst.config.cpus, inst.config.memory_limit * 2,
                           interleaving=inst.config.interleaving)
        out.append(case(f"ac2/{100 + i}/s{i % 3}", g, cfg, i % 3))
    spec = wl.ChainSpec(4, [[3, 2, 1], [2, 2]], 3)
    out.append(case("chain/s3", wl.module_chain(spec), DeviceConfig(3, 1, 40), 3))
    with open(os.path.join(HERE, "dpl.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(len(out), "cases")


if __name__ == "__main__":
    main()
