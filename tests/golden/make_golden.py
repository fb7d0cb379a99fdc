"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs /root/reference and oracle/_ref built):

    make -C oracle all ref
    python tests/golden/make_golden.py [--standins] [--c2]

Outputs (all committed):
  random_instances.json  random_instance(seed) dumped by the compiled reference
                         test builders (tests/support/builders.cpp) via
                         dump_builders.cpp — pins workloads.random_instance
  dp_corpus.json         reference objectives: AC-1 corpus (seeds 0..199,
                         inference), AC-2 (mirrored, memory x2, training),
                         interleaving sweeps (seeds 800..829), seeded sweeps
                         from test_dp_solver.cpp, fixed known answers
  ideals.json            reference ideal lists (ordinal order) for small graphs
  standins.json          reference objectives for the C1..C4 / sweep stand-ins
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import time
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle_bind as ob  # noqa: E402
from paper_2006_16423_b200 import _abi  # noqa: E402
from paper_2006_16423_b200.errors import InfeasibleError  # noqa: E402
from paper_2006_16423_b200.graph import INF, DeviceConfig, Interleaving, is_inf  # noqa: E402
from paper_2006_16423_b200 import workloads as wl  # noqa: E402
from golden_io import graph_to_json, rat_to_json  # noqa: E402

REF = "/root/reference/proj"
JSON_DIR = None


def dump_builders():
    exe = os.path.join(ROOT, "oracle", "_ref", "dump_builders")
    objs = [os.path.join(ROOT, "oracle", "_ref", "obj", f) for f in sorted(os.listdir(os.path.join(ROOT, "oracle", "_ref", "obj")))]
    subprocess.run(["g++", "-O2", "-std=c++20", "-w", f"-I{REF}/include", f"-I{REF}/tests", "-o", exe,
                    os.path.join(HERE, "dump_builders.cpp"), f"{REF}/tests/support/builders.cpp", *objs],
                   check=True)
    out = {}
    for allow in (1, 0):
        lines = subprocess.run([exe, "0", "300", str(allow)], check=True, capture_output=True,
                               text=True).stdout.splitlines()
        out["allow_unsupported" if allow else "supported_only"] = [json.loads(l) for l in lines]
    return out


def ref_obj(mode, g, cfg):
    try:
        return rat_to_json(ob.dp("ref", mode, g, cfg).objective)
    except InfeasibleError:
        return "inf"


def dp_corpus():
    cases = []

    def add(name, mode, g, cfg, extra=None):
        t = time.time()
        obj = ref_obj(mode, g, cfg)
        cases.append(dict(name=name, mode=mode, graph=graph_to_json(g), k=cfg.accelerators,
                          l=cfg.cpus, M=rat_to_json(cfg.memory_limit), interleaving=int(cfg.interleaving),
                          objective=obj, ref_seconds=round(time.time() - t, 4), **(extra or {})))

    # AC-1: inference corpus (acceptance.cpp:74-94)
    for seed in range(200):
        inst = wl.random_instance(seed)
        add(f"ac1/{seed}", 0, inst.graph, inst.config)
    # AC-2: mirrored training corpus with memory x2 (acceptance.cpp:98-116)
    for seed in range(200):
        inst = wl.random_instance(seed)
        cfg = DeviceConfig(inst.config.accelerators, inst.config.cpus, inst.config.memory_limit * 2)
        add(f"ac2/{seed}", 1, wl.mirror_training(inst.graph), cfg)
    # interleaving modes (test_dp_solver.cpp:267-289)
    for mode_i in (Interleaving.HalfDuplexMax, Interleaving.FullDuplexMax):
        for seed in range(800, 830):
            inst = wl.random_instance(seed)
            cfg = DeviceConfig(inst.config.accelerators, inst.config.cpus, inst.config.memory_limit,
                               interleaving=mode_i)
            add(f"interleave{int(mode_i)}/{seed}", 0, inst.graph, cfg)
    # training exactness sweep (test_dp_solver.cpp:131-143)
    for seed in range(40, 64):
        inst = wl.random_instance(seed, allow_unsupported=False)
        cfg = DeviceConfig(inst.config.accelerators, max(inst.config.cpus, 1),
                           inst.config.memory_limit * 2)
        add(f"train_exact/{seed}", 1, wl.mirror_training(inst.graph), cfg)
    # monotone in k (test_dp_solver.cpp:325-338)
    for seed in range(600, 615):
        inst = wl.random_instance(seed, allow_unsupported=False)
        for k in (1, 2, 3):
            cfg = DeviceConfig(k, 1, inst.config.memory_limit)
            add(f"monotone/{seed}/k{k}", 0, inst.graph, cfg)
    # fixed known answers (test_dp_solver.cpp:82-122, 267-289)
    d4 = wl.diamond4()
    add("d4_k2_M4", 0, d4, DeviceConfig(2, 0, 4), dict(expect="6"))
    add("single", 0, wl.Graph([wl.make_node(1, 10, 2, 1, 1)]), DeviceConfig(1, 0, 4), dict(expect="2"))
    add("path2_tight", 0, wl.path_graph(2, 10, 2, 1, 1), DeviceConfig(1, 1, 1), dict(expect="10"))
    add("infeasible", 0, wl.Graph([wl.make_node(1, 1, 1, 0, 10)]), DeviceConfig(1, 0, 4),
        dict(expect="inf"))
    add("mirror_d4", 1, wl.mirror_training(d4), DeviceConfig(2, 0, 8), dict(expect="12"))
    add("d4_half", 0, d4, DeviceConfig(2, 0, 4, interleaving=Interleaving.HalfDuplexMax),
        dict(expect="4"))
    add("d4_training_on_inference_graph", 1, d4, DeviceConfig(2, 0, 4), dict(expect="6"))
    two = wl.Graph([wl.make_node(1, 0, 0, 0, 1), wl.make_node(2, 5, 5, 0, 1), wl.make_node(3, 3, 3, 0, 1),
                    wl.make_node(4, 1, 1, 0, 1), wl.make_node(5, 3, 3, 0, 1), wl.make_node(6, 0, 0, 0, 1)],
                   [wl.Edge(1, 2), wl.Edge(2, 3), wl.Edge(3, 6), wl.Edge(1, 4), wl.Edge(4, 5), wl.Edge(5, 6)])
    add("two_branch", 0, two, DeviceConfig(2, 0, 6), dict(expect="6"))
    return cases


def ideals():
    cases = []

    def add(name, g, within=None, budget=_abi.DSG_DEFAULT_IDEAL_BUDGET):
        try:
            ix = ob.enumerate_ideals("ref", g, within, budget)
            rows = [[int(x) for x in r] for r in ix.bits]
            cases.append(dict(name=name, graph=graph_to_json(g), within=within, budget=budget,
                              ideals=rows, level_offsets=[int(x) for x in ix.level_offsets]))
        except Exception as e:  # IdealBudgetExceeded
            cases.append(dict(name=name, graph=graph_to_json(g), within=within, budget=budget,
                              error=type(e).__name__))

    add("diamond4", wl.diamond4())
    add("path3", wl.path_graph(3, 1, 1, 0, 1))
    add("edgeless8", wl.edgeless(8))
    add("edgeless10", wl.edgeless(10))
    add("edgeless20_budget1000", wl.edgeless(20), budget=1000)
    add("d4_budget5", wl.diamond4(), budget=5)
    add("d4_budget6", wl.diamond4(), budget=6)
    for seed in range(15):
        g = wl.random_instance(seed).graph
        add(f"random/{seed}", g)
    for seed in range(40, 52):
        g = wl.mirror_training(wl.random_instance(seed).graph)
        add(f"mirror_fw/{seed}", g, within=sorted(g.forward_set()))
    c1 = wl.standin("C1")
    add("C1_fw", c1.graph, within=sorted(c1.graph.forward_set()))
    add("C3_chain", wl.module_chain(wl.SPECS["C3"]))
    return cases


def standins(include_c2: bool):
    out = []
    names = ["C1", "C3", "C4"] + (["C2"] if include_c2 else [])
    for name in names:
        w = wl.standin(name)
        t = time.time()
        obj = ref_obj(1 if w.training else 0, w.graph, w.config)
        dt = time.time() - t
        nv, ni, npairs = w.counts
        out.append(dict(name=name, objective=obj, ref_seconds=round(dt, 3), nodes=w.graph.size(),
                        fw_nodes=nv, ideals=ni, pairs=npairs, k=w.config.accelerators,
                        l=w.config.cpus, M=rat_to_json(w.config.memory_limit)))
        print(name, obj, f"{dt:.1f}s", flush=True)
    for pt in [(2, 8, 20, 100), (4, 3, 6, 30), (16, 1, 1, 20)]:
        w = wl.sweep(*pt)
        t = time.time()
        obj = ref_obj(0, w.graph, w.config)
        nv, ni, npairs = w.counts
        out.append(dict(name=f"sweep{pt}", point=list(pt), objective=obj,
                        ref_seconds=round(time.time() - t, 3), nodes=nv, ideals=ni, pairs=npairs,
                        k=w.config.accelerators, l=w.config.cpus, M=rat_to_json(w.config.memory_limit)))
        print(out[-1]["name"], obj, flush=True)
    return out


def main():
    if not ob.available("ref"):
        sys.exit("build oracle/_ref first: make -C oracle ref")
    with open(os.path.join(HERE, "random_instances.json"), "w") as f:
        json.dump(dump_builders(), f, separators=(",", ":"))
    with open(os.path.join(HERE, "dp_corpus.json"), "w") as f:
        json.dump(dp_corpus(), f, separators=(",", ":"))
    with open(os.path.join(HERE, "ideals.json"), "w") as f:
        json.dump(ideals(), f, separators=(",", ":"))
    if "--standins" in sys.argv or "--c2" in sys.argv:
        path = os.path.join(HERE, "standins.json")
        data = standins("--c2" in sys.argv)
        with open(path, "w") as f:
            json.dump(data, f, indent=1)


if __name__ == "__main__":
    main()
