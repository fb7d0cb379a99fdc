"""Robustness sweep: solve configurations across the supported range (wide
bitsets, training, many cells, int64, large lattices) on the device, check
every split with the independent verifier, and print status and time.

    python tools/stress.py
"""
import os
import sys
import time
import traceback
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import _abi, solver, workloads as wl  # noqa: E402
from paper_2006_16423_b200.graph import DeviceConfig, verify_split  # noqa: E402

cases = []
for pt in [(8, 2, 7, 1900), (8, 2, 7, 3900), (16, 1, 2, 1900), (4, 4, 8, 1400)]:
    cases.append((f"sweep{pt}", wl.sweep(*pt), 0))
for pt in [(8, 2, 7, 1400)]:
    cases.append((f"sweep{pt}@int64", wl.sweep(*pt), _abi.DSG_FLAG_FORCE_INT64))
# training on wide graphs
for n_stem, mods in [(900, [[3, 2]] * 4), (1900, [[4, 2]] * 3)]:
    g = wl.module_chain(wl.ChainSpec(n_stem, mods, 2))
    tr = wl.mirror_training(g)
    cases.append((f"train stem{n_stem} n{tr.size()}", (tr, DeviceConfig(6, 2, 10 ** 6)), 0))
# many cells (generic cells): K = 16, L = 4
g = wl.module_chain(wl.ChainSpec(1000, [[3, 2]] * 4, 2))
cases.append(("K16 L4 n%d" % g.size(), (g, DeviceConfig(16, 4, 10 ** 6)), 0))
for name, w, flags in cases:
    if isinstance(w, tuple):
        g, cfg = w
        training = g.has_backward_nodes()
    else:
        g, cfg, training = w.graph, w.config, w.training
    t = time.time()
    try:
        f = solver.solve_maxload_training if training else solver.solve_maxload_inference
        split = f(g, cfg, solver.SolveOptions(flags=flags))
        bad = verify_split(g, cfg, split, training=training)
        print(f"{name:34s} ok obj {split.objective_value} ideals {split.stats['n_ideals']} "
              f"pairs {split.stats['n_pairs']} bits {split.stats['value_bits']} "
              f"{(time.time() - t) * 1e3:.1f} ms verify {'OK' if not bad else bad}", flush=True)
    except Exception as e:
        print(f"{name:34s} FAIL {type(e).__name__}: {e}", flush=True)
        traceback.print_exc(limit=2)
