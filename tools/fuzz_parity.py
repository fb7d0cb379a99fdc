"""Randomised parity sweep on the device against the oracle port: module-chain
graphs of 60-900 nodes (ragged and wide word counts), K in 1..16, L in 0..4,
inference, replication (bandwidth, both combine rules) and mirrored training,
all three interleaving modes, with and without binding memory limits.

    python tools/fuzz_parity.py [N] [SEED]
"""
import os
import random
import sys
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402
from paper_2006_16423_b200 import solver, workloads as wl  # noqa: E402
from paper_2006_16423_b200.errors import InfeasibleError  # noqa: E402
from paper_2006_16423_b200.graph import (INF, DeviceConfig, Interleaving,  # noqa: E402
                                         ReplicationCombine, verify_split)

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
fails = 0
t0 = time.time()
for i in range(n_cases):
    mods = [[rng.randint(2, 4), rng.randint(1, 3)] for _ in range(rng.randint(1, 2))]
    spec = wl.ChainSpec(rng.randint(30, 850), mods, rng.randint(0, 3))
    g = wl.module_chain(spec, seed=rng.randint(1, 10 ** 6), decimals=rng.choice([1, 2]))
    training = rng.random() < 0.35
    if training:
        g = wl.mirror_training(g)
    K, L = rng.randint(1, 16), rng.randint(0, 4)
    if K + L < 1:
        K = 1
    total_mem = sum(n.mem_size for n in g.nodes())
    M = rng.choice([Fraction(10 ** 9), total_mem / max(1, K) * Fraction(rng.randint(12, 30), 10)])
    replicated = not training and rng.random() < 0.25
    if replicated:
        K = min(K, 8)
        cfg = DeviceConfig(K, L, M, interleaving=Interleaving(rng.randint(0, 2)),
                           bandwidth=Fraction(rng.randint(1, 40), rng.choice([1, 10])),
                           replication_combine=ReplicationCombine(rng.randint(0, 1)))
    else:
        cfg = DeviceConfig(K, L, M, interleaving=Interleaving(rng.randint(0, 2)))
    mode = 1 if training else (2 if replicated else 0)
    try:
        want = ob.dp("port", mode, g, cfg).objective
    except InfeasibleError:
        want = INF
    f = (solver.solve_maxload_training if training else
         solver.solve_maxload_replicated if replicated else solver.solve_maxload_inference)
    try:
        split = f(g, cfg)
        got = split.objective_value
        bad = verify_split(g, cfg, split, training=training)
    except InfeasibleError:
        got, bad = INF, []
    ok = got == want and not bad
    fails += 0 if ok else 1
    print(f"{i:3d} n={g.size():4d} mode={mode} K={K:2d} L={L} il={int(cfg.interleaving)} "
          f"{'ok' if ok else 'MISMATCH'} got={got} want={want} {bad if bad else ''}", flush=True)
print(f"{n_cases - fails}/{n_cases} ok in {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
