"""TEST INFRASTRUCTURE: an independent checker for path graphs at sizes the
oracle ports cannot reach (up to 4,096 nodes = 64 bitset words).

On a path the ideals are exactly the n+1 prefixes, so the reference DP
(dp_solver.cpp:319-351: apply_candidate's accelerator branch + monotone_pass,
L = 0) reduces to dp[i][k] = min(dp[i][k-1], min_j max(dp[j][k-1], cost(j, i)))
with cost(j, i) = acc_cost of nodes j..i-1 (graph.cpp:397-473, Sum mode):
Σacc + comm[j-1] (producer j-1, j > 0) + comm[i-1] (i < n), ∞ when
Σmem > M.  Integer weights keep it exact in int64 numpy."""
from __future__ import annotations

import numpy as np

from paper_2006_16423_b200.graph import Edge, Graph, make_node

INF64 = np.iinfo(np.int64).max // 4


def random_path(n: int, seed: int):
    rng = np.random.default_rng(seed)
    acc = rng.integers(1, 20, n)
    comm = rng.integers(0, 10, n)
    mem = rng.integers(1, 5, n)
    cpu = rng.integers(10, 100, n)
    nodes = [make_node(i + 1, int(cpu[i]), int(acc[i]), int(comm[i]), int(mem[i])) for i in range(n)]
    g = Graph(nodes, [Edge(i, i + 1) for i in range(1, n)])
    return g, acc, comm, mem


def path_maxload(acc, comm, mem, K: int, M: int) -> int:
    n = len(acc)
    pa = np.concatenate([[0], np.cumsum(acc)])
    pm = np.concatenate([[0], np.cumsum(mem)])
    j = np.arange(n + 1)
    cin = np.where(j > 0, np.concatenate([[0], comm])[j], 0)
    prev = np.full(n + 1, INF64, dtype=np.int64)
    prev[0] = 0  # k = 0: only the empty prefix
    for _ in range(K):
        cur = prev.copy()  # monotone pass: dp[i][k] <= dp[i][k-1]
        cur[0] = 0
        for i in range(1, n + 1):
            js = j[:i]
            cost = pa[i] - pa[js] + cin[js] + (comm[i - 1] if i < n else 0)
            cost = np.where(pm[i] - pm[js] > M, INF64, cost)
            cand = np.maximum(prev[js], cost).min()
            cur[i] = min(cur[i], cand)
        prev = cur
    return int(prev[n])
