"""Multi-GPU wavefront protocol, world_size 2 over gloo on CPU.

The device path (persistent.cu + dsg_session_shard_*) shards each level's
target units across ranks: a level with >= 16 targets is cut into groups of
32 targets, a smaller level into single-target units; rank r owns the units
with unit % world == r, and every finished dp row is delivered to every
rank before any rank may read it.  This test runs that exact partition and
exchange (rows all-gathered per level) on a plain Python DP, and checks that
both ranks end with the same table as an unsharded solve, and with the
oracle's optimum.  It also exercises ShardComm.from_torch (the handle
all-gather and barrier the CUDA path uses) on a real gloo group.
"""
import os
import socket
from fractions import Fraction

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def units_of_level(T: int):
    """Target units of a level, as in capi.cu's plan (kSmallLevel = 16)."""
    if T < 16:
        return [[t] for t in range(T)]
    return [list(range(u * 32, min(T, u * 32 + 32))) for u in range((T + 31) // 32)]


def dp_rows(g, cfg, ideals, level_off, targets, table, K, L):
    """dp rows of `targets` (ordinals) from the finished rows in `table`
    (apply_candidate + monotone_pass, dp_solver.cpp:180-233)."""
    from paper_2006_16423_b200.graph import INF, acc_cost, cpu_cost
    out = {}
    for t in targets:
        I = ideals[t]
        row = [[INF] * (L + 1) for _ in range(K + 1)]
        lvl = next(s for s in range(len(level_off) - 1) if level_off[s] <= t < level_off[s + 1])
        for s in range(level_off[lvl]):
            if not ideals[s] <= I:
                continue
            block = I - ideals[s]
            acc = acc_cost(g, block, cfg)
            cpu = cpu_cost(g, block)
            src = table[s]
            for k in range(K + 1):
                for l in range(L + 1):
                    if k >= 1 and acc != INF and src[k - 1][l] != INF:
                        row[k][l] = min(row[k][l], max(src[k - 1][l], acc))
                    if l >= 1 and src[k][l - 1] != INF:
                        row[k][l] = min(row[k][l], max(src[k][l - 1], cpu))
        for k in range(K + 1):
            for l in range(L + 1):
                if k > 0:
                    row[k][l] = min(row[k][l], row[k - 1][l])
                if l > 0:
                    row[k][l] = min(row[k][l], row[k][l - 1])
        out[t] = row
    return out


def sharded_dp(g, cfg, ideals, level_off, rank, world, all_gather):
    K, L = cfg.accelerators, cfg.cpus
    table = {0: [[Fraction(0)] * (L + 1) for _ in range(K + 1)]}
    for s in range(1, len(level_off) - 1):
        lo, hi = level_off[s], level_off[s + 1]
        mine = [lo + t for u, unit in enumerate(units_of_level(hi - lo)) if u % world == rank
                for t in unit]
        rows = dp_rows(g, cfg, ideals, level_off, mine, table, K, L)
        for part in all_gather(rows):  # the NVLink row exchange
            table.update(part)
        assert all(t in table for t in range(lo, hi)), "a target of the level was not delivered"
    return table


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_16423_b200.solver import ShardComm
        import oracle_bind as ob
        from paper_2006_16423_b200 import workloads as wl
        from dag_gen import random_dag
        comm = ShardComm.from_torch()
        # the handle exchange: byte blobs come back in rank order
        blobs = comm.all_gather_bytes(bytes([rank]) * 200)
        assert [b[0] for b in blobs] == list(range(world)) and all(len(b) == 200 for b in blobs)
        comm.barrier()

        def gather(rows):
            out = [None] * world
            dist.all_gather_object(out, rows)
            return out

        results = []
        cases = [(wl.diamond4(), wl.DeviceConfig(2, 0, 4)),
                 (wl.module_chain(wl.ChainSpec(2, [[3, 2, 2]], 1)), wl.DeviceConfig(3, 1, 30))]
        for seed in (3, 11, 27):
            cases.append(random_dag(seed, n_lo=6, n_hi=9))
        for g, cfg in cases:
            ix = ob.enumerate_ideals("port", g)
            ideals = ix.ideals
            level_off = [int(x) for x in ix.level_offsets]
            table = sharded_dp(g, cfg, ideals, level_off, rank, world, gather)
            full = sharded_dp(g, cfg, ideals, level_off, 0, 1, lambda rows: [rows])
            assert table == full
            best = table[len(ideals) - 1][cfg.accelerators][cfg.cpus]
            want = ob.objective_or_inf("port", 0, g, cfg)
            assert best == want, (best, want)
            results.append(str(best))
        q.put((rank, results))
    except Exception as e:  # surface worker failures to the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libdsg_oracle.so")),
                    reason="oracle not built")
def test_two_rank_wavefront_matches_unsharded():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(isinstance(v, list) for v in out.values()), out
    assert out[0] == out[1]


def test_unit_partition_covers_every_target_once():
    for T in [1, 5, 15, 16, 17, 31, 32, 33, 100, 1000]:
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                seen += [t for u, unit in enumerate(units_of_level(T)) if u % world == r for t in unit]
            assert sorted(seen) == list(range(T))
