"""Multi-process (replicas-only) plumbing of bench.py on CPU with gloo, world size 2.

The path does not shard: each rank factors its own replica and the
only cross-rank operations are a barrier and the max-over-ranks timing reduction.
Each rank here runs the CPU oracle on its own config-5-family replica, checks it,
and the aggregate throughput is computed exactly as bench.py does."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    import time

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import bench
    from oracle.bind import Checker, pivoting_matrix
    from paper_1802_10453_b200 import configs

    r, local, w = bench.dist_env()
    assert (r, local, w) == (rank, rank, world)
    dist = bench.init_dist(w, "gloo")
    wl = configs.Workload(5, 128, 131, 64, 5 + rank, "replica")
    a = configs.generate(wl)
    bench.barrier(dist)
    t0 = time.perf_counter()
    f = Checker("oracle").ldlt(wl.p, a)
    ms = (time.perf_counter() - t0) * 1e3 + 10.0 * rank  # distinct per-rank times
    tmax = bench.max_over_ranks(dist, ms)
    bench.barrier(dist)
    pi = pivoting_matrix(f)
    ok = f.rank == wl.r and all(
        (pi[i, j] == 1) == (j == p) for i, p in enumerate(configs.config5_partners(wl)) for j in range(wl.n)
        if p >= 0) 
    value = w * (2.0 * wl.n ** 3 / 3.0) / (tmax / 1e3)
    q.put((rank, ms, tmax, ok, value))
    dist.destroy_process_group()


def test_replicas_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    tmax = max(o[1] for o in out)
    for rank, ms, t, ok, value in out:
        assert ok, f"rank {rank}: replica factorization does not reveal R"
        assert abs(t - tmax) < 1e-9, "max-over-ranks reduction disagrees"
    assert abs(out[0][4] - out[1][4]) < 1e-6
