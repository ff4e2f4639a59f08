"""Multi-process host logic of the N>1 bench path, on CPU with gloo (world 2):
disjoint pulse shards per (step, rank), max-over-ranks timing, and that the
per-rank shards reproduce the single-process oracle results exactly (pulses
are independent units; Philox counters and ids use global pulse indices)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    import bench
    import oracle
    from workloads import make_workload
    r, w_, _ = bench.dist_setup("gloo")
    assert (r, w_) == (rank, world)
    wl = make_workload("C4", 0.1)
    B = 700
    got = []
    for step in range(3):
        start, cnt = bench.shard(wl.n_pulses, B, step, rank, world)
        ids = np.arange(start, start + cnt)
        o, d, t = wl.pulses(start, cnt)
        res = oracle.simulate(wl.scene, wl.params, o, d, t, ids.astype(np.uint64), n_threads=2)
        got.append((start, cnt, res.n_returns.copy(), res.sub_prim.copy()))
    mx = bench.max_over_ranks(float(rank + 1) * 1.5, world)
    bench.barrier(world)
    q.put((rank, mx, got))
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert all(mx == 3.0 for _, mx, _ in out)  # max over ranks of 1.5, 3.0
    ranges = [(s, c) for _, _, got in out for s, c, _, _ in got]
    spans = sorted(ranges)
    for (s0, c0), (s1, _) in zip(spans, spans[1:]):
        assert s0 + c0 <= s1  # disjoint
    # per-rank results equal a single-process run over the same pulses
    sys.path.insert(0, ROOT)
    import oracle
    from workloads import make_workload
    wl = make_workload("C4", 0.1)
    for _, _, got in out:
        for start, cnt, nret, prim in got:
            o, d, t = wl.pulses(start, cnt)
            ref = oracle.simulate(wl.scene, wl.params, o, d, t,
                                  np.arange(start, start + cnt, dtype=np.uint64), n_threads=4)
            assert np.array_equal(ref.n_returns, nret)
            assert np.array_equal(ref.sub_prim, prim)


def test_shard_covers_workload_without_overlap_single_rank():
    import bench
    seen = set()
    for step in range(10):
        s, c = bench.shard(10_000, 1000, step, 0, 1)
        assert (s, c) not in seen and s % 1000 == 0 and c == 1000
        seen.add((s, c))
