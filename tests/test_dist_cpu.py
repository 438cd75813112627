"""Multi-rank plumbing on CPU (gloo, world_size 2): byte-balanced shard
ranges + the record all-gather used by bench.py / multi-GPU runs. The
per-rank evaluator here is the oracle standing in for each rank's engine
(test double); the result must equal the single-rank evaluation exactly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1902_09215_b200.sharding import shard_ranges


def test_shard_ranges_cover_and_balance():
    rng = np.random.default_rng(0)
    sizes = (10 ** rng.uniform(4, 6, 4000)).astype(np.uint64) | 1
    for world in (1, 2, 4, 8):
        r = shard_ranges(sizes, world)
        assert r[0][0] == 0 and sum(c for _, c in r) == 4000
        assert all(r[g][0] + r[g][1] == r[g + 1][0] for g in range(world - 1))
        loads = [int(sizes[f:f + c].sum()) for f, c in r]
        assert max(loads) - min(loads) <= 2 * int(sizes.max())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_1902_09215_b200 as ltgp
    from paper_1902_09215_b200.sharding import gather_records
    from tests._oracle import load_oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = load_oracle()
        suite = ltgp.make_suite(ltgp.suite_seed(3))
        sizes = ltgp.corpus_sizes(9, 60, 2.0, 4.0)
        ranges = shard_ranges(sizes, world)
        first, count = ranges[rank]
        buf, offs, sz = ltgp.corpus(9, 60, 2.0, 4.0, first=first, n=count)
        local = o.evaluate_population(buf, offs, sz, suite, threads=1)
        t = torch.from_numpy(local.view(np.uint8).copy())
        full = gather_records(t, ranges)
        q.put((rank, full.tobytes()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_gather_equals_single_rank(oracle):
    import paper_1902_09215_b200 as ltgp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    suite = ltgp.make_suite(ltgp.suite_seed(3))
    buf, offs, sz = ltgp.corpus(9, 60, 2.0, 4.0)
    exp = oracle.evaluate_population(buf, offs, sz, suite, threads=1)
    assert res[0] == res[1] == exp.tobytes()
