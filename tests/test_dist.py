"""Multi-process plumbing of the sharded bench path on CPU (gloo, world 2):
item shards cover the batch exactly once, the step time is the max over
ranks, and per-rank results reassemble in item order."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_0906_2704_b200 import dist


def test_shard_partition():
    for total in (0, 1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = dist.shard(total, r, world)
                seen.extend(range(s, s + c))
            assert seen == list(range(total))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    r, w, _ = dist.init(backend="gloo")
    total = 11
    start, count = dist.shard(total, r, w)
    local = torch.arange(start, start + count, dtype=torch.float64)[:, None] * torch.ones(1, 3)
    t = dist.max_over_ranks(1.0 + r)
    s = dist.sum_over_ranks(float(count))
    full = dist.gather_items(local, total)
    if r == 0:
        q.put((t, s, full[:, 0].tolist()))
    dist.finalize()


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, s, items = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0 and s == 11.0 and items == list(range(11))
