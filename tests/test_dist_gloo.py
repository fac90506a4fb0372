"""World-size-2 coverage of the N>1 host path on CPU (gloo): request sharding, blob exchange, and the
max-over-ranks timing the bench reports.  The data path has no collective, so this is all there is
to exchange between ranks."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2605_22850_b200 import dist as ocd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = ocd.shard_requests(11, world, rank)
        blobs = ocd.exchange_blobs(f"store-of-rank-{rank}".encode() * (rank + 1))
        t = ocd.max_over_ranks(1.5 + rank)
        s = ocd.sum_over_ranks(len(mine))
        homes = [i % 3 for i in range(9)]
        aff = ocd.shard_requests(9, world, rank, homes)
        q.put((rank, mine, blobs, t, s, aff))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, m0, b0, t0, s0, a0), (r1, m1, b1, t1, s1, a1) = res
    assert sorted(m0 + m1) == list(range(11)) and not set(m0) & set(m1)
    assert abs(len(m0) - len(m1)) <= 1
    assert b0 == b1 == [b"store-of-rank-0", b"store-of-rank-1" * 2]
    assert t0 == t1 == 2.5
    assert s0 == s1 == 11
    assert a0 == [0, 2, 3, 5, 6, 8] and a1 == [1, 4, 7]


def test_shard_single_rank_and_errors():
    assert ocd.shard_requests(5, 1, 0) == [0, 1, 2, 3, 4]
    assert ocd.max_over_ranks(3.0) == 3.0
    assert ocd.exchange_blobs(b"x") == [b"x"]
    with pytest.raises(ValueError):
        ocd.shard_requests(5, 2, 2)
    with pytest.raises(ValueError):
        ocd.shard_requests(5, 2, 0, homes=[0, 1])
