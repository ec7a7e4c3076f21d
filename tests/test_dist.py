"""CPU, world_size 2 over gloo: the host side of the sharded count --
128-bit limb all-reduce, partial-row exchange and shard ownership."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1608_05138_b200.dist import (exchange_partials, limbs_to_u128, shard_range,
                                        u128_to_limbs, allreduce_u128)


def test_limbs_roundtrip():
    vals = [0, 1, 2**64 - 1, 2**64, 2**127 + 12345, 2**128 - 1]
    assert limbs_to_u128(u128_to_limbs(vals)) == vals
    with pytest.raises(OverflowError):
        u128_to_limbs([2**128])


def test_shard_ranges_cover_once():
    for m in (0, 1, 7, 100, 12345):
        for w in (1, 2, 3, 8):
            seen = []
            for r in range(w):
                b, e = shard_range(m, w, r)
                seen += list(range(b, e))
            assert seen == list(range(m))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # exact 128-bit sums across ranks (carry across limbs)
        vals = [2**127 - 1 + rank, 2**64 - 1, rank * 3]
        tot = allreduce_u128(vals)
        # per-edge partial rows: rank r contributes r+1 to x7 and -(r) to y (wraps)
        m = 11
        plen = ((m + world - 1) // world) * world
        parts = torch.zeros(2 * plen, dtype=torch.int64)
        parts[0:2 * m:2] = rank + 1
        parts[1:2 * m:2] = -rank
        shard = exchange_partials(parts, world)
        b, e = shard_range(m, world, rank)
        q.put((rank, tot, shard[: 2 * (e - b)].tolist(), b, e))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, tot, shard, b, e in out:
        assert tot == [2 * (2**127 - 1) + 1, 2 * (2**64 - 1), 3]
        assert shard == [3, -1] * (e - b)
    assert out[0][3] == 0 and out[-1][4] == 11
