"""CPU, world_size 2 over gloo: the multi-GPU host logic of the decode path
(unit partition, max-over-ranks timing, head all-gather) -- the same code
bench.py runs over NCCL."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_12820_b200 import shard


def test_partition_covers_units_once():
    for n in [1, 7, 32, 33, 128]:
        for world in [1, 2, 3, 4, 8]:
            owned = [u for r in range(world) for u in shard.partition(n, world, r)]
            assert owned == list(range(n))
            sizes = [len(shard.partition(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.partition(4, 2, 2)


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
        out = {}
        for n_heads in (32, 7):  # even and uneven head splits
            mine = shard.partition(n_heads, world, rank)
            # each rank "decodes" its heads: a deterministic function of the head id
            local = torch.stack([torch.full((2, 8), float(h)) + torch.arange(8.0) for h in mine])
            out[n_heads] = shard.gather_heads(local, n_heads).tolist()
        q.put((rank, out, shard.max_over_ranks(1.0 + rank)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_gather_and_max():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, slowest in res:
        for n_heads, full in out.items():
            want = torch.stack([torch.full((2, 8), float(h)) + torch.arange(8.0) for h in range(n_heads)])
            assert full == want.tolist()
        assert slowest == 2.0
