"""GPU: the multi-GPU decode path.

* pqkv_decode_sharded on a one-rank NCCL communicator: a batch of layers
  decoded and all-gathered in one call equals the per-layer pqkv_decode
  outputs bit for bit, in the documented [rank][layer][unit] layout
  (including padding rows of a short shard).
* Two processes (world size 2, gloo) on cuda:0: each rank decodes its head
  shard of the same layer with pqkv_decode and the shards are all-gathered;
  the result equals one process decoding every head (only one GPU is
  available here, and NCCL refuses two ranks on one device, so the two-rank
  run gathers over gloo; the NCCL all-gather itself is the one-rank case)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _layer(ctx, P, S, g, seed, b=6):
    import torch

    import paper_2407_12820_b200 as pq

    n_init, n_local = 4, 64
    keys, vals, q = ctx.gen_workload(S, 128, h_kv=P, g=g, kind="gaussian", seed=seed)
    s_mid = S - n_init - n_local
    cen, codes = ctx.pq_build(keys[:, n_init:n_init + s_mid].contiguous(), 2, b, 4, list(range(seed, seed + P)))
    tabs = ctx.tuple_tables(codes, b)
    torch.cuda.synchronize()
    return pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=S, n_init=n_init,
                          n_local=n_local, b=b, tables=tabs), q


def test_decode_sharded_one_rank_equals_decode(ctx):
    import torch

    import paper_2407_12820_b200 as pq
    from paper_2407_12820_b200 import shard

    S, k, g = 20000, 4000, 2
    layers, qs = zip(*[_layer(ctx, P, S, g, seed) for P, seed in ((6, 3), (5, 11))])  # second shard is short
    comm = ctx.comm_init(pq.comm_unique_id(), 1, 0)
    try:
        out = ctx.decode_sharded(comm, list(layers), list(qs), k, units_per_rank=6)
        torch.cuda.synchronize()
    finally:
        comm.close()
    assert tuple(out.shape) == (1, 2, 6, g, 128)
    for li, (layer, q) in enumerate(zip(layers, qs)):
        want = ctx.decode(layer, q, k)
        n = layer.keys.shape[0]
        assert torch.equal(out[0, li, :n], want), f"layer {li}"
        assert torch.count_nonzero(out[0, li, n:]) == 0  # padding rows
    full = shard.unshard(out, 6)
    assert tuple(full.shape) == (2, 6, g, 128)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, path):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2407_12820_b200 as pq
    from paper_2407_12820_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = pq.Context(0)
    layer, q = _layer(ctx, 7, 12000, 4, 21)  # same seeds on every rank: the same layer
    hr = shard.partition(7, world, rank)
    th, ch = layer.tables
    sub = pq.DecodeLayer(keys=layer.keys[hr.start:hr.stop], values=layer.values[hr.start:hr.stop],
                         centroids=layer.centroids[hr.start:hr.stop], codes=layer.codes[hr.start:hr.stop],
                         total=layer.total, n_init=layer.n_init, n_local=layer.n_local, b=layer.b,
                         tables=(th[hr.start:hr.stop], ch[hr.start:hr.stop]))
    local = ctx.decode(sub, q[hr.start:hr.stop].contiguous(), 2400).cpu()
    full = shard.gather_heads(local, 7)
    if rank == 0:
        np.save(path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()


def test_two_ranks_decode_shards_and_gather(ctx, tmp_path):
    import torch
    import torch.multiprocessing as mp

    path = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(2, _free_port(), path), nprocs=2, join=True, start_method="spawn")
    got = np.load(path)
    layer, q = _layer(ctx, 7, 12000, 4, 21)
    want = ctx.decode(layer, q, 2400).cpu().numpy()
    assert got.shape == want.shape
    # a shard's chunking differs from the full layer's (fp32 merge order)
    assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max()
