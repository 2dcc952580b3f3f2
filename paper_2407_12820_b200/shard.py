"""Multi-GPU plumbing for the decode path.

(request, layer, kv_head) units are independent in both hot paths, so the
path shards without any data exchange: each rank owns a contiguous range of
units.  The only collective is the all-gather of per-head attention outputs
when one layer's heads are split across ranks (BASELINE cfg4), which the next
layer's projection needs: in the product it runs inside the C ABI
(pqkv_decode_sharded: the rank's decodes of a batch of layers, then one NCCL
all-gather on a collective stream); torch.distributed only exchanges the NCCL
unique id (nccl_comm) and, in the CPU tests, stands in for the gather over
gloo (gather_heads).
"""
from __future__ import annotations


def partition(n_units: int, world: int, rank: int) -> range:
    """Contiguous balanced range of units owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard: bad world/rank")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_heads(local_out, n_heads: int):
    """All-gather per-head outputs [h_local][g][d_h] of a head-sharded layer
    into [n_heads][g][d_h] on every rank (head order = rank order)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local_out
    world = dist.get_world_size()
    sizes = [len(partition(n_heads, world, r)) for r in range(world)]
    rest = tuple(local_out.shape[1:])
    if len(set(sizes)) == 1:
        out = torch.empty((n_heads,) + rest, dtype=local_out.dtype, device=local_out.device)
        dist.all_gather_into_tensor(out, local_out.contiguous())
        return out
    # uneven split: pad every rank's slice to the largest, gather, trim
    mx = max(sizes)
    pad = torch.zeros((mx,) + rest, dtype=local_out.dtype, device=local_out.device)
    pad[: local_out.shape[0]] = local_out
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], 0)


def nccl_comm(ctx):
    """The libpqkv NCCL communicator of this torch.distributed job: rank 0's
    unique id is broadcast over the process group (any backend)."""
    import torch.distributed as dist

    import paper_2407_12820_b200 as pq

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    box = [pq.comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(box, src=0)
    return ctx.comm_init(box[0], world, rank)


def unshard(gathered, n_heads: int):
    """[n_ranks][n_layers][units_per_rank][g][d_h] from pqkv_decode_sharded ->
    [n_layers][n_heads][g][d_h] in head order (drops the padding rows of
    ranks that own fewer heads)."""
    import torch

    world = gathered.shape[0]
    sizes = [len(partition(n_heads, world, r)) for r in range(world)]
    return torch.cat([gathered[r, :, :sizes[r]] for r in range(world)], dim=1)
