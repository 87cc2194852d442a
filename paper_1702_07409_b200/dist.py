"""Multi-GPU plumbing of the encode path -- host logic only.

One process per GPU.  The units of work are independent: stripes ("partitions are
processed independent of each other") for multi-stripe encodes, or, for a single large stripe,
coded-row ranges (reading R16) or byte-column ranges (every symbol XOR is bytewise, so columns are
independent; fs_encode_range).  The only collective is step a2: rank 0 generates the
graph (fs_graph_create) and broadcasts its CSR; the other ranks rebuild it with
fs_graph_from_csr.  There is no data-path collective.

Works with any torch.distributed backend: NCCL (device tensors) on the GPU box, gloo (CPU
tensors) in the CPU tests.
"""
import numpy as np
import torch

from . import fsb


def shard(total, world_size, rank):
    """Contiguous [begin, end) share of `total` units for `rank` (sizes differ by at most 1)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad world_size / rank")
    return rank * total // world_size, (rank + 1) * total // world_size


def col_shard(t, world_size, rank, align=64):
    """Contiguous byte range [c0, c1) of a t-byte symbol for `rank` (NEXT-4 column partition):
    boundaries on `align`-byte multiples (64 = one SMEM slice) except the final end t."""
    if t % 16:
        raise ValueError("t must be a multiple of 16")
    units = (t + align - 1) // align
    a, b = shard(units, world_size, rank)
    return min(a * align, t), min(b * align, t)


def broadcast_graph(cfg, group=None, device="cpu", host_only=False):
    """Step a2: rank 0 generates the graph, every rank returns an fsb.Graph with identical CSR.

    The four int32 CSR arrays travel as one flat tensor (one size broadcast, one data
    broadcast) on `device` (a CUDA device for NCCL, "cpu" for gloo)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if rank == 0:
        g = fsb.Graph.create(cfg, host_only=host_only)
        arrs = g.csr()
        sizes = torch.tensor([len(a) for a in arrs], dtype=torch.int64, device=device)
    else:
        g, arrs = None, None
        sizes = torch.zeros(4, dtype=torch.int64, device=device)
    dist.broadcast(sizes, 0, group=group)
    n = [int(x) for x in sizes.tolist()]
    if rank == 0:
        flat = torch.from_numpy(np.concatenate(arrs).astype(np.int32)).to(device)
    else:
        flat = torch.empty(sum(n), dtype=torch.int32, device=device)
    dist.broadcast(flat, 0, group=group)
    if rank == 0:
        return g
    host = flat.cpu().numpy()
    parts = np.split(host, np.cumsum(n)[:-1])
    return fsb.Graph.from_csr(cfg, *parts, host_only=host_only)


def gather_stripes(local, total, group=None):
    """the coded output to rank 0.  Every rank holds its contiguous stripe
    shard (`shard(total, world_size, rank)`) as `local` [S_r, ...]; rank 0 returns the whole
    [total, ...] tensor, the other ranks None.  Point-to-point receives straight into rank 0's
    slices (shards may differ in size by one, so no equal-size gather)."""
    import torch.distributed as dist
    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    if rank != 0:
        if local.shape[0]:
            for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(), 0, group)]):
                req.wait()
        return None
    out = torch.empty((total,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    b0, e0 = shard(total, ws, 0)
    out[b0:e0].copy_(local)
    ops = []
    for r in range(1, ws):
        b, e = shard(total, ws, r)
        if e > b:
            ops.append(dist.P2POp(dist.irecv, out[b:e], r, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out


def max_over_ranks(value, group=None, device="cpu"):
    """The max of a float over all ranks (the bench's timing rule)."""
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
