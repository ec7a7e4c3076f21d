"""One-process-per-GPU plumbing for the sharded count (torch.distributed).

The graph is replicated on every rank; each rank runs its cost-balanced share
of the clique and cycle work (gl_count_begin), the per-edge int64 partial rows
are summed with ONE reduce-scatter so that rank r owns the rows of edge shard
r (micro counts are then finalised per shard), and the 128-bit unrestricted
sums are combined with one all-reduce over 32-bit limbs (exact for any world
size below 2^31).  NCCL over NVLink on B200; gloo on CPU for the tests.
"""
from __future__ import annotations

import numpy as np

MASK32 = (1 << 32) - 1


def u128_to_limbs(vals) -> np.ndarray:
    """Each value -> 4 little-endian 32-bit limbs stored in int64."""
    out = np.zeros(4 * len(vals), dtype=np.int64)
    for i, v in enumerate(vals):
        v = int(v)
        if v < 0 or v >> 128:
            raise OverflowError("not an unsigned 128-bit value")
        for k in range(4):
            out[4 * i + k] = (v >> (32 * k)) & MASK32
    return out


def limbs_to_u128(arr) -> list:
    arr = np.asarray(arr, dtype=np.int64)
    vals = []
    for i in range(len(arr) // 4):
        v = 0
        for k in range(4):
            v += int(arr[4 * i + k]) << (32 * k)
        if v >> 128:
            raise OverflowError("128-bit count accumulator overflow")
        vals.append(v)
    return vals


def shard_range(m: int, world: int, rank: int):
    """Edge ids owned by `rank` after the reduce-scatter of the padded rows."""
    shard = (m + world - 1) // world if world else 0
    b = min(m, rank * shard)
    return b, min(m, b + shard)


def allreduce_u128(vals, group=None, device=None):
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(u128_to_limbs(vals))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return limbs_to_u128(t.cpu().numpy())


def exchange_partials(partials, world: int, group=None):
    """Sum the (2*plen,) int64 partial rows across ranks; return this rank's
    (2*shard,) slice.  NCCL: reduce_scatter_tensor; other backends: all_reduce
    + slice (gloo has no reduce-scatter)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return partials
    shard2 = partials.numel() // world
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(shard2, dtype=partials.dtype, device=partials.device)
        dist.reduce_scatter_tensor(out, partials, op=dist.ReduceOp.SUM, group=group)
        return out
    dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    return partials[rank * shard2:(rank + 1) * shard2].clone()


def allreduce_triangles(graph, world: int, group=None, stream=None):
    """Sum the per-edge uint32 triangle counts in place across ranks."""
    if world == 1:
        return
    import torch
    import torch.distributed as dist
    ptr, m = graph.triangle_counts_device()
    if m == 0:
        return
    dev = torch.device("cuda", graph.device)
    # uint32 counts are summed as int32 (wrap-around is exact mod 2^32 and
    # every final count is < 2^32): view the library buffer as a tensor.
    t = _tensor_from_ptr(ptr, m, torch.int32, dev)
    with torch.cuda.stream(stream or torch.cuda.current_stream(dev)):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def _tensor_from_ptr(ptr: int, n: int, dtype, device):
    """Zero-copy torch view of library-owned device memory (DLPack-free)."""
    import torch
    class _Arr:
        pass
    a = _Arr()
    a.__cuda_array_interface__ = {"shape": (n,), "typestr": torch.empty(0, dtype=dtype).numpy().dtype.str,
                                  "data": (ptr, False), "version": 3, "strides": None}
    return torch.as_tensor(a, device=device)


def sharded_step(graph, partials, rank: int, world: int, stream, group=None):
    """One full count with this rank's share of the work (see the C-ABI
    sequence in include/graphlet_b200.h).  `partials`: int64 device tensor of
    2*graph.partials_len(world).  Returns (X, (edge_begin, edge_end))."""
    import torch
    from . import global_from_unrestricted
    dev = partials.device
    if stream is None or stream.cuda_stream == 0:
        # the library maps a NULL stream to the graph's own non-blocking stream,
        # which nothing here would order against torch's collectives
        raise ValueError("sharded_step needs a dedicated (non-default) CUDA stream")
    graph.count_begin(rank, world, partials.data_ptr(), stream.cuda_stream)
    with torch.cuda.stream(stream):
        allreduce_triangles(graph, world, group, stream=stream)
        graph.count_mid(partials.data_ptr(), stream.cuda_stream)
        shard = exchange_partials(partials, world, group)
        b, e = shard_range(graph.num_edges(), world, rank)
        C = graph.count_finish(shard.data_ptr(), b, e, stream.cuda_stream)
        Ctot = allreduce_u128(C, group, device=dev) if world > 1 else C
    return global_from_unrestricted(Ctot, graph.num_vertices(), graph.num_edges()), (b, e)


def count_sharded(graph, rank: int, world: int, group=None, stream=None):
    """Full sharded count on this rank's GPU. Returns (X, (edge_begin, edge_end))."""
    import torch
    dev = torch.device("cuda", graph.device)
    partials = torch.empty(2 * graph.partials_len(world), dtype=torch.int64, device=dev)
    cur = torch.cuda.current_stream(dev)
    s = torch.cuda.Stream(dev) if stream is None else stream
    s.wait_stream(cur)  # partials were allocated / zeroed on the current stream
    out = sharded_step(graph, partials, rank, world, s, group)
    cur.wait_stream(s)
    return out
