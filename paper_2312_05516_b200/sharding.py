"""KV-head sharding across GPUs (SURVEY §8 e).

Rank r of G owns kv heads [r*n_kv/G, (r+1)*n_kv/G) and the query heads that read them
(head h reads kv head h / group, proj/src/attention.cpp:91, so they are the contiguous block
[r*n_head/G, (r+1)*n_head/G)).  Spans, block tables and slot ids are identical on every
rank — "each worker follows the same migration plan" — so the only
control-plane traffic is one broadcast of the batch descriptors per step; the attention
itself has no collective.  n_kv % G == 0 is required (proj/src/model_config.cpp:25-26).
"""
from __future__ import annotations

import numpy as np

from . import abi
from .abi import AttnShape, Batch


def shard_shape(shape: AttnShape, rank: int, world: int) -> AttnShape:
    """The rank's shard shape (pb_shard_shape; ConfigError for a bad rank, DimensionMismatch
    when n_kv_head % world != 0)."""
    return abi.shard_shape(shape, rank, world)[0]


def shard_heads(shape: AttnShape, rank: int, world: int):
    """(first query head, first kv head) of the rank's shard."""
    _, h0, k0 = abi.shard_shape(shape, rank, world)
    return h0, k0


def pack_batch(b: Batch) -> np.ndarray:
    """Flatten the descriptors into one int64 vector (what rank 0 broadcasts)."""
    n = b.n_spans
    return np.concatenate([np.array([n, b.bt_off[-1]], np.int64), b.query_len, b.causal_offset,
                           b.bt[: int(b.bt_off[-1])].astype(np.int64), b.bt_off])


def unpack_batch(v: np.ndarray) -> Batch:
    n, nbt = int(v[0]), int(v[1])
    ql = v[2:2 + n]
    co = v[2 + n:2 + 2 * n]
    bt = v[2 + 2 * n:2 + 2 * n + nbt].astype(np.int32)
    off = v[2 + 2 * n + nbt:2 + 3 * n + nbt + 1]
    return Batch(ql, co, [bt[off[i]:off[i + 1]] for i in range(n)])


def broadcast_batch(batch, group=None, src: int = 0) -> Batch:
    """Rank `src` sends its batch descriptors to every rank (torch.distributed, gloo or nccl
    — with nccl the caller passes a CPU-capable group or the tensor is staged on the GPU)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    n = torch.zeros(1, dtype=torch.int64, device=dev)
    if rank == src:
        flat = torch.from_numpy(pack_batch(batch)).to(dev)
        n[0] = flat.numel()
    dist.broadcast(n, src, group=group)
    if rank != src:
        flat = torch.empty(int(n.item()), dtype=torch.int64, device=dev)
    dist.broadcast(flat, src, group=group)
    return unpack_batch(flat.cpu().numpy())
