"""KV-head sharding host logic on CPU with torch.distributed gloo, world_size 2 (the N>1 path
of bench.py): rank 0 broadcasts the batch descriptors, every rank builds its shard's plan,
and together the shards cover every (token, head) row exactly once with the same spans and
block tables."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_05516_b200.abi import AttentionPlan
        from paper_2312_05516_b200.sharding import broadcast_batch, pack_batch, shard_heads, shard_shape
        from paper_2312_05516_b200.workloads import config

        w = config(4)  # Llama-2-70B GQA-8: 8 kv heads
        batch = broadcast_batch(w.batch() if rank == 0 else None)
        shape = shard_shape(w.shape(), rank, world)
        plan = AttentionPlan(shape, batch)
        st = plan.stats()
        digest = torch.tensor([float(np.sum(pack_batch(batch).astype(np.float64) * np.arange(1, pack_batch(batch).size + 1)))])
        gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, digest.double())
        rows = torch.tensor([float(st["rows"])], dtype=torch.float64)
        dist.all_reduce(rows)
        flops = torch.tensor([st["flops"]], dtype=torch.float64)
        dist.all_reduce(flops)
        q.put((rank, shard_heads(w.shape(), rank, world), shape.n_head, shape.n_kv_head,
               [float(g.item()) for g in gathered], float(rows.item()), float(flops.item()),
               w.total_tokens * w.n_head, w.flops_bytes()[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_kv_head_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, h0, nh, nkv, digests, rows, flops, want_rows, want_flops) = res[0]
    assert nh == 64 // world and nkv == 8 // world
    assert [r[1] for r in res] == [(r * nh, r * nkv) for r in range(world)]
    assert len(set(digests)) == 1  # identical descriptors everywhere
    assert rows == want_rows  # shards tile every (token, head) row once
    assert flops == pytest.approx(want_flops, rel=1e-12)


def test_shard_shape_rejects_indivisible_heads():
    from paper_2312_05516_b200.abi import DimensionMismatch
    from paper_2312_05516_b200.sharding import shard_shape
    from paper_2312_05516_b200.workloads import config

    with pytest.raises(DimensionMismatch):
        shard_shape(config(3).shape(), 0, 4)  # 10 kv heads over 4 ranks
