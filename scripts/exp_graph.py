#!/usr/bin/env python
"""Back-to-back layer launches: eager stream launches vs the same 16 launches replayed from a
CUDA graph.  Config 4 at kv-head shards N = 1 / 8 (rank 0's shard) and configs 2 / 3."""
import json
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, AttentionPlan  # noqa: E402
from paper_2312_05516_b200.sharding import shard_shape  # noqa: E402
from paper_2312_05516_b200.workloads import config  # noqa: E402

L = 16
dev = torch.device("cuda", 0)
res = []
for cfg, world in [(4, 1), (4, 8), (4, 4), (2, 1), (3, 1)]:
    w = config(cfg)
    shape = shard_shape(w.shape(), 0, world)
    pool = w.n_slots * w.chunk * shape.n_kv_head * w.head_size
    ks = [torch.empty(pool, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    vs = [torch.empty(pool, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    for l in range(L):
        abi.fill_unit(ks[l].data_ptr(), PB_BF16, pool, 11, 2 * l * pool)
        abi.fill_unit(vs[l].data_ptr(), PB_BF16, pool, 11, (2 * l + 1) * pool)
    q = torch.empty(w.total_tokens * shape.n_head * w.head_size, dtype=torch.bfloat16, device=dev)
    abi.fill_unit(q.data_ptr(), PB_BF16, q.numel(), 12, 0)
    out = torch.empty_like(q)
    s = torch.cuda.Stream()
    plan = AttentionPlan(shape, w.batch())
    plan.upload(s.cuda_stream)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device=dev)

    def layers():
        for l in range(L):
            plan.run(q.data_ptr(), ks[l].data_ptr(), vs[l].data_ptr(), out.data_ptr(), ws.data_ptr(), s.cuda_stream)

    with torch.cuda.stream(s):
        for _ in range(3):
            layers()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        layers()
    torch.cuda.synchronize()
    ref = out.clone()

    def timed(fn):
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            fn()
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / L)
        return statistics.median(ts)

    with torch.cuda.stream(s):
        e1 = timed(layers)
        g1 = timed(g.replay)
        e2 = timed(layers)
        g2 = timed(g.replay)
    same = torch.equal(out.view(torch.int16), ref.view(torch.int16))
    res.append({"cfg": cfg, "world": world, "eager_us": [round(e1, 2), round(e2, 2)],
                "graph_us": [round(g1, 2), round(g2, 2)], "same_bytes": same})
    print(json.dumps(res[-1]), flush=True)
    del ks, vs, g
    torch.cuda.empty_cache()
