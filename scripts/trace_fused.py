#!/usr/bin/env python
"""Diagnostics: per-CTA timeline of one fused launch (pb_attn_set_trace).  Prints, per mode,
how many CTAs started there, when the passes began/ended relative to the launch start, and
the idle tail (last CTA end - median CTA end)."""
import json
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import gpu_helpers as gh  # noqa: E402
from paper_2312_05516_b200.abi import AttentionPlan  # noqa: E402
from paper_2312_05516_b200.workloads import config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # rank 0 of an N-way kv-head shard
w = config(cfg)
from paper_2312_05516_b200.sharding import shard_shape  # noqa: E402
shape = shard_shape(w.shape(), 0, world)
w.n_kv_head, w.n_head = shape.n_kv_head, shape.n_head
q, k, v = gh.device_inputs(w)
plan = AttentionPlan(shape, w.batch())
stream = torch.cuda.current_stream().cuda_stream
plan.upload(stream)
out = torch.empty_like(q)
ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
tr = torch.zeros(148 * 2 * 4, dtype=torch.int64, device="cuda")
for i in range(4):
    if i == 3:
        plan.set_trace(tr.data_ptr())
    plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), stream)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(148, 2, 4)
t0 = t[:, :, 2][t[:, :, 2] > 0].min()
rows = []
for b in range(148):
    for ps in range(2):
        mode, _, beg, end = t[b, ps]
        if beg > 0:
            rows.append((b, ps, int(mode), (beg - t0) / 1e3, (end - t0) / 1e3))
res = {"config": cfg, "world": world, "stats": plan.stats()}
for mode in (0, 1):
    first = [r for r in rows if r[1] == 0 and r[2] == mode]
    second = [r for r in rows if r[1] == 1 and r[2] == mode]
    res[f"mode{mode}"] = {
        "ctas_first": len(first),
        "first_end_us": [round(min(r[4] for r in first), 1), round(statistics.median(r[4] for r in first), 1),
                         round(max(r[4] for r in first), 1)] if first else None,
        "ctas_stealing": len(second),
        "steal_dur_us": [round(min(r[4] - r[3] for r in second), 1),
                         round(statistics.median(r[4] - r[3] for r in second), 1),
                         round(max(r[4] - r[3] for r in second), 1)] if second else None,
    }
ends = [max(r[4] for r in rows if r[0] == b) for b in range(148) if any(r[0] == b for r in rows)]
res["cta_end_us"] = [round(min(ends), 1), round(statistics.median(ends), 1), round(max(ends), 1)]
print(json.dumps(res))
