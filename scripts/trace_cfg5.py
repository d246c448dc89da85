#!/usr/bin/env python
"""Diagnostics: the config-5 (ShareGPT-like trace) attention batches — plan statistics and a
per-CTA timeline of one launch per planned step (no swaps)."""
import json
import math
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, AttentionPlan, AttnShape  # noqa: E402

steps, dev_slots, host_slots = bench.plan_sharegpt_steps(96, 6)
n_head, n_kv, d, chunk = 40, 10, 128, 16
dev = torch.device("cuda", 0)
page_elems = chunk * n_kv * d
k = torch.empty((dev_slots, page_elems), dtype=torch.bfloat16, device=dev)
v = torch.empty_like(k)
abi.fill_unit(k.data_ptr(), PB_BF16, k.numel(), 5, 0)
abi.fill_unit(v.data_ptr(), PB_BF16, v.numel(), 5, k.numel())
shape = AttnShape(n_head, n_kv, d, chunk, dev_slots, PB_BF16, math.sqrt(d))
stream = torch.cuda.current_stream().cuda_stream
for i, p in enumerate(steps[:3]):
    b = p.batch()
    plan = AttentionPlan(shape, b)
    plan.upload(stream)
    q = torch.empty(max(1, b.total_tokens) * n_head * d, dtype=torch.bfloat16, device=dev)
    abi.fill_unit(q.data_ptr(), PB_BF16, q.numel(), 6, 0)
    out = torch.empty_like(q)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device=dev)
    tr = torch.zeros(148 * 2 * 4, dtype=torch.int64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for r in range(5):
        if r == 4:
            plan.set_trace(tr.data_ptr())
            ev[0].record()
        plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), stream)
    ev[1].record()
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(148, 2, 4)
    begins = t[:, :, 2][t[:, :, 2] > 0]
    ends = t[:, :, 3][t[:, :, 3] > 0]
    st = plan.stats()
    ql = list(b.query_len)
    res = {"step": i, "spans": b.n_spans, "tokens": int(b.total_tokens), "prefill_spans": sum(1 for x in ql if x > 1),
           "max_q": int(max(ql)) if ql else 0, "ctx_max": int(max(b.context_len)) if ql else 0,
           "stats": {kk: st[kk] for kk in ("prefill_tiles", "decode_units", "split_spans", "bytes")},
           "launch_us": round(ev[0].elapsed_time(ev[1]) * 1e3, 1)}
    if len(begins):
        t0 = begins.min()
        res["ctas"] = int((t[:, 0, 2] > 0).sum())
        res["cta_end_us"] = [round((ends.min() - t0) / 1e3, 1), round(statistics.median((ends - t0) / 1e3), 1),
                             round((ends.max() - t0) / 1e3, 1)]
    res["hbm_gbs"] = round(st["bytes"] / (res["launch_us"] * 1e-6) / 1e9, 1)
    print(json.dumps(res))
