#!/usr/bin/env python
"""Diagnostics: per-SM streaming rate of the tcgen05 decode pipeline.  A decode-only batch of
n spans x 4096 cached tokens, one kv head, GQA-8, d 128 (whole-span units, PB_PLAN_NO_SPLIT),
so n CTAs each stream 4 MiB of K+V.  Prints GB/s per active CTA for several n; the fused
launch's decode CTAs run in this regime (a few dozen CTAs next to tensor-bound tiles)."""
import json
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import gpu_helpers as gh  # noqa: E402
from paper_2312_05516_b200.abi import PB_PLAN_NO_SPLIT, AttentionPlan  # noqa: E402
from paper_2312_05516_b200.workloads import PB_BF16, SplitMix64, _build  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 16  # page tokens (TMA box rows)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"ctx": ctx, "chunk": chunk}
for n in (20, 148):
    w = _build(f"dec{n}", 8, 1, 128, chunk, PB_BF16, 7, [[(ctx, 1)] for _ in range(n)], SplitMix64(7))
    q, k, v = gh.device_inputs(w)
    plan = AttentionPlan(w.shape(), w.batch(), PB_PLAN_NO_SPLIT)
    st = torch.cuda.current_stream().cuda_stream
    plan.upload(st)
    out = torch.empty_like(q)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):  # four back-to-back launches: host enqueue latency off the clock
            plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), st)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 4)
    us = statistics.median(ts[3:])
    by = n * ctx * 2 * 128 * 2
    res[n] = {"us": round(us, 1), "GBs": round(by / us / 1e3, 1), "GBs_per_cta": round(by / us / 1e3 / min(n, 148), 1),
              "units": plan.stats()["decode_units"]}
    del q, k, v, out, ws, plan
    torch.cuda.empty_cache()
print(json.dumps(res))
