#!/usr/bin/env python
"""Diagnostics: streaming rate of decode units inside a fused launch.  A batch of n decode
spans x ctx cached tokens (64 query / 8 kv heads, d 128, 16-token pages) plus one 2-token
prefill span, so the launch is fused; with n_kv % 8 == 0 the decode units are head-group units
(one per span, decode_hg_cta.cuh).  Compared with the same spans as per-head units in the
stand-alone decode kernel (PB_PLAN_SEPARATE_DECODE + PB_PLAN_NO_SPLIT)."""
import json
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import gpu_helpers as gh  # noqa: E402
from paper_2312_05516_b200.abi import PB_PLAN_NO_SPLIT, PB_PLAN_SEPARATE_DECODE, AttentionPlan  # noqa: E402
from paper_2312_05516_b200.workloads import PB_BF16, SplitMix64, _build  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"ctx": ctx}
for n in (8, 20, 40):
    w = _build(f"hg{n}", 64, 8, 128, 16, PB_BF16, 7, [[(ctx, 1)] for _ in range(n)] + [[(0, 2)]], SplitMix64(7))
    q, k, v = gh.device_inputs(w)
    st = torch.cuda.current_stream().cuda_stream
    out = torch.empty_like(q)
    for name, flags in (("fused_hg", 0), ("separate_per_head", PB_PLAN_SEPARATE_DECODE | PB_PLAN_NO_SPLIT)):
        plan = AttentionPlan(w.shape(), w.batch(), flags)
        plan.upload(st)
        ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(13):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(4):
                plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), st)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / 4)
        us = statistics.median(ts[3:])
        by = n * ctx * 8 * 2 * 128 * 2
        res[f"{name}_{n}"] = {"us": round(us, 1), "GBs": round(by / us / 1e3, 1), "units": plan.stats()["decode_units"]}
        del plan, ws
    del q, k, v, out
    torch.cuda.empty_cache()
print(json.dumps(res))
