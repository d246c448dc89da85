#!/usr/bin/env python
"""Diagnostics: what bounds the tile pipeline on the config-4 prefill spans?  Times the tile
items alone (the 16 prefill spans of config 4, no decode units) with the page size varied, so
the number of TMA boxes per 64-row kv tile changes (16-token pages: 8 boxes per K or V tile;
32: 4; 64: 2) while the arithmetic stays identical.  Run once per variant library (the
ablation builds) to separate tensor, softmax and TMA-issue costs.

  python scripts/exp_tile_bounds.py [reps] [page sizes, default 16]
"""
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
from paper_2312_05516_b200.workloads import PB_BF16, SplitMix64, _build, config  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
chunks = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16]
base = config(4)
pre = [(off, q) for _, off, q in base.spans if q > 1]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"spans": len(pre)}
for chunk in chunks:
    w = _build(f"cfg4-prefill-c{chunk}", 64, 8, 128, chunk, PB_BF16, 4, [[s] for s in pre], SplitMix64(4))
    q, k, v = gh.device_inputs(w)
    plan = AttentionPlan(w.shape(), w.batch())
    st = torch.cuda.current_stream().cuda_stream
    plan.upload(st)
    out = torch.empty_like(q)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), st)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = statistics.median(ts[3:])
    fl, _ = w.flops_bytes()
    res[f"chunk{chunk}"] = {"us": round(us, 1), "tflops": round(fl / us / 1e6, 1), "stats": plan.stats()}
    del q, k, v, out, ws, plan
    torch.cuda.empty_cache()
print(json.dumps(res))
