#!/usr/bin/env python
"""Diagnostics: how the config-4 batch's time splits between its tile items and decode units.
Times one layer (CUDA events, L2 flushed before each rep) of: the fused launch (product
default), the same batch as separate tile + decode launches (PB_PLAN_SEPARATE_DECODE), the
prefill spans alone and the decode spans alone.

  python scripts/exp_fused_split.py [cfg] [world] [reps]
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
from paper_2312_05516_b200.abi import PB_PLAN_NO_SPLIT, PB_PLAN_SEPARATE_DECODE, AttentionPlan  # noqa: E402
from paper_2312_05516_b200.sharding import shard_shape  # noqa: E402
from paper_2312_05516_b200.workloads import PB_BF16, SplitMix64, _build, config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
base = config(cfg)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(w, flags=0):
    shape = shard_shape(w.shape(), 0, world)
    w.n_kv_head, w.n_head = shape.n_kv_head, shape.n_head
    q, k, v = gh.device_inputs(w)
    plan = AttentionPlan(shape, w.batch(), flags)
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
    r = {"us": round(statistics.median(ts[3:]), 1), "stats": plan.stats()}
    del q, k, v, out, ws, plan
    torch.cuda.empty_cache()
    return r


convs = [[(off, ql)] for _, off, ql in base.spans]
pre = [[(off, ql)] for _, off, ql in base.spans if ql > 1]
dec = [[(off, ql)] for _, off, ql in base.spans if ql == 1]
mk = lambda name, cv: _build(name, base.n_head, base.n_kv_head, base.head_size, base.chunk, PB_BF16, cfg, cv,
                             SplitMix64(cfg))
res = {"config": cfg, "world": world,
       "fused": timed(mk("all", convs)),
       "separate": timed(mk("all", convs), PB_PLAN_SEPARATE_DECODE),
       "fused_no_split": timed(mk("all", convs), PB_PLAN_NO_SPLIT),
       "tiles_only": timed(mk("pre", pre)),
       "decode_only": timed(mk("dec", dec))}
print(json.dumps(res))
