#!/usr/bin/env python
"""Diagnostics: per-CTA end times of one launch of the config-4 prefill tiles alone (rank 0 of
an N-way kv-head shard), grouped vs strict-LPT tile queue (PB_PLAN_LPT_ORDER).  Prints the
launch time and the deciles of the CTA end times (us from the first CTA start)."""
import json
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gpu_helpers as gh  # noqa: E402
from paper_2312_05516_b200.abi import PB_PLAN_LPT_ORDER, AttentionPlan  # noqa: E402
from paper_2312_05516_b200.sharding import shard_shape  # noqa: E402
from paper_2312_05516_b200.workloads import PB_BF16, SplitMix64, _build, config  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
base = config(4)
pre = [[(off, ql)] for _, off, ql in base.spans if ql > 1]
w = _build("pre", base.n_head, base.n_kv_head, base.head_size, base.chunk, PB_BF16, 4, pre, SplitMix64(4))
shape = shard_shape(w.shape(), 0, world)
w.n_kv_head, w.n_head = shape.n_kv_head, shape.n_head
q, k, v = gh.device_inputs(w)
st = torch.cuda.current_stream().cuda_stream
out = torch.empty_like(q)
res = {"world": world}
for name, flags in (("grouped", 0), ("lpt", PB_PLAN_LPT_ORDER)):
    plan = AttentionPlan(shape, w.batch(), flags)
    plan.upload(st)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    tr = torch.zeros(148 * 2 * 4, dtype=torch.int64, device="cuda")
    ts = []
    for i in range(8):
        if i == 7:
            plan.set_trace(tr.data_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), st)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    t = tr.cpu().numpy().reshape(148, 2, 4)
    beg = t[:, 0, 2][t[:, 0, 2] > 0]
    end = t[:, 0, 3][t[:, 0, 3] > 0]
    t0 = beg.min()
    e = np.sort((end - t0) / 1e3)
    entry = t[:, 0, 1][t[:, 0, 1] > 0]
    exitt = t[:, 1, 1][t[:, 1, 1] > 0]
    res[name] = {"us": round(statistics.median(ts[3:7]), 1), "start_spread_us": round((beg.max() - t0) / 1e3, 1),
                 "end_deciles_us": [round(float(np.percentile(e, p)), 1) for p in (0, 10, 25, 50, 75, 90, 100)],
                 "entry_us": [round((entry.min() - t0) / 1e3, 1), round((entry.max() - t0) / 1e3, 1)],
                 "exit_us": [round((exitt.min() - t0) / 1e3, 1), round((exitt.max() - t0) / 1e3, 1)]}
print(json.dumps(res))
