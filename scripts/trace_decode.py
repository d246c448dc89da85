#!/usr/bin/env python
"""Diagnostics (needs a -DPB_TILE_TRACE=1 build): per-tile clock64 timeline of the tcgen05
decode pipeline (decode_tc_cta.cuh) on a decode-only batch of n spans x ctx cached tokens, one
kv head, GQA-8 (whole-span units).  Prints median phase durations (cycles) per role:
softmax {wait S, reduce+barrier, exp/P^T/arrive, period}, MMA {K wait + S issue, P wait,
V wait, PV issue, period}, K/V producers {stage wait, period}."""
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
from paper_2312_05516_b200.abi import PB_PLAN_NO_SPLIT, AttentionPlan  # noqa: E402
from paper_2312_05516_b200.workloads import PB_BF16, SplitMix64, _build  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
w = _build("dec", 8, 1, 128, 16, PB_BF16, 7, [[(ctx, 1)] for _ in range(n)], SplitMix64(7))
q, k, v = gh.device_inputs(w)
plan = AttentionPlan(w.shape(), w.batch(), PB_PLAN_NO_SPLIT)
st = torch.cuda.current_stream().cuda_stream
plan.upload(st)
out = torch.empty_like(q)
ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
tr = torch.zeros(148 * 2 * 4 + 8 * 6 * 1024 * 8, dtype=torch.int64, device="cuda")
for i in range(4):
    if i == 3:
        plan.set_trace(tr.data_ptr())
    plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), st)
torch.cuda.synchronize()
t = tr.cpu().numpy()[148 * 2 * 4:].reshape(8, 6, 1024, 8)
res = {"n": n, "ctx": ctx}


def med(vals):
    return int(statistics.median(vals)) if vals else None


for role, name, fields in ((0, "softmax", ["wait_S", "reduce", "exp_arrive"]),
                           (0, "softmax_detail", ["wait_S", "reduce", "exp_pstore", "vzero_rescale", "fence"]),
                           (2, "mma", ["k_wait_s_issue", "p_wait", "v_wait", "pv_issue"]),
                           (3, "k_prod", ["stage_wait"]), (4, "v_prod", ["stage_wait"])):
    d = {f: [] for f in fields}
    per = []
    for c in range(8):
        ev = t[c, role]
        ev = ev[ev[:, 0] > 0]
        for i in range(1, len(ev)):
            seq = [0, 1, 2, 4, 5, 6] if name == "softmax_detail" else list(range(len(fields) + 1))
            for fi, f in enumerate(fields):
                a, b = seq[fi], seq[fi + 1]
                if ev[i, b] and ev[i, a]:
                    d[f].append(int(ev[i, b] - ev[i, a]))
            per.append(int(ev[i, 0] - ev[i - 1, 0]))
    res[name] = {f: med(vs) for f, vs in d.items()}
    res[name]["period"] = med(per)
print(json.dumps(res))
