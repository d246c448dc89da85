#!/usr/bin/env python
"""Diagnostics (needs a -DPB_TILE_TRACE=1 build): per-tile clock64 timeline of the tile
pipeline in the first 8 CTAs for one config-4 layer.  Prints, per role, the median phase
durations (cycles) and the steady-state tile period, so the critical path of the softmax ->
MMA chain can be read off: softmax {wait S, load+max, exp/pack, store+arrive}, MMA {K wait +
S issue, V wait, P_A wait, P_B wait}."""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import gpu_helpers as gh  # noqa: E402
from paper_2312_05516_b200.abi import AttentionPlan, PB_PLAN_SEPARATE_DECODE  # noqa: E402
from paper_2312_05516_b200.workloads import config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # rank 0 of an N-way kv-head shard
w = config(cfg)
if world > 1:
    from paper_2312_05516_b200.sharding import shard_shape  # noqa: E402
    _sh = shard_shape(w.shape(), 0, world)
    w.n_kv_head, w.n_head = _sh.n_kv_head, _sh.n_head
q, k, v = gh.device_inputs(w)
plan = AttentionPlan(_sh if world > 1 else w.shape(), w.batch(), PB_PLAN_SEPARATE_DECODE)
stream = torch.cuda.current_stream().cuda_stream
plan.upload(stream)
out = torch.empty_like(q)
ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
n = 148 * 2 * 4 + 8 * 6 * 1024 * 8
tr = torch.zeros(n, dtype=torch.int64, device="cuda")
for i in range(4):
    if i == 3:
        plan.set_trace(tr.data_ptr())
    plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), stream)
torch.cuda.synchronize()
t = tr.cpu().numpy()[148 * 2 * 4:].reshape(8, 6, 1024, 8)
res = {}
for role, name in ((0, "softmax_A"), (1, "softmax_B")):
    d = {"wait_S": [], "ld_max": [], "exp": [], "st_arrive": [], "period": []}
    for c in range(8):
        ev = t[c, role]
        ev = ev[ev[:, 0] > 0]
        for i in range(1, len(ev)):
            d["wait_S"].append(ev[i, 1] - ev[i, 0])
            d["ld_max"].append(ev[i, 2] - ev[i, 1])
            d["exp"].append(ev[i, 3] - ev[i, 2])
            d["st_arrive"].append(ev[i, 4] - ev[i, 3])
            d["period"].append(ev[i, 4] - ev[i - 1, 4])
    res[name] = {k: int(statistics.median(v)) for k, v in d.items() if v}
    res[name]["tiles"] = len(d["period"])
    res[name]["mean_period"] = float(np.mean(d["period"]))
d = {"k_wait_s_issue": [], "v_wait": [], "pA_wait": [], "pB_wait": [], "tail": [], "period": []}
for c in range(8):
    ev = t[c, 2]
    ev = ev[ev[:, 0] > 0]
    for i in range(1, len(ev)):
        d["k_wait_s_issue"].append(ev[i, 1] - ev[i, 0])
        d["v_wait"].append(ev[i, 2] - ev[i, 1])
        if ev[i, 3]:
            d["pA_wait"].append(ev[i, 3] - ev[i, 2])
        if ev[i, 4]:
            d["pB_wait"].append(ev[i, 4] - max(ev[i, 3], ev[i, 2]))
        d["tail"].append(ev[i, 5] - max(ev[i, 3], ev[i, 4], ev[i, 2]))
        d["period"].append(ev[i, 5] - ev[i - 1, 5])
res["mma"] = {k: int(statistics.median(v)) for k, v in d.items() if v}
res["mma"]["mean_period"] = float(np.mean(d["period"]))
# one CTA's first 40 softmax-A tiles, raw (relative cycles)
ev = t[0, 0]
ev = ev[ev[:, 0] > 0][:40]
base = ev[0, 0]
res["cta0_A_first"] = [[int(x - base) for x in e[:5]] + [int(e[5]), int(e[6]), int(e[7])] for e in ev]
ev = t[0, 2]
ev = ev[ev[:, 0] > 0][:40]
res["cta0_mma_first"] = [[int(x - base) if x else 0 for x in e[:6]] + [int(e[6]), int(e[7])] for e in ev]
# item boundaries (CTA 0..7): K producer {ticket, item read, q_empty passed, K(0) issued, last
# K issued}; MMA {item read, q_full, k_full(0), S(0) issued}; softmax A {item read, last tile
# done, o_ready, epilogue done}
for role, name, fields in ((3, "prod_item", ["read", "q_empty", "k0_issued", "all_k_issued"]),
                           (4, "mma_item", ["read", "q_full", "k0_full", "s0_issued"]),
                           (5, "softA_item", ["read", "tiles", "o_ready", "tmem_out", "store_half0", "store_half1"])):
    d = {f: [] for f in fields}
    for c in range(8):
        ev = t[c, role]
        ev = ev[ev[:, 0] > 0]
        for e in ev:
            if int(e[7]) < 0:
                continue
            seq = [0, 1, 2, 3, 5, 6, 4] if role == 5 else list(range(len(fields) + 1))
            for i, f in enumerate(fields):
                a, b = seq[i], seq[i + 1]
                if e[b] and e[a]:
                    d[f].append(int(e[b]) - int(e[a]))
    res[name] = {f: int(statistics.median(v)) for f, v in d.items() if v}
    ev = t[0, role]
    ev = ev[ev[:, 0] > 0][:6]
    res[name + "_cta0"] = [[int(x - base) if x else 0 for x in e[:7]] + [int(e[7])] for e in ev]
# per-CTA item timeline (softmax A, first 8 CTAs, us at 1.9 GHz): item, start, tiles done, epilogue done
tl = {}
for c in range(8):
    ev = t[c, 5]
    ev = ev[ev[:, 0] > 0]
    b0 = t[c, 0][t[c, 0][:, 0] > 0]
    if len(b0) == 0:
        continue
    z = int(b0[0, 0])
    tl[c] = [[int(e[7]), round((int(e[1]) - z) / 1900, 1), round((int(e[2]) - z) / 1900, 1),
              round((int(e[4]) - z) / 1900, 1)] for e in ev if int(e[7]) >= 0]
res["timeline"] = tl
print(json.dumps(res))
