#!/usr/bin/env python
"""Single-GPU emulation of the KV-head-sharded multi-GPU run.

Every rank of an N-way shard runs the same spans and block tables over n_kv/N heads, with no
collective on the attention path, so the job time at N GPUs is one rank's time.  This times
rank 0's shard of config 4 (Llama-2-70B, 8 kv heads) for N = 1, 2, 4, 8 on one B200 and
prints the implied aggregate TFLOP/s and strong-scaling efficiency.  It is a prediction; the
measured multi-GPU numbers come from `torchrun ... bench.py --gpus N`.
"""
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

n_layer = int(os.environ.get("LAYERS", "16"))
w = config(4)
batch = w.batch()
fl, by = w.flops_bytes()
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
rows = []
base = None
for world in [int(x) for x in os.environ.get("WORLDS", "1,2,4,8").split(",")]:
    shape = shard_shape(w.shape(), 0, world)
    pool = w.n_slots * w.chunk * shape.n_kv_head * w.head_size
    ks = [torch.empty(pool, dtype=torch.bfloat16, device=dev) for _ in range(n_layer)]
    vs = [torch.empty(pool, dtype=torch.bfloat16, device=dev) for _ in range(n_layer)]
    for l in range(n_layer):
        abi.fill_unit(ks[l].data_ptr(), PB_BF16, pool, 11, 2 * l * pool)
        abi.fill_unit(vs[l].data_ptr(), PB_BF16, pool, 11, (2 * l + 1) * pool)
    q = torch.empty(w.total_tokens * shape.n_head * w.head_size, dtype=torch.bfloat16, device=dev)
    abi.fill_unit(q.data_ptr(), PB_BF16, q.numel(), 12, 0)
    out = torch.empty_like(q)
    plan = AttentionPlan(shape, batch)
    plan.upload(stream.cuda_stream)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device=dev)
    # the layer loop as one graph launch (pb_attn_run_layers), as bench.py runs it
    args = ([q.data_ptr()] * n_layer, [x.data_ptr() for x in ks], [x.data_ptr() for x in vs],
            [out.data_ptr()] * n_layer, ws.data_ptr(), stream.cuda_stream)
    for _ in range(3):
        plan.run_layers(*args)
    times = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        plan.run_layers(*args)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / n_layer)
    ms = statistics.median(times)
    tflops = fl / (ms / 1e3) / 1e12  # whole-job work / one rank's time
    base = base or tflops
    rows.append({"gpus": world, "ms_per_layer_per_rank": ms, "job_tflops": tflops,
                 "efficiency_vs_1": tflops / base / world, "items": plan.stats()["prefill_tiles"],
                 "decode_units": plan.stats()["decode_units"]})
    del ks, vs
    torch.cuda.empty_cache()
print(json.dumps({"workload": w.name, "layers": n_layer, "rows": rows}))
