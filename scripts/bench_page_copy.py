#!/usr/bin/env python
"""Page movers on their own: pb_kv_gather_pages / pb_kv_scatter_pages (page_copy_kernel, the
device-side replacement of the copy-out gather of /root/reference/proj/src/attention.cpp:259-269
and of the swap staging) over a Llama-2-13B-shaped pool (16-token pages, 10 kv heads, d 128:
40 KiB per page and layer), 40 layers, random Fisher-Yates slot lists.  Reports HBM GB/s
(read + write bytes) against the measured copy peak, CUDA events, inputs larger than L2.
Also the ncu target for the page movers (scripts/gpu_r2b.sh)."""
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_05516_b200 import abi  # noqa: E402

n_layer, page = 40, 16 * 10 * 128 * 2
n_slots = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dev = torch.device("cuda", 0)
pool = torch.empty(n_layer * n_slots * page, dtype=torch.uint8, device=dev)
pool.random_(0, 256)
stage = torch.empty(n_layer * n * page, dtype=torch.uint8, device=dev)
rng = np.random.default_rng(1)
slots = torch.from_numpy(rng.permutation(n_slots)[:n].astype(np.int32)).to(dev)
st = torch.cuda.current_stream().cuda_stream
res = {"layers": n_layer, "page_bytes": page, "pages": n, "bytes_moved_each": n * n_layer * page}
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
for name, fn in (("gather", lambda: abi.gather_pages(pool.data_ptr(), n_slots * page, n_layer, page, slots.data_ptr(),
                                                      n, stage.data_ptr(), 0, st)),
                 ("scatter", lambda: abi.scatter_pages(stage.data_ptr(), n_slots * page, n_layer, page,
                                                        slots.data_ptr(), n, pool.data_ptr(), 0, st))):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = sorted(ts)[len(ts) // 2]
    gbs = 2 * n * n_layer * page / t / 1e9  # read + write
    res[name] = {"us": t * 1e6, "gbs_read_plus_write": gbs, "frac_of_copy_peak": gbs / peaks["hbm_gbs"]}
print(json.dumps(res))
