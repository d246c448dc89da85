"""GPU bring-up probe: runs one named attention case through the C-ABI and prints the max
error against the CPU oracle.  Each case runs in its own process under `timeout` (see
scripts/gpu_check.sh) so a hung kernel cannot take the others down."""
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gpu_helpers as gh  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16  # noqa: E402
from paper_2312_05516_b200.workloads import SplitMix64, _build, config  # noqa: E402

CASES = {
    # name: (n_head, n_kv, d, convs[[(off, q)]])
    "p1": (1, 1, 128, [[(0, 128)]]),
    "p2": (1, 1, 128, [[(128, 128)]]),
    "p3": (1, 1, 128, [[(0, 37)]]),
    "p4": (4, 1, 128, [[(300, 50)]]),
    "p5": (8, 1, 128, [[(1000, 200)], [(0, 3)]]),
    "p6": (2, 2, 64, [[(77, 130)]]),
    "d1": (1, 1, 128, [[(10, 1)]]),
    "d2": (4, 1, 128, [[(2000, 1)], [(5, 1)]]),
    "d3": (8, 1, 128, [[(4095, 1)], [(1030, 1)], [(0, 1)]]),
    "d4": (4, 4, 64, [[(700, 1)]]),
    "mix": (8, 2, 128, [[(500, 1)], [(100, 300)], [(3000, 1)], [(0, 17)]]),
}


def run(name):
    torch.cuda.set_device(0)
    if name.startswith("cfg"):
        w = config(int(name[3:]))
        ids = [i for i in range(len(w.spans)) if w.flops_bytes([i])[0] < 3e9][:6]
    else:
        nh, nkv, d, convs = CASES[name]
        w = _build(name, nh, nkv, d, 16, PB_BF16, 5, convs, SplitMix64(5))
        ids = list(range(len(w.spans)))
    q, k, v = gh.device_inputs(w)
    flags = int(os.environ.get("PB_FLAGS", "0"))
    t0 = time.time()
    got, plan = gh.run_plan(w, q, k, v, flags=flags)
    dt = time.time() - t0
    shape, batch, hq, hk, hv = w.compact_host_inputs(ids)
    st, want = Oracle().attention(shape, batch, hq, hk, hv)
    g = gh.gather_out_rows(got, w, ids)
    err = np.abs(g.astype(np.float64) - want)
    ok, _ = gh.bf16_close(g, want)
    row = w.n_head * w.head_size
    bad_rows = np.unique(np.nonzero(err > 2e-2 + 1e-2 * np.abs(want))[0] // row)
    print(f"{name}: ok={ok} max_err={err.max():.3e} nan={int(np.isnan(g).sum())} "
          f"bad_token_rows={bad_rows[:10].tolist()} n_bad={len(bad_rows)} stats={plan.stats()} t={dt:.2f}s",
          flush=True)


if __name__ == "__main__":
    run(sys.argv[1])
