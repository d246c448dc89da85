"""Regenerates tests/golden/* from the UNMODIFIED reference (oracle/_ref/libkvsim_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures are committed so the CPU and GPU test suites never need /root/reference at run
time.  Each fixture records the generator parameters next to the reference's outputs.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2312_05516_b200.workloads import PB_F32, SplitMix64, random_instance  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def attention_golden(ref: Reference) -> None:
    """Acceptance-criterion-2-style instances (proj/tests/acceptance.cpp:100-166 shapes:
    head pairs incl. GQA, head_size 8, page 16|32, 1-4 spans, one long context) run through
    the reference's paged_multi_token_attention; plus single-token and copy-out outputs."""
    rng = SplitMix64(20260814)
    pairs = [(1, 1), (3, 3), (8, 8), (2, 1), (4, 2), (8, 4), (4, 1), (8, 2)]
    cases, outs = [], {}
    for trial in range(40):
        nh, nkv = pairs[rng.next() % 8]
        chunk = 16 if rng.next() % 2 == 0 else 32
        n_spans = 1 + rng.next() % 4
        all_dec = trial % 3 == 2
        w = random_instance(rng, nh, nkv, 8, chunk, PB_F32, n_spans, 1024 if trial % 4 else 2048,
                            all_decode=all_dec, max_q=16)
        shape, batch = w.shape(), w.batch()
        q, k, v = w.host_q(), w.host_pool("k"), w.host_pool("v")
        st, out, _ = ref.attention(shape, batch, q, k, v, mode=0)
        assert st == 0, st
        outs[f"paged_{trial}"] = out
        if all_dec:
            st, single, _ = ref.attention(shape, batch, q, k, v, mode=1)
            assert st == 0
            outs[f"single_{trial}"] = single
        st, cp, gathered = ref.attention(shape, batch, q, k, v, mode=2)
        assert st == 0
        cases.append({"trial": trial, "n_head": nh, "n_kv_head": nkv, "chunk": chunk,
                      "seed": w.seed, "spans": w.spans, "tables": [t.tolist() for t in w.conv_tables],
                      "n_slots": w.n_slots, "pool_first_draw": w.pool_first_draw,
                      "all_decode": all_dec, "copyout_gathered_values": gathered,
                      "copyout_equals_paged": bool(np.array_equal(cp, out))})
    np.savez_compressed(os.path.join(HERE, "attention_ref_outputs.npz"), **outs)
    with open(os.path.join(HERE, "attention_ref_cases.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py::attention_golden",
                   "reference": "proj/src/attention.cpp:73-285 via oracle/_ref",
                   "cases": cases}, f)


def splitmix_golden(ref: Reference) -> None:
    data = {"reference": "proj/src/workload.cpp:30-40; KAT proj/tests/test_workload.cpp:209-214",
            "seed0_first3": ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x06c45d188009454f"],
            "streams": {str(s): [hex(x) for x in ref.splitmix(s, 16)] for s in (0, 1, 2, 3, 4, 42, 20260814)}}
    with open(os.path.join(HERE, "splitmix.json"), "w") as f:
        json.dump(data, f, indent=1)


def model_golden(ref: Reference) -> None:
    rows = {}
    for preset in ("opt-13b", "opt-66b", "llama2-13b", "llama2-70b"):
        for chunk in (1, 16, 32):
            st, tok, ch = ref.model_bytes(preset, chunk)
            rows[f"{preset}/{chunk}"] = [tok, ch]
    with open(os.path.join(HERE, "model_bytes.json"), "w") as f:
        json.dump({"reference": "proj/src/model_config.cpp:29-40 (per-worker chunk bytes)",
                   "kv_token_bytes_chunk_bytes": rows}, f, indent=1)


if __name__ == "__main__":
    r = Reference()
    splitmix_golden(r)
    model_golden(r)
    attention_golden(r)
    print("golden fixtures written to", HERE)
