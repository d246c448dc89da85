#!/usr/bin/env python
"""Straw-man baselines for the multi-token paged kernel.

The paper's kernel microbenchmark: 32 conversations, 8 new query tokens each, past context
swept; compare the generalized multi-token PagedAttention kernel against
  * contiguous-KV "ideal": the same kernel over KV laid out contiguously per conversation
    (what paging costs);
  * copy-out + dense: gather every conversation's pages into a contiguous buffer, then dense
    attention over it (proj/src/attention.cpp:247-285, the reference's CopyOut straw-man);
  * multi-round single-token: one single-token launch per query position (query i attends
    to past + i + 1 tokens), as a decode-only PagedAttention kernel would have to do it;
  * flash_attn varlen (dense, contiguous KV), an external yardstick on the same B200, when the
    package imports.
Shape: OPT-13B attention (40 heads, d = 128, 16-token pages, bf16), pages scattered by a
Fisher-Yates shuffle (proj/tests/acceptance.cpp:143-146).  Times are CUDA-event medians with
an L2 flush (256 MB write) before every repetition.

  python scripts/bench_strawmen.py [--contexts 256,1024,4096] [--reps 20] [--out profiles/strawmen_r1.json]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, AttentionPlan, AttnShape, Batch  # noqa: E402
from paper_2312_05516_b200.workloads import SplitMix64  # noqa: E402

N_HEAD, N_KV, D, CHUNK = 40, 40, 128, 16


def timed(fn, reps, flush):
    ts = []
    for _ in range(reps + 2):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts[2:])


def run_context(past: int, n_conv: int, q_len: int, reps: int, flush) -> dict:
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream().cuda_stream
    ctx = past + q_len
    pages_per = (ctx + CHUNK - 1) // CHUNK
    n_slots = n_conv * pages_per
    rng = SplitMix64(1000 + past)
    perm = list(range(n_slots))
    for i in range(n_slots - 1, 0, -1):  # Fisher-Yates
        j = rng.next() % (i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    scattered = [perm[c * pages_per:(c + 1) * pages_per] for c in range(n_conv)]
    contiguous = [list(range(c * pages_per, (c + 1) * pages_per)) for c in range(n_conv)]
    page_elems = CHUNK * N_KV * D
    k = torch.empty(n_slots * page_elems, dtype=torch.bfloat16, device=dev)
    v = torch.empty_like(k)
    abi.fill_unit(k.data_ptr(), PB_BF16, k.numel(), 7, 0)
    abi.fill_unit(v.data_ptr(), PB_BF16, v.numel(), 7, k.numel())
    tokens = n_conv * q_len
    q = torch.empty(tokens * N_HEAD * D, dtype=torch.bfloat16, device=dev)
    abi.fill_unit(q.data_ptr(), PB_BF16, q.numel(), 8, 0)
    out = torch.empty_like(q)
    shape = AttnShape(N_HEAD, N_KV, D, CHUNK, n_slots, PB_BF16, math.sqrt(D))

    def plan_for(tables, qlen=q_len, off=past, flags=0):
        b = Batch([qlen] * n_conv, [off] * n_conv, tables)
        pl = AttentionPlan(shape, b, flags)
        pl.upload(stream)
        ws = torch.zeros(max(1, pl.workspace_bytes()), dtype=torch.uint8, device=dev)
        return pl, ws

    res = {}
    # 1. the multi-token paged kernel over scattered pages
    pl, ws = plan_for(scattered)
    res["pensieve_paged"] = timed(lambda: pl.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                                 ws.data_ptr(), stream), reps, flush)
    flops = pl.stats()["flops"]
    # 2. contiguous-KV ideal: same kernel, pages of a conversation consecutive
    pc, wc = plan_for(contiguous)
    res["contiguous_ideal"] = timed(lambda: pc.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                                   wc.data_ptr(), stream), reps, flush)
    # 3. copy-out + dense: gather the scattered pages into a contiguous staging pool, then run
    slots = torch.tensor([s for t in scattered for s in t], dtype=torch.int32, device=dev)
    ks = torch.empty_like(k)
    vs = torch.empty_like(v)
    page_bytes = page_elems * 2

    def copyout():
        abi.gather_pages(k.data_ptr(), 0, 1, page_bytes, slots.data_ptr(), n_slots, ks.data_ptr(), 0, stream)
        abi.gather_pages(v.data_ptr(), 0, 1, page_bytes, slots.data_ptr(), n_slots, vs.data_ptr(), 0, stream)
        pc.run(q.data_ptr(), ks.data_ptr(), vs.data_ptr(), out.data_ptr(), wc.data_ptr(), stream)
    res["copyout_dense"] = timed(copyout, reps, flush)
    # 4. multi-round single-token: q_len decode launches, round i sees past + i + 1 tokens
    rounds = []
    q_round = torch.empty(n_conv * N_HEAD * D, dtype=torch.bfloat16, device=dev)
    o_round = torch.empty_like(q_round)
    for i in range(q_len):
        ctx_i = past + i + 1
        tabs = [t[:(ctx_i + CHUNK - 1) // CHUNK] for t in scattered]
        rounds.append(plan_for(tabs, qlen=1, off=past + i, flags=abi.PB_PLAN_SINGLE_TOKEN))

    def multiround():
        for pr, wr in rounds:
            pr.run(q_round.data_ptr(), k.data_ptr(), v.data_ptr(), o_round.data_ptr(), wr.data_ptr(), stream)
    res["multiround_single_token"] = timed(multiround, reps, flush)
    # 5. external yardstick: flash_attn varlen over contiguous (unpaged) KV
    try:
        from flash_attn import flash_attn_varlen_func
        kd = k.view(n_slots * CHUNK, N_KV, D)[: n_conv * pages_per * CHUNK]
        kk = torch.cat([kd[c * pages_per * CHUNK: c * pages_per * CHUNK + ctx] for c in range(n_conv)])
        vd = v.view(n_slots * CHUNK, N_KV, D)[: n_conv * pages_per * CHUNK]
        vv = torch.cat([vd[c * pages_per * CHUNK: c * pages_per * CHUNK + ctx] for c in range(n_conv)])
        qq = q.view(tokens, N_HEAD, D)
        cu_q = torch.arange(0, (n_conv + 1) * q_len, q_len, dtype=torch.int32, device=dev)
        cu_k = torch.arange(0, (n_conv + 1) * ctx, ctx, dtype=torch.int32, device=dev)
        res["flash_attn2_varlen_dense"] = timed(
            lambda: flash_attn_varlen_func(qq, kk, vv, cu_q, cu_k, q_len, ctx, causal=True), reps, flush)
    except Exception as e:  # noqa: BLE001  (yardstick only)
        res["flash_attn2_varlen_dense"] = f"unavailable: {type(e).__name__}: {e}"[:160]
    return {"past": past, "q_len": q_len, "conversations": n_conv, "flops": flops,
            "us": res, "speedup_vs": {k2: (v2 / res["pensieve_paged"] if isinstance(v2, float) else None)
                                       for k2, v2 in res.items() if k2 != "pensieve_paged"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="128,512,1024,2048,4096")
    ap.add_argument("--conversations", type=int, default=32)
    ap.add_argument("--q-len", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "strawmen.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for c in [int(x) for x in args.contexts.split(",")]:
        r = run_context(c, args.conversations, args.q_len, args.reps, flush)
        print(json.dumps(r), flush=True)
        rows.append(r)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"shape": {"n_head": N_HEAD, "n_kv_head": N_KV, "head_size": D, "page_tokens": CHUNK,
                         "dtype": "bf16"}, "gpu": torch.cuda.get_device_name(0), "rows": rows},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
