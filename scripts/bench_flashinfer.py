#!/usr/bin/env python
"""External Blackwell yardstick: flashinfer 0.6.11's trtllm-gen sm100 paged
attention kernels (prebuilt cubins, library code) on exactly the same pools, block tables and
ragged spans as this repo's fused kernel, for configs 2, 3 and 4 (one layer).

flashinfer reads the same [slot][page_tokens][n_kv][d] K and V pools ("NHD", a (K, V) tuple),
one block-table row per span, seq_lens = context_len, and bottom-right aligned causal masking,
which is the reference's semantics (token i of a span sees [0, causal_offset + i],
/root/reference/proj/src/attention.cpp:95-108).  Its outputs are checked against ours before
anything is timed.  Times are CUDA-event medians with a 256 MB L2 flush before every
repetition, on the launching stream.

  python scripts/bench_flashinfer.py [--configs 2,3,4] [--reps 20] [--out profiles/r2_flashinfer.json]
"""
from __future__ import annotations

import argparse
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
from paper_2312_05516_b200.abi import AttentionPlan  # noqa: E402
from paper_2312_05516_b200.workloads import config  # noqa: E402


def timed(fn, reps, flush):
    ts = []
    for _ in range(reps + 3):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts[3:])


def run(cfg: int, reps: int, flush) -> dict:
    import flashinfer

    w = config(cfg)
    q, k, v = gh.device_inputs(w)
    dev = q.device
    d, nh, nkv, chunk = w.head_size, w.n_head, w.n_kv_head, w.chunk
    batch = w.batch()
    n = batch.n_spans
    stream = torch.cuda.current_stream().cuda_stream

    plan = AttentionPlan(w.shape(), batch)
    plan.upload(stream)
    out = torch.empty_like(q)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device=dev)

    def ours():
        plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), stream)

    ours()
    torch.cuda.synchronize()

    # flashinfer descriptors over the same pools
    ql = np.array([int(x) for x in batch.query_len], dtype=np.int64)
    co = np.array([int(x) for x in batch.causal_offset], dtype=np.int64)
    ctx = ql + co
    max_pages = int(max(len(batch.table(i)) for i in range(n)))
    bt = np.zeros((n, max_pages), dtype=np.int32)
    for i in range(n):
        t = batch.table(i)
        bt[i, :len(t)] = t
    k4 = k[: w.pool_elems].view(w.n_slots, chunk, nkv, d)
    v4 = v[: w.pool_elems].view(w.n_slots, chunk, nkv, d)
    q3 = q[: w.q_elems].view(w.total_tokens, nh, d)
    bt_d = torch.from_numpy(bt).to(dev)
    seq_d = torch.from_numpy(ctx.astype(np.int32)).to(dev)
    cq = np.zeros(n + 1, dtype=np.int32)
    cq[1:] = np.cumsum(ql)
    ck = np.zeros(n + 1, dtype=np.int32)
    ck[1:] = np.cumsum(ctx)
    cq_d = torch.from_numpy(cq).to(dev)
    ck_d = torch.from_numpy(ck).to(dev)
    fws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    fout = torch.empty_like(q3)
    scale = 1.0 / w.scale

    def fi_context():
        flashinfer.prefill.trtllm_batch_context_with_kv_cache(
            q3, (k4, v4), fws, bt_d, seq_d, int(ql.max()), int(ctx.max()), scale, 1.0, n, cq_d, ck_d,
            out=fout, kv_layout="NHD", causal=True)

    res = {"config": cfg, "spans": n, "tokens": int(w.total_tokens)}
    fl, by = w.flops_bytes()
    res["algorithmic"] = {"gflop": fl / 1e9, "gbytes": by / 1e9}
    t_ours = timed(ours, reps, flush)
    res["ours_us"] = t_ours
    want = out[: w.q_elems].float().view(w.total_tokens, nh, d)
    try:
        fi_context()
        torch.cuda.synchronize()
        diff = (fout.float() - want).abs().max().item()
        res["fi_context_maxdiff_vs_ours"] = diff
        res["fi_context_us"] = timed(fi_context, reps, flush)
    except Exception as e:  # noqa: BLE001
        res["fi_context_error"] = f"{type(e).__name__}: {e}"[:300]
    # decode spans through the decode kernel (+ prefill spans through the context kernel)
    dec = np.nonzero(ql == 1)[0]
    pre = np.nonzero(ql > 1)[0]
    if len(dec):
        try:
            tok0 = cq[:-1]
            qd = q3[torch.from_numpy(tok0[dec]).to(dev)].contiguous()
            btd = bt_d[torch.from_numpy(dec).to(dev)].contiguous()
            sd = seq_d[torch.from_numpy(dec).to(dev)].contiguous()
            dout = torch.empty_like(qd)

            def fi_decode():
                flashinfer.decode.trtllm_batch_decode_with_kv_cache(
                    qd, (k4, v4), fws, btd, sd, int(ctx[dec].max()), scale, 1.0, out=dout, kv_layout="NHD")

            fi_decode()
            torch.cuda.synchronize()
            res["fi_decode_maxdiff_vs_ours"] = (dout.float() - want[torch.from_numpy(tok0[dec]).to(dev)]).abs().max().item()
            res["fi_decode_us"] = timed(fi_decode, reps, flush)
            if len(pre):
                qp_idx = np.concatenate([np.arange(cq[i], cq[i + 1]) for i in pre])
                qp = q3[torch.from_numpy(qp_idx).to(dev)].contiguous()
                btp = bt_d[torch.from_numpy(pre).to(dev)].contiguous()
                sp = seq_d[torch.from_numpy(pre).to(dev)].contiguous()
                cqp = torch.from_numpy(np.concatenate([[0], np.cumsum(ql[pre])]).astype(np.int32)).to(dev)
                ckp = torch.from_numpy(np.concatenate([[0], np.cumsum(ctx[pre])]).astype(np.int32)).to(dev)
                pout = torch.empty_like(qp)

                def fi_prefill():
                    flashinfer.prefill.trtllm_batch_context_with_kv_cache(
                        qp, (k4, v4), fws, btp, sp, int(ql[pre].max()), int(ctx[pre].max()), scale, 1.0,
                        len(pre), cqp, ckp, out=pout, kv_layout="NHD", causal=True)

                fi_prefill()
                torch.cuda.synchronize()
                res["fi_prefill_maxdiff_vs_ours"] = (pout.float() - want[torch.from_numpy(qp_idx).to(dev)]).abs().max().item()
                res["fi_prefill_us"] = timed(fi_prefill, reps, flush)

                def fi_both():
                    fi_prefill()
                    fi_decode()

                res["fi_prefill_plus_decode_us"] = timed(fi_both, reps, flush)
        except Exception as e:  # noqa: BLE001
            res["fi_decode_error"] = f"{type(e).__name__}: {e}"[:300]
    best = [res[k_] for k_ in ("fi_context_us", "fi_prefill_plus_decode_us") if k_ in res]
    if cfg == 3 and "fi_decode_us" in res:
        best.append(res["fi_decode_us"])
    if best:
        res["fi_best_us"] = min(best)
        res["ours_speedup_vs_fi_best"] = min(best) / t_ours
    res["ours_tflops"] = fl / t_ours / 1e6
    res["ours_gbs"] = by / t_ours / 1e3
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "flashinfer.json"))
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for c in [int(x) for x in a.configs.split(",")]:
        r = run(c, a.reps, flush)
        print(json.dumps(r), flush=True)
        rows.append(r)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    import flashinfer
    with open(a.out, "w") as f:
        json.dump({"flashinfer": flashinfer.__version__, "gpu": torch.cuda.get_device_name(0), "rows": rows}, f,
                  indent=1)


if __name__ == "__main__":
    main()
