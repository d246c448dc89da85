"""Device-side harness for the GPU parity tests: builds a workload's pools and queries in
HBM through the product's own fill kernel, runs a plan, and builds compact CPU-oracle inputs
for sampled spans (the oracle only needs the pages those spans touch)."""
from __future__ import annotations

import numpy as np
import torch

from paper_2312_05516_b200 import abi
from paper_2312_05516_b200.abi import PB_BF16, PB_F32, AttentionPlan, Batch
from paper_2312_05516_b200.workloads import Workload, round_bf16

TORCH_DT = {PB_F32: torch.float32, PB_BF16: torch.bfloat16}


def device_inputs(w: Workload, layer: int = 0, dev: str = "cuda:0"):
    dt = TORCH_DT[w.dtype]
    k = torch.empty(max(1, w.pool_elems), dtype=dt, device=dev)
    v = torch.empty_like(k)
    q = torch.empty(max(1, w.q_elems), dtype=dt, device=dev)
    abi.fill_unit(k.data_ptr(), w.dtype, w.pool_elems, w.seed, w.k_first_draw(layer))
    abi.fill_unit(v.data_ptr(), w.dtype, w.pool_elems, w.seed, w.v_first_draw(layer))
    abi.fill_unit(q.data_ptr(), w.dtype, w.q_elems, w.seed, w.q_first_draw())
    return q, k, v


def run_plan(w: Workload, q, k, v, flags: int = 0, batch: Batch = None, shape=None):
    shape = shape or w.shape()
    batch = batch or w.batch()
    plan = AttentionPlan(shape, batch, flags)
    stream = torch.cuda.current_stream().cuda_stream
    plan.upload(stream)
    out = torch.zeros(max(1, batch.total_tokens * shape.n_head * shape.head_size), dtype=q.dtype,
                      device=q.device)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device=q.device)
    plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), stream)
    torch.cuda.synchronize()
    return out.float().cpu().numpy()[: batch.total_tokens * shape.n_head * shape.head_size], plan


def sampled_oracle_inputs(w: Workload, span_ids, layer: int = 0):
    return w.compact_host_inputs(span_ids, layer)


def gather_out_rows(out: np.ndarray, w: Workload, span_ids) -> np.ndarray:
    rows = out.reshape(w.total_tokens, w.n_head * w.head_size)
    tok = w.span_token_offsets()
    return np.concatenate([rows[tok[i]:tok[i + 1]] for i in span_ids]).reshape(-1)


def bf16_close(got: np.ndarray, ref: np.ndarray, atol: float = 2e-2, rtol: float = 1e-2):
    """North-star bf16 parity: |got - ref| <= 2e-2 + 1e-2 * |ref| elementwise."""
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    bound = atol + rtol * np.abs(ref.astype(np.float64))
    return bool(np.all(err <= bound)), float(err.max(initial=0.0))


def group_oracle(oracle, w: Workload, span_ids, kvh: int, threads: int = 0, block: int = 64, layer: int = 0):
    """CPU oracle restricted to one kv-head group (kv head `kvh` and its query heads, which
    are independent of every other head: src/attention.cpp:90-92), with every span cut into
    token blocks that run on `threads` host threads (each block is a span of its own:
    causal_offset + t0, the table truncated to ceil(context / chunk); results are
    independent of evaluation order).  Returns [tokens of span_ids][g][d]."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    from paper_2312_05516_b200.descriptors import AttnShape

    g = w.n_head // w.n_kv_head
    d = w.head_size
    shape, full, q, keys, values = w.compact_host_inputs(span_ids, layer)
    keys = np.ascontiguousarray(keys.reshape(-1, w.chunk, w.n_kv_head, d)[:, :, kvh, :]).reshape(-1)
    values = np.ascontiguousarray(values.reshape(-1, w.chunk, w.n_kv_head, d)[:, :, kvh, :]).reshape(-1)
    q = np.ascontiguousarray(q.reshape(-1, w.n_head, d)[:, kvh * g:(kvh + 1) * g, :])
    gshape = AttnShape(g, 1, d, w.chunk, shape.n_slots, shape.dtype, shape.scale)
    jobs, t = [], 0
    for i in range(full.n_spans):
        ql, co, table = int(full.query_len[i]), int(full.causal_offset[i]), full.table(i)
        for t0 in range(0, ql, block):
            nt = min(block, ql - t0)
            ctx = co + t0 + nt
            jobs.append((t + t0, nt, co + t0, table[: (ctx + w.chunk - 1) // w.chunk]))
        t += ql
    out = np.zeros_like(q)

    def run(job):
        tok, nt, off, table = job
        b = Batch([nt], [off], [table])
        st, o = oracle.attention(gshape, b, q[tok:tok + nt].reshape(-1), keys, values)
        assert st == 0, st
        out[tok:tok + nt] = o.reshape(nt, g, d)

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1) as ex:
        list(ex.map(run, jobs))
    return out


def group_rows(out: np.ndarray, w: Workload, span_ids, kvh: int) -> np.ndarray:
    """GPU output rows of span_ids restricted to kv head kvh's query heads: [tokens][g][d]."""
    g = w.n_head // w.n_kv_head
    rows = out.reshape(w.total_tokens, w.n_head, w.head_size)
    tok = w.span_token_offsets()
    return np.concatenate([rows[tok[i]:tok[i + 1], kvh * g:(kvh + 1) * g] for i in span_ids])
