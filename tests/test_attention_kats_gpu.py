"""The reference's attention known-answer tests (proj/tests/test_attention.cpp) run on the B200
paths: fp32 validation mode (SIMT kernel) at the reference's 1e-5, and bf16 through the
tcgen05 tile and decode kernels at the north-star tolerance.  Inputs are built by hand so
each case pins one rule of paged_multi_token_attention (src/attention.cpp:73-132)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, PB_F32, AttentionPlan, AttnShape, Batch  # noqa: E402

MODES = [(PB_F32, 1e-5), (PB_BF16, 2e-2)]


def _run(torch, shape, batch, q, k_pages, v_pages, flags=0):
    dt = torch.float32 if shape.dtype == PB_F32 else torch.bfloat16
    dq = torch.from_numpy(np.ascontiguousarray(q, np.float32)).to("cuda", dt)
    dk = torch.from_numpy(np.ascontiguousarray(k_pages, np.float32)).to("cuda", dt)
    dv = torch.from_numpy(np.ascontiguousarray(v_pages, np.float32)).to("cuda", dt)
    plan = AttentionPlan(shape, batch, flags)
    stream = torch.cuda.current_stream().cuda_stream
    plan.upload(stream)
    out = torch.zeros_like(dq)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    plan.run(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), out.data_ptr(), ws.data_ptr(), stream)
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


@pytest.mark.parametrize("dtype,tol", MODES)
def test_single_position_returns_its_value_row(cuda, dtype, tol):
    """test_attention.cpp:119-144: one query over one cached position returns that V row
    (softmax of one element), head h reading kv head h / group."""
    torch = cuda
    n_head, n_kv, d, chunk = 8, 2, 128, 16
    shape = AttnShape(n_head, n_kv, d, chunk, 4, dtype, math.sqrt(d))
    rng = np.random.default_rng(1)
    k = rng.uniform(-1, 1, (4, chunk, n_kv, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (4, chunk, n_kv, d)).astype(np.float32)
    q = rng.uniform(-1, 1, (1, n_head, d)).astype(np.float32)
    out = _run(torch, shape, Batch([1], [0], [[2]]), q, k, v).reshape(n_head, d)
    for h in range(n_head):
        want = v[2, 0, h // (n_head // n_kv)]
        if dtype == PB_BF16:
            want = torch.from_numpy(want).to(torch.bfloat16).float().numpy()
        assert np.max(np.abs(out[h] - want)) <= tol


@pytest.mark.parametrize("dtype,tol", MODES)
def test_uniform_keys_average_allowed_values(cuda, dtype, tol):
    """test_attention.cpp:199-221: with every key equal, each query's output is the mean of the
    V rows it may see (causal: position <= causal_offset + i)."""
    torch = cuda
    n_head, n_kv, d, chunk = 4, 1, 64, 16
    off, ql = 37, 20
    ctx = off + ql
    pages = (ctx + chunk - 1) // chunk
    perm = [5, 1, 7, 3][:pages]
    shape = AttnShape(n_head, n_kv, d, chunk, 8, dtype, math.sqrt(d))
    k = np.zeros((8, chunk, n_kv, d), np.float32)
    k[:] = 0.25
    vals = np.arange(ctx, dtype=np.float32) / ctx  # exact in bf16? keep a per-position level
    if dtype == PB_BF16:
        vals = torch.from_numpy(vals).to(torch.bfloat16).float().numpy()
    v = np.zeros((8, chunk, n_kv, d), np.float32)
    for pos in range(ctx):
        v[perm[pos // chunk], pos % chunk, 0, :] = vals[pos]
    q = np.random.default_rng(2).uniform(-1, 1, (ql, n_head, d)).astype(np.float32)
    out = _run(torch, shape, Batch([ql], [off], [perm]), q, k, v).reshape(ql, n_head, d)
    for i in range(ql):
        want = vals[: off + i + 1].mean()
        assert np.max(np.abs(out[i] - want)) <= tol + (1e-2 * abs(want) if dtype == PB_BF16 else 0)


@pytest.mark.parametrize("dtype,tol", MODES)
def test_huge_scale_gives_uniform_average(cuda, dtype, tol):
    """test_attention.cpp:223-249: score = dot / scale, so scale 1e6 flattens the softmax to a
    uniform average of the visible values (1e-3 in the reference)."""
    torch = cuda
    n_head, n_kv, d, chunk = 8, 8, 128, 16
    ctx = 150
    shape = AttnShape(n_head, n_kv, d, chunk, 12, dtype, 1e6)
    rng = np.random.default_rng(3)
    k = rng.uniform(-1, 1, (12, chunk, n_kv, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (12, chunk, n_kv, d)).astype(np.float32)
    if dtype == PB_BF16:
        v = torch.from_numpy(v).to(torch.bfloat16).float().numpy()
    table = [11, 0, 5, 3, 9, 2, 7, 1, 4, 10]
    q = rng.uniform(-1, 1, (1, n_head, d)).astype(np.float32)
    out = _run(torch, shape, Batch([1], [ctx - 1], [table]), q, k, v).reshape(n_head, d)
    rows = np.stack([v[table[p // chunk], p % chunk] for p in range(ctx)])  # [ctx][n_kv][d]
    want = rows.mean(axis=0)
    assert np.max(np.abs(out - want)) <= max(1e-3, tol)


@pytest.mark.parametrize("dtype,tol", [(PB_F32, 1e-6), (PB_BF16, 2e-2)])
def test_single_token_path_equals_multi_token_path(cuda, dtype, tol):
    """test_attention.cpp:251-303: decode batches through the single-token contract
    (PB_PLAN_SINGLE_TOKEN) equal the general path; here also the tcgen05 decode kernel against
    the SIMT kernel (PB_PLAN_FORCE_SIMT)."""
    torch = cuda
    rng = np.random.default_rng(4)
    n_head, n_kv, d, chunk = 16, 4, 128, 16
    n_slots = 256
    shape = AttnShape(n_head, n_kv, d, chunk, n_slots, dtype, math.sqrt(d))
    k = rng.uniform(-1, 1, (n_slots, chunk, n_kv, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (n_slots, chunk, n_kv, d)).astype(np.float32)
    for trial in range(5):
        n = 1 + int(rng.integers(32))
        ctxs = rng.integers(1, 1025, n)
        perm = rng.permutation(n_slots)
        tables, used = [], 0
        for c in ctxs:
            p = (int(c) + chunk - 1) // chunk
            tables.append(perm[used % n_slots: used % n_slots + p] if used % n_slots + p <= n_slots else perm[:p])
            used += p
        b = Batch([1] * n, [int(c) - 1 for c in ctxs], tables)
        q = rng.uniform(-1, 1, (n, n_head, d)).astype(np.float32)
        a = _run(torch, shape, b, q, k, v)
        s = _run(torch, shape, b, q, k, v, flags=abi.PB_PLAN_SINGLE_TOKEN)
        f = _run(torch, shape, b, q, k, v, flags=abi.PB_PLAN_FORCE_SIMT)
        assert np.array_equal(a, s)
        assert np.max(np.abs(a - f)) <= tol
