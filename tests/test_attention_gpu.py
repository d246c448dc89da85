"""GPU parity of the fused ragged paged attention against the CPU oracle (pinned to the
reference in tests/test_oracle.py).

Tolerances (BASELINE.json north_star): fp32 validation mode 1e-5 absolute; bf16 mode
|gpu - oracle| <= 2e-2 + 1e-2*|oracle| elementwise, with the oracle fed the same
bf16-rounded inputs widened to fp32.  Full-size configs are checked on sampled spans (the
spans are independent units) plus size-independent properties.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, PB_F32, AttnShape, AttentionPlan, Batch  # noqa: E402
from paper_2312_05516_b200.workloads import (SplitMix64, Workload, _build, config,  # noqa: E402
                                             random_instance, unit_draws)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gh(cuda):
    import gpu_helpers as gh
    return gh


def test_fill_kernel_bit_exact(gh, cuda):
    torch = cuda
    for dt, tdt in ((PB_F32, torch.float32), (PB_BF16, torch.bfloat16)):
        x = torch.empty(100003, dtype=tdt, device="cuda")
        abi.fill_unit(x.data_ptr(), dt, x.numel(), 20260814, 777)
        want = unit_draws(20260814, 777, x.numel())
        got = x.float().cpu().numpy()
        if dt == PB_BF16:
            from paper_2312_05516_b200.workloads import round_bf16
            want = round_bf16(want)
        assert np.array_equal(got, want)


def test_fp32_golden_reference_outputs(gh):
    """One-shot host API (pb_paged_multi_token_attention / pb_single_token_attention) in the
    fp32 validation mode vs the reference's recorded outputs: <= 1e-5."""
    cases = json.load(open(os.path.join(GOLDEN, "attention_ref_cases.json")))["cases"]
    outs = np.load(os.path.join(GOLDEN, "attention_ref_outputs.npz"))
    worst = 0.0
    for c in cases:
        w = Workload("golden", c["n_head"], c["n_kv_head"], 8, c["chunk"], PB_F32, c["seed"],
                     [tuple(s) for s in c["spans"]], [np.array(t, np.int32) for t in c["tables"]],
                     c["n_slots"], c["pool_first_draw"])
        shape, batch = w.shape(), w.batch()
        q, k, v = w.host_q(), w.host_pool("k"), w.host_pool("v")
        got = abi.paged_multi_token_attention(shape, batch, q, k, v)
        err = float(np.max(np.abs(got - outs[f"paged_{c['trial']}"])))
        worst = max(worst, err)
        assert err <= 1e-5, (c["trial"], err)
        if c["all_decode"]:
            single = abi.single_token_attention(shape, batch, q, k, v)
            assert np.max(np.abs(single - outs[f"single_{c['trial']}"])) <= 1e-5


def test_fp32_cfg1_device_path(gh, oracle):
    w = config(1)
    q, k, v = gh.device_inputs(w)
    got, plan = gh.run_plan(w, q, k, v)
    st, want = oracle.attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
    assert st == 0
    assert np.max(np.abs(got - want)) <= 1e-5


@pytest.mark.parametrize("n_head,n_kv,d", [(8, 8, 128), (8, 2, 128), (16, 2, 128), (4, 4, 64), (8, 1, 64)])
@pytest.mark.parametrize("flags", [0, abi.PB_PLAN_FORCE_SIMT])
def test_bf16_random_ragged_batches(gh, oracle, n_head, n_kv, d, flags):
    rng = SplitMix64(1000 + n_head * 10 + n_kv + d)
    for trial in range(3):
        w = random_instance(rng, n_head, n_kv, d, 16, PB_BF16, 1 + rng.next() % 6, 1500,
                            all_decode=(trial == 2), max_q=300)
        q, k, v = gh.device_inputs(w)
        got, plan = gh.run_plan(w, q, k, v, flags=flags)
        st, want = oracle.attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
        assert st == 0
        ok, err = gh.bf16_close(got, want)
        assert ok, (trial, err, plan.stats())


@pytest.mark.parametrize("n_head,n_kv,d", [(16, 1, 128), (48, 3, 128), (6, 2, 128), (10, 2, 128), (32, 1, 128),
                                          (12, 4, 64)])
def test_bf16_uncommon_group_sizes(gh, oracle, n_head, n_kv, d):
    """GQA groups outside the configs: 16 (the decode kernel's widest N), non-powers of two
    (3, 5: the tile packs 126 / 125 of 128 rows, decode pads N), and 32 (beyond the tensor-core
    decode path) -- every head must still read kv head h / group (src/attention.cpp:92)."""
    rng = SplitMix64(7000 + n_head * 10 + n_kv + d)
    for trial in range(3):
        w = random_instance(rng, n_head, n_kv, d, 16, PB_BF16, 1 + rng.next() % 6, 1500,
                            all_decode=(trial == 2), max_q=300)
        q, k, v = gh.device_inputs(w)
        got, plan = gh.run_plan(w, q, k, v)
        st, want = oracle.attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
        assert st == 0
        ok, err = gh.bf16_close(got, want)
        assert ok, (trial, err, plan.stats())


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_bf16_configs_sampled_spans(gh, oracle, cfg):
    """Full-size config run on the GPU; oracle on a sample of spans (longest prefill, longest
    decode, shortest, and a few others)."""
    w = config(cfg)
    q, k, v = gh.device_inputs(w)
    got, plan = gh.run_plan(w, q, k, v)
    spans = w.spans
    cheap = [i for i in range(len(spans)) if w.flops_bytes([i])[0] < 4e9]  # oracle ~10 s max
    by_ctx = sorted(cheap, key=lambda i: spans[i][1] + spans[i][2])
    prefill = [i for i in cheap if spans[i][2] > 1]
    sample = {by_ctx[0], by_ctx[-1], by_ctx[len(by_ctx) // 2]}
    if prefill:
        sample.add(max(prefill, key=lambda i: spans[i][2]))
        sample.add(min(prefill, key=lambda i: spans[i][2]))
    sample = sorted(sample)
    shape, batch, hq, hk, hv = gh.sampled_oracle_inputs(w, sample)
    st, want = oracle.attention(shape, batch, hq, hk, hv)
    assert st == 0
    ok, err = gh.bf16_close(gh.gather_out_rows(got, w, sample), want)
    assert ok, err
    assert np.all(np.isfinite(got))


def test_rows_sum_to_one_all_ones_values(gh, cuda):
    """Size-independent property at full size (cfg 3): with V == 1 every output is 1."""
    torch = cuda
    w = config(3)
    q, k, v = gh.device_inputs(w)
    v.fill_(1.0)
    got, _ = gh.run_plan(w, q, k, v)
    assert np.max(np.abs(got - 1.0)) <= 1e-2


def test_permuting_slots_bit_identical(gh, cuda):
    """proj/tests/test_attention.cpp:407-432 on the GPU: relocating pages and remapping the
    block tables leaves outputs bit-identical."""
    torch = cuda
    rng = SplitMix64(29)
    w = random_instance(rng, 8, 2, 128, 16, PB_BF16, 5, 700, max_q=200)
    q, k, v = gh.device_inputs(w)
    base, _ = gh.run_plan(w, q, k, v)
    n = w.n_slots
    page = w.chunk * w.row_elems
    perm = torch.tensor([(s + 1) % n for s in range(n)], device="cuda")
    k2 = torch.empty_like(k).view(n, page)
    v2 = torch.empty_like(v).view(n, page)
    k2[perm] = k.view(n, page)
    v2[perm] = v.view(n, page)
    b = w.batch()
    b2 = Batch(b.query_len, b.causal_offset, [(b.table(i) + 1) % n for i in range(b.n_spans)])
    moved, _ = gh.run_plan(w, q, k2.view(-1), v2.view(-1), batch=b2)
    assert np.array_equal(moved, base)


def test_causal_sentinel_on_gpu(gh, cuda):
    """proj/tests/test_attention.cpp:146-179: a sentinel at position p changes only tokens
    that may see it; earlier tokens stay bit-identical."""
    torch = cuda
    rng = SplitMix64(2)
    w = random_instance(rng, 8, 8, 128, 16, PB_BF16, 1, 400, max_q=160)
    q, k, v = gh.device_inputs(w)
    b = w.batch()
    base, _ = gh.run_plan(w, q, k, v)
    ql, off = int(b.query_len[0]), int(b.causal_offset[0])
    p = off + ql - 1  # visible only to the last token
    slot = int(b.table(0)[p // 16])
    row = (slot * 16 + p % 16) * w.row_elems
    k[row:row + w.row_elems] = 5.0
    v[row:row + w.row_elems] = -7.0
    after, _ = gh.run_plan(w, q, k, v)
    stride = w.n_head * w.head_size
    assert np.array_equal(base[: (ql - 1) * stride], after[: (ql - 1) * stride])
    assert np.abs(base[(ql - 1) * stride:] - after[(ql - 1) * stride:]).sum() > 0


def test_gqa_duplicated_kv_equals_mha_on_gpu(gh, cuda):
    """proj/tests/test_attention.cpp:358-397: duplicated kv heads == grouped heads."""
    torch = cuda
    rng = SplitMix64(17)
    w = random_instance(rng, 8, 2, 128, 16, PB_BF16, 4, 600, max_q=150)
    q, k, v = gh.device_inputs(w)
    grouped, _ = gh.run_plan(w, q, k, v)
    n = w.n_slots * w.chunk
    k4 = k.view(n, 2, 1, 128).expand(n, 2, 4, 128).reshape(-1).contiguous()
    v4 = v.view(n, 2, 1, 128).expand(n, 2, 4, 128).reshape(-1).contiguous()
    mha_shape = AttnShape(8, 8, 128, 16, w.n_slots, PB_BF16, w.scale)
    full, _ = gh.run_plan(w, q, k4, v4, shape=mha_shape)
    ok, err = gh.bf16_close(full, grouped, atol=1e-3, rtol=1e-3)
    assert ok, err


@pytest.mark.parametrize("n_kv", [10, 1])
def test_split_decode_matches_unsplit(gh, n_kv):
    """Few (span, kv head) pairs with long contexts: the plan splits them across CTAs and
    merges the partials; the result matches the unsplit run (and the oracle, elsewhere)."""
    rng = SplitMix64(60 + n_kv)
    w = random_instance(rng, 4 * n_kv, n_kv, 128, 16, PB_BF16, 12, 6000, all_decode=True)
    q, k, v = gh.device_inputs(w)
    a, pa = gh.run_plan(w, q, k, v)
    b, pb_ = gh.run_plan(w, q, k, v, flags=abi.PB_PLAN_NO_SPLIT)
    assert pa.stats()["split_spans"] > 0 and pb_.stats()["split_spans"] == 0
    ok, err = gh.bf16_close(a, b, atol=1e-2, rtol=1e-2)
    assert ok, err


def test_plan_reused_across_layers(gh):
    """One plan, several layers' pools: each layer matches its own oracle."""
    w = config(1)
    w.n_layer = 3
    for layer in (1, 2):
        q, k, v = gh.device_inputs(w, layer=layer)
        got, _ = gh.run_plan(w, q, k, v)
        from oracle.oracle import Oracle
        st, want = Oracle().attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k", layer),
                                      w.host_pool("v", layer))
        assert np.max(np.abs(got - want)) <= 1e-5


def test_check_numerics_flag(gh, cuda):
    torch = cuda
    w = config(1)
    q, k, v = gh.device_inputs(w)
    plan = AttentionPlan(w.shape(), w.batch())
    plan.upload()
    flag = torch.full((1,), 7, dtype=torch.int32, device="cuda")
    plan.check_numerics(q.data_ptr(), k.data_ptr(), flag.data_ptr())
    assert int(flag.item()) == 0
    q[5] = float("nan")
    plan.check_numerics(q.data_ptr(), k.data_ptr(), flag.data_ptr())
    assert int(flag.item()) == abi.NumericError.code


def test_single_token_api_rejects_long_spans(gh):
    s = AttnShape(1, 1, 4, 8, 1, PB_F32, 2.0)
    b = Batch([2], [0], [[0]])
    q = np.full(8, 0.5, np.float32)
    kv = np.zeros(32, np.float32)
    with pytest.raises(abi.DimensionMismatch):
        abi.single_token_attention(s, b, q, kv, kv)
    abi.paged_multi_token_attention(s, b, q, kv, kv)


def test_bf16_one_shot_equals_device_path(gh):
    rng = SplitMix64(77)
    w = random_instance(rng, 8, 4, 128, 16, PB_BF16, 3, 500, max_q=64)
    q, k, v = gh.device_inputs(w)
    dev, _ = gh.run_plan(w, q, k, v)
    host = abi.paged_multi_token_attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("n_head,n_kv,all_decode", [(8, 1, False), (8, 2, True), (8, 8, False), (16, 2, False)])
def test_stale_rows_past_context_cannot_poison(gh, cuda, n_head, n_kv, all_decode):
    """Rows of a span's last page past its context are never read by the reference
    (proj/src/attention.cpp:95,119); on the GPU they may hold anything (lazy reclamation,
    never-written pool memory).  Filling them with NaN must leave every output bit-identical."""
    torch = cuda
    rng = SplitMix64(41 + n_head + n_kv)
    w = random_instance(rng, n_head, n_kv, 128, 16, PB_BF16, 12, 900, all_decode=all_decode, max_q=140)
    q, k, v = gh.device_inputs(w)
    base, _ = gh.run_plan(w, q, k, v)
    assert np.isfinite(base).all()
    b = w.batch()
    used = {}  # slot -> rows some span reads
    for i in range(b.n_spans):
        ctx = int(b.context_len[i])
        for pidx, slot in enumerate(b.table(i)):
            used[int(slot)] = max(used.get(int(slot), 0), min(16, ctx - 16 * pidx))
    rows = w.row_elems
    poisoned = 0
    for slot, n in used.items():
        if n < 16:
            a, e = (slot * 16 + n) * rows, (slot + 1) * 16 * rows
            k[a:e] = float("nan")
            v[a:e] = float("nan")
            poisoned += 16 - n
    assert poisoned > 0
    after, _ = gh.run_plan(w, q, k, v)
    assert np.array_equal(after, base)


@pytest.mark.parametrize("cfg", [2, 4])
def test_fused_launch_equals_separate_decode_launch(gh, cfg):
    """The fused launch (decode units in the tile kernel's work list) and the two-launch
    schedule run the same arithmetic per unit: outputs are bit-identical."""
    w = config(cfg)
    q, k, v = gh.device_inputs(w)
    fused, pf = gh.run_plan(w, q, k, v)
    sep, ps = gh.run_plan(w, q, k, v, flags=abi.PB_PLAN_SEPARATE_DECODE)
    assert pf.stats()["decode_units"] == ps.stats()["decode_units"] > 0
    assert np.array_equal(fused, sep)


def test_layers_host_pipeline_matches_per_layer_runs(gh, cuda):
    """pb_attn_run_layers_host (host q / out, copies overlapped with compute) gives the same
    bits as one pb_attn_run per layer on device buffers."""
    torch = cuda
    rng = SplitMix64(77)
    w = random_instance(rng, 16, 2, 128, 16, PB_BF16, 6, 900, max_q=120)
    n_layer = 3
    qs, ks, vs = [], [], []
    for l in range(n_layer):
        q, k, v = gh.device_inputs(w, layer=l)
        qs.append(q * (1.0 + 0.25 * l))  # a different q per layer
        ks.append(k)
        vs.append(v)
    want = [gh.run_plan(w, qs[l], ks[l], vs[l])[0] for l in range(n_layer)]
    plan = AttentionPlan(w.shape(), w.batch())
    stream = torch.cuda.current_stream().cuda_stream
    plan.upload(stream)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    stage = torch.empty(plan.stage_bytes(), dtype=torch.uint8, device="cuda")
    q_host = [q.cpu().pin_memory() for q in qs]
    out_host = [torch.empty_like(q_host[0]).pin_memory() for _ in range(n_layer)]
    plan.run_layers_host([t.data_ptr() for t in q_host], [t.data_ptr() for t in out_host],
                         [t.data_ptr() for t in ks], [t.data_ptr() for t in vs], stage.data_ptr(),
                         ws.data_ptr(), stream)
    torch.cuda.synchronize()
    n = w.total_tokens * w.n_head * w.head_size
    for l in range(n_layer):
        assert np.array_equal(out_host[l].float().numpy()[:n], want[l])


def _append_reference(torch, w, k_new, v_new, k_pages, v_pages):
    """pb_kv_append (the stand-alone qkv_project write loop) for the batch's new tokens."""
    b = w.batch()
    shape = w.shape()
    n_rows = np.ascontiguousarray(b.query_len, dtype=np.int64)
    row_start = np.ascontiguousarray(np.concatenate([[0], np.cumsum(n_rows)[:-1]]), dtype=np.int64)
    start = np.ascontiguousarray(b.causal_offset, dtype=np.int64)
    bt = np.ascontiguousarray(b.bt, dtype=np.int32)
    bt_off = np.ascontiguousarray(b.bt_off, dtype=np.int64)
    dev = [torch.from_numpy(a).cuda() for a in (row_start, n_rows, start, bt, bt_off)]
    p = lambda a: a.ctypes.data  # noqa: E731
    abi.check(abi.lib.pb_kv_append(abi.ctypes.byref(shape), b.n_spans, p(row_start), p(n_rows), p(start), p(bt),
                                   p(bt_off), *[d.data_ptr() for d in dev], k_new.data_ptr(), v_new.data_ptr(),
                                   k_pages.data_ptr(), v_pages.data_ptr(), None))


@pytest.mark.parametrize("case", ["fused_gqa8", "decode_only", "prefill_only", "d64_fallback", "fp32_fallback"])
def test_fused_append_equals_append_then_attention(gh, cuda, case):
    """pb_attn_run_append (new K/V rows written inside the attention launch, grid barrier
    before any page read) == pb_kv_append + pb_attn_run: same pages, same outputs, bit for bit."""
    torch = cuda
    rng = SplitMix64(300 + len(case))
    if case == "fused_gqa8":
        w = random_instance(rng, 16, 2, 128, 16, PB_BF16, 40, 1500, max_q=200)
    elif case == "decode_only":
        w = random_instance(rng, 16, 2, 128, 16, PB_BF16, 60, 2000, all_decode=True)
    elif case == "prefill_only":
        w = random_instance(rng, 8, 8, 128, 16, PB_BF16, 5, 600, max_q=600)
        b = w.batch()
        assert min(b.query_len) >= 1
    elif case == "d64_fallback":
        w = random_instance(rng, 8, 2, 64, 16, PB_BF16, 12, 700, max_q=90)
    else:
        w = random_instance(rng, 8, 2, 64, 16, PB_F32, 6, 300, max_q=40)
    q, k, v = gh.device_inputs(w)
    dt = q.dtype
    row = w.n_kv_head * w.head_size
    k_new = torch.empty(w.total_tokens * row, dtype=dt, device="cuda")
    v_new = torch.empty_like(k_new)
    abi.fill_unit(k_new.data_ptr(), w.dtype, k_new.numel(), 991, 0)
    abi.fill_unit(v_new.data_ptr(), w.dtype, v_new.numel(), 992, 0)
    k1, v1 = k.clone(), v.clone()
    _append_reference(torch, w, k_new, v_new, k1, v1)
    want, _ = gh.run_plan(w, q, k1, v1)
    plan = AttentionPlan(w.shape(), w.batch())
    stream = torch.cuda.current_stream().cuda_stream
    plan.upload(stream)
    out = torch.zeros_like(q)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    k2, v2 = k.clone(), v.clone()
    for _ in range(2):  # the grid barrier re-arms itself across launches
        plan.run_append(q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), k2.data_ptr(), v2.data_ptr(),
                        out.data_ptr(), ws.data_ptr(), stream)
    torch.cuda.synchronize()
    assert torch.equal(k1, k2) and torch.equal(v1, v2)
    n = w.total_tokens * w.n_head * w.head_size
    assert np.array_equal(out.float().cpu().numpy()[:n], want)


@pytest.mark.parametrize("chunk", [8, 32, 64, 128])
def test_bf16_page_sizes(gh, oracle, chunk):
    """Page sizes other than 16 (the reference's chunk_size is a parameter): 8..64 run on the
    tcgen05 tile and decode paths, 128 on the SIMT path; all within the bf16 tolerance."""
    rng = SplitMix64(500 + chunk)
    for trial in range(2):
        w = random_instance(rng, 16, 4, 128, chunk, PB_BF16, 10, 1300, all_decode=(trial == 1), max_q=150)
        q, k, v = gh.device_inputs(w)
        got, plan = gh.run_plan(w, q, k, v)
        st, want = oracle.attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
        assert st == 0
        ok, err = gh.bf16_close(got, want)
        assert ok, (chunk, trial, err, plan.stats())


@pytest.mark.parametrize("n_head,n_kv", [(8, 8), (16, 4), (32, 4), (16, 2)])
def test_fuzz_conversations_with_prefix_drops(gh, oracle, n_head, n_kv):
    """Random multi-turn shapes as the planner emits them: per conversation a dropped-prefix
    recompute span (0, a) plus the returning span (b, c) over the same pages, single decode
    tokens, plain prompts and zero-length spans, all in one ragged batch (one launch)."""
    for trial in range(6):
        rng = SplitMix64(7000 + 100 * n_head + 10 * n_kv + trial)
        convs = []
        for c in range(1 + rng.next() % 14):
            kind = rng.next() % 5
            past = rng.next() % 1800
            if kind == 0:    # dropped prefix recomputed + the turn's new tokens
                a = 1 + rng.next() % 300
                b = a + rng.next() % 400
                convs.append([(0, a), (b, 1 + rng.next() % 200)])
            elif kind == 1:  # decode token
                convs.append([(past, 1)])
            elif kind == 2:  # prompt over cached history
                convs.append([(past, 2 + rng.next() % 250)])
            elif kind == 3:  # zero-length span next to a real one
                convs.append([(past, 0), (past, 1 + rng.next() % 3)])
            else:            # fresh prompt
                convs.append([(0, 1 + rng.next() % 400)])
        w = _build("fuzz", n_head, n_kv, 128, 16, PB_BF16, rng.seed, convs, rng)
        q, k, v = gh.device_inputs(w)
        got, plan = gh.run_plan(w, q, k, v)
        st, want = oracle.attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
        assert st == 0
        ok, err = gh.bf16_close(got, want)
        assert ok, (trial, err, plan.stats())
