"""Pins the CPU oracle (oracle/attn_oracle.c) before anything is checked against it.

* the reference's own known-answer tests for attention (proj/tests/test_attention.cpp) and
  SplitMix64 (proj/tests/test_workload.cpp:209-214), re-run against the oracle;
* the golden outputs of the reference in tests/golden/ (tests/golden/make_golden.py);
* bit-identity with the reference library itself (oracle/_ref) on acceptance-style
  instances, including the causal-independence check with the CORRECTED predicate
  (proj/tests/acceptance.cpp:261-264 selects the wrong token).
"""
import json
import math
import os

import numpy as np
import pytest

from paper_2312_05516_b200.abi import PB_F32, AttnShape, Batch
from paper_2312_05516_b200.workloads import SplitMix64, Workload, random_instance, unit_draws

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_unit(rng, n):
    return np.array([float(2.0 * rng.u01() - 1.0) for _ in range(n)], dtype=np.float32)


def test_splitmix_kat(oracle):
    # proj/tests/test_workload.cpp:209-214
    assert oracle.splitmix(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    g = json.load(open(os.path.join(GOLDEN, "splitmix.json")))
    for seed, vals in g["streams"].items():
        assert [hex(x) for x in oracle.splitmix(int(seed), 16)] == vals
        r = SplitMix64(int(seed))
        assert [hex(r.next()) for _ in range(16)] == vals


def test_counter_fill_matches_sequential(oracle):
    for seed in (0, 3, 20260814):
        seq = oracle.fill_unit(seed, 4096)
        assert np.array_equal(unit_draws(seed, 0, 4096), seq)
        assert np.array_equal(unit_draws(seed, 1000, 96), seq[1000:1096])


def one_span(q_len, ctx, table, n_head, hs, n_kv, chunk, n_slots, scale=None):
    shape = AttnShape(n_head, n_kv, hs, chunk, n_slots, PB_F32, scale or math.sqrt(hs))
    batch = Batch([q_len], [ctx - q_len], [table])
    return shape, batch


def test_kat_single_position_returns_v_row(oracle):
    # proj/tests/test_attention.cpp:119-144
    rng = SplitMix64(1)
    n_slots, chunk, nkv, hs = 2, 4, 2, 8
    keys = np.zeros(n_slots * chunk * nkv * hs, np.float32)
    vals = np.zeros_like(keys)
    row = 1 * chunk * nkv * hs
    for e in range(16):
        keys[row + e] = rand_unit(rng, 1)[0]
        vals[row + e] = rand_unit(rng, 1)[0]
    q = rand_unit(rng, 16)
    shape, batch = one_span(1, 1, [1], 2, hs, nkv, chunk, n_slots)
    st, out = oracle.attention(shape, batch, q, keys, vals)
    assert st == 0
    assert np.array_equal(out, vals[row:row + 16])
    st, single = oracle.attention(shape, batch, q, keys, vals, single=True)
    assert st == 0 and np.array_equal(single, out)


def test_kat_causal_sentinel(oracle):
    # proj/tests/test_attention.cpp:146-179
    rng = SplitMix64(2)
    hs = 8
    keys = np.zeros(8 * hs, np.float32)
    vals = np.zeros_like(keys)
    for p in range(5):
        for e in range(hs):
            keys[p * hs + e] = rand_unit(rng, 1)[0]
            vals[p * hs + e] = rand_unit(rng, 1)[0]
    q = rand_unit(rng, 2 * hs)
    shape, batch = one_span(2, 5, [0], 1, hs, 1, 8, 1)
    st, before = oracle.attention(shape, batch, q, keys, vals)
    keys[4 * hs:5 * hs] = 5.0
    vals[4 * hs:5 * hs] = -7.0
    st2, after = oracle.attention(shape, batch, q, keys, vals)
    assert st == st2 == 0
    assert np.array_equal(before[:hs], after[:hs])
    assert np.abs(before[hs:] - after[hs:]).sum() > 0


def test_kat_uniform_keys(oracle):
    # proj/tests/test_attention.cpp:199-221
    hs = 4
    keys = np.zeros(8 * hs, np.float32)
    vals = np.zeros_like(keys)
    for p in range(4):
        keys[p * hs:(p + 1) * hs] = 1.0
        vals[p * hs:(p + 1) * hs] = p
    q = np.array([0.3, -0.2, 0.9, 0.1], np.float32)
    shape, batch = one_span(1, 4, [0], 1, hs, 1, 8, 1, scale=2.0)
    st, out = oracle.attention(shape, batch, q, keys, vals)
    assert st == 0
    assert np.allclose(out, 1.5, rtol=1e-6)


def test_kat_errors(oracle):
    # proj/tests/test_attention.cpp:305-320 and :493-509
    shape, batch = one_span(2, 2, [0], 1, 4, 1, 8, 1, scale=2.0)
    q = np.full(8, 0.5, np.float32)
    kv = np.zeros(32, np.float32)
    assert oracle.attention(shape, batch, q, kv, kv, single=True)[0] == 1  # DimensionMismatch
    assert oracle.attention(shape, batch, q, kv, kv)[0] == 0
    qn = q.copy()
    qn[0] = np.nan
    assert oracle.attention(shape, batch, qn, kv, kv)[0] == 2  # NumericError
    short = Batch([2], [0], [[]], context_len=[2])
    assert oracle.attention(shape, short, q, kv, kv)[0] == 1
    bad_ctx = Batch([2], [0], [[0]], context_len=[3])
    assert oracle.attention(shape, bad_ctx, q, kv, kv)[0] == 1
    oob = Batch([2], [0], [[5]])
    assert oracle.attention(shape, oob, q, kv, kv)[0] == 3  # Error (out-of-range slot)
    kn = kv.copy()
    kn[0] = np.inf  # k_row[0] of position 0
    assert oracle.attention(shape, batch, q, kn, kv)[0] == 2


def test_kat_gqa_duplicated_equals_mha(oracle):
    # proj/tests/test_attention.cpp:358-397: grouped heads == duplicated kv heads, bit-exact
    rng = SplitMix64(17)
    hs, chunk, n_head, ctx = 8, 8, 4, 24
    table = [2, 0, 1]
    gk = np.zeros(3 * chunk * 2 * hs, np.float32)
    gv = np.zeros_like(gk)
    mk = np.zeros(3 * chunk * 4 * hs, np.float32)
    mv = np.zeros_like(mk)
    for p in range(ctx):
        slot, row = table[p // chunk], p % chunk
        for kvh in range(2):
            for e in range(hs):
                kval, vval = rand_unit(rng, 2)
                gk[(slot * chunk + row) * 2 * hs + kvh * hs + e] = kval
                gv[(slot * chunk + row) * 2 * hs + kvh * hs + e] = vval
                for dup in range(2):
                    mk[(slot * chunk + row) * 4 * hs + (kvh * 2 + dup) * hs + e] = kval
                    mv[(slot * chunk + row) * 4 * hs + (kvh * 2 + dup) * hs + e] = vval
    q = rand_unit(rng, 4 * n_head * hs)
    sg, bg = one_span(4, ctx, table, n_head, hs, 2, chunk, 3)
    sm, bm = one_span(4, ctx, table, n_head, hs, 4, chunk, 3)
    st1, grouped = oracle.attention(sg, bg, q, gk, gv)
    st2, full = oracle.attention(sm, bm, q, mk, mv)
    assert st1 == st2 == 0 and np.array_equal(grouped, full)


def test_golden_reference_outputs(oracle):
    """Oracle == reference outputs recorded in tests/golden (bit-exact)."""
    cases = json.load(open(os.path.join(GOLDEN, "attention_ref_cases.json")))["cases"]
    outs = np.load(os.path.join(GOLDEN, "attention_ref_outputs.npz"))
    for c in cases:
        w = Workload("golden", c["n_head"], c["n_kv_head"], 8, c["chunk"], PB_F32, c["seed"],
                     [tuple(s) for s in c["spans"]], [np.array(t, np.int32) for t in c["tables"]],
                     c["n_slots"], c["pool_first_draw"])
        shape, batch = w.shape(), w.batch()
        q, k, v = w.host_q(), w.host_pool("k"), w.host_pool("v")
        st, out = oracle.attention(shape, batch, q, k, v)
        assert st == 0
        assert np.array_equal(out, outs[f"paged_{c['trial']}"]), c["trial"]
        if c["all_decode"]:
            st, single = oracle.attention(shape, batch, q, k, v, single=True)
            assert st == 0 and np.array_equal(single, outs[f"single_{c['trial']}"])
        assert c["copyout_equals_paged"]


def test_oracle_bit_identical_to_reference(oracle, reference):
    """Acceptance criterion 2 shapes (proj/tests/acceptance.cpp:201-306): oracle == reference
    bit for bit; row sums; causal independence with the corrected predicate; slot
    permutation invariance."""
    rng = SplitMix64(20260814)
    pairs = [(1, 1), (3, 3), (8, 8), (2, 1), (4, 2), (8, 4), (4, 1), (8, 2)]
    for trial in range(30):
        nh, nkv = pairs[rng.next() % 8]
        chunk = 16 if rng.next() % 2 == 0 else 32
        w = random_instance(rng, nh, nkv, 8, chunk, PB_F32, 1 + rng.next() % 4, 1024, max_q=16)
        shape, batch = w.shape(), w.batch()
        q, k, v = w.host_q(), w.host_pool("k"), w.host_pool("v")
        st, ours = oracle.attention(shape, batch, q, k, v)
        rst, theirs, _ = reference.attention(shape, batch, q, k, v)
        assert st == rst == 0
        assert np.array_equal(ours, theirs)
        # row sums with all-ones values
        st, ones = oracle.attention(shape, batch, q, k, np.ones_like(v))
        assert np.max(np.abs(ones - 1.0)) <= 1e-6
        # causal independence: perturb the last context position of span 0; only its last
        # token may change (corrected predicate)
        if batch.query_len[0] >= 2:
            k2, v2 = k.copy(), v.copy()
            p = int(batch.context_len[0]) - 1
            slot = batch.table(0)[p // chunk]
            r0 = (slot * chunk + p % chunk) * w.row_elems
            k2[r0:r0 + w.row_elems] += 10.0
            v2[r0:r0 + w.row_elems] += 10.0
            st, after = oracle.attention(shape, batch, q, k2, v2)
            stride = nh * 8
            tok = np.arange(ours.size) // stride
            last = int(batch.query_start[0] + batch.query_len[0] - 1)
            keep = tok != last
            assert np.array_equal(ours[keep], after[keep])
        # slot permutation: relocate pages and remap tables -> bit-identical
        perm = np.arange(w.n_slots)
        for i in range(len(perm), 1, -1):
            j = rng.next() % i
            perm[i - 1], perm[j] = perm[j], perm[i - 1]
        page = chunk * w.row_elems
        k3 = np.empty_like(k)
        v3 = np.empty_like(v)
        for s in range(w.n_slots):
            k3[perm[s] * page:(perm[s] + 1) * page] = k[s * page:(s + 1) * page]
            v3[perm[s] * page:(perm[s] + 1) * page] = v[s * page:(s + 1) * page]
        b3 = Batch(batch.query_len, batch.causal_offset, [perm[batch.table(i)] for i in range(batch.n_spans)])
        st, moved = oracle.attention(shape, b3, q, k3, v3)
        assert np.array_equal(moved, ours)


def test_dense_matches_paged(oracle, reference):
    rng = SplitMix64(42)
    w = random_instance(rng, 4, 2, 8, 16, PB_F32, 3, 96)
    shape, batch = w.shape(), w.batch()
    q, k, v = w.host_q(), w.host_pool("k"), w.host_pool("v")
    st, paged = oracle.attention(shape, batch, q, k, v)
    row = w.row_elems
    for i in range(batch.n_spans):
        ctx = int(batch.context_len[i])
        kd = np.concatenate([k[(batch.table(i)[p // 16] * 16 + p % 16) * row:][:row] for p in range(ctx)])
        vd = np.concatenate([v[(batch.table(i)[p // 16] * 16 + p % 16) * row:][:row] for p in range(ctx)])
        qs, ql = int(batch.query_start[i]), int(batch.query_len[i])
        qi = q[qs * 4 * 8:(qs + ql) * 4 * 8]
        st, d = oracle.dense(qi, kd, vd, ql, ctx, int(batch.causal_offset[i]), 4, 2, 8, w.scale)
        assert st == 0
        assert np.max(np.abs(d - paged[qs * 32:(qs + ql) * 32])) <= 1e-5


def test_page_copy_oracle_roundtrip(oracle):
    rng = np.random.default_rng(0)
    pool = rng.integers(0, 255, size=16 * 512, dtype=np.uint8)
    slots = np.array([3, 15, 0, 7], np.int32)
    st = oracle.gather(pool, 512, slots)
    for i, s in enumerate(slots):
        assert np.array_equal(st[i * 512:(i + 1) * 512], pool[s * 512:(s + 1) * 512])
    pool2 = np.zeros_like(pool)
    oracle.scatter(st, 512, slots, pool2)
    for s in slots:
        assert np.array_equal(pool2[s * 512:(s + 1) * 512], pool[s * 512:(s + 1) * 512])


def test_group_oracle_is_the_whole_oracle(oracle):
    """tests/gpu_helpers.group_oracle (one kv-head group, spans cut into token blocks on
    host threads) is bit-identical to the whole-batch oracle on those rows: heads are
    independent (src/attention.cpp:90-92) and a token block is a span of its own."""
    import gpu_helpers as gh
    from paper_2312_05516_b200.abi import PB_BF16
    from paper_2312_05516_b200.workloads import SplitMix64, random_instance
    rng = SplitMix64(99)
    w = random_instance(rng, 8, 2, 64, 16, PB_BF16, 4, 300, max_q=150)
    st, want = oracle.attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
    assert st == 0
    ids = list(range(len(w.spans)))
    for kvh in range(2):
        got = gh.group_oracle(oracle, w, ids, kvh, threads=4, block=37)
        assert np.array_equal(got, gh.group_rows(want, w, ids, kvh))
