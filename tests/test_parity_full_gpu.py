"""GPU parity at full span lengths (the long causal, multi-kv-tile, multi-item pipelines of
the headline configs) against the CPU oracle, and KV-head shard reassembly.

The oracle restates paged_multi_token_attention (/root/reference/proj/src/attention.cpp:73-132)
and is pinned to the reference in tests/test_oracle.py.  A kv-head group's outputs depend
only on that kv head and its query heads (:90-92), so the oracle runs one group per check,
with spans cut into token blocks over all host threads (tests/gpu_helpers.group_oracle,
itself checked bit-exact against the whole-batch oracle in tests/test_oracle.py).
Tolerance (BASELINE.json north_star, bf16): |gpu - oracle| <= 2e-2 + 1e-2 * |oracle|.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200.abi import PB_BF16  # noqa: E402
from paper_2312_05516_b200.workloads import SplitMix64, _build, config, random_instance  # noqa: E402


@pytest.fixture(scope="module")
def gh(cuda):
    import gpu_helpers as gh
    return gh


def _heaviest_prefill(w, n):
    pre = [i for i, (_, _, q) in enumerate(w.spans) if q > 1]
    return sorted(pre, key=lambda i: -w.flops_bytes([i])[0])[:n]


@pytest.mark.parametrize("cfg", [4, 2])
def test_heaviest_prefill_spans_full_length(gh, oracle, cfg):
    """The 3 heaviest prefill spans of the config (cfg4: q up to 1024 over up to 2048 past
    tokens, ~80 GF each), whole batch on the GPU, each span checked on one kv-head group."""
    w = config(cfg)
    q, k, v = gh.device_inputs(w)
    got, plan = gh.run_plan(w, q, k, v)
    assert np.all(np.isfinite(got))
    for n, i in enumerate(_heaviest_prefill(w, 3)):
        kvh = (3 * i + n) % w.n_kv_head
        want = gh.group_oracle(oracle, w, [i], kvh)
        ok, err = gh.bf16_close(gh.group_rows(got, w, [i], kvh).reshape(-1), want.reshape(-1))
        assert ok, (cfg, i, w.spans[i], kvh, err)


@pytest.mark.parametrize("n_head,n_kv", [(64, 8), (40, 10), (16, 16), (32, 4)])
def test_random_long_spans(gh, oracle, n_head, n_kv):
    """Random ragged batches with query spans up to 1024 tokens over contexts up to 4096
    (prefill, dropped-prefix-recompute-like spans with a long past, and decode), every span
    checked on two kv-head groups."""
    rng = SplitMix64(31000 + n_head + n_kv)
    for trial in range(2):
        w = random_instance(rng, n_head, n_kv, 128, 16, PB_BF16, 3 + rng.next() % 4, 4096, max_q=1024)
        q, k, v = gh.device_inputs(w)
        got, plan = gh.run_plan(w, q, k, v)
        ids = list(range(len(w.spans)))
        for kvh in sorted({0, n_kv - 1, (trial * 5) % n_kv})[:2]:
            want = gh.group_oracle(oracle, w, ids, kvh)
            ok, err = gh.bf16_close(gh.group_rows(got, w, ids, kvh).reshape(-1), want.reshape(-1))
            assert ok, (trial, kvh, err, w.spans, plan.stats())


def test_long_mixed_batch_with_recompute_spans(gh, oracle):
    """A conversation's dropped-prefix recompute span and its prompt span in one batch (the
    scheduler's two spans of one request), next to decode spans of long contexts."""
    rng = SplitMix64(4242)
    convs = [[(0, 700), (1600, 500)], [(4000, 1)], [(2500, 1)], [(0, 1024)], [(3071, 1)], [(900, 333)]]
    w = _build("mixed", 64, 8, 128, 16, PB_BF16, rng.seed, convs, rng)
    q, k, v = gh.device_inputs(w)
    got, _ = gh.run_plan(w, q, k, v)
    ids = list(range(len(w.spans)))
    for kvh in (2, 7):
        want = gh.group_oracle(oracle, w, ids, kvh)
        ok, err = gh.bf16_close(gh.group_rows(got, w, ids, kvh).reshape(-1), want.reshape(-1))
        assert ok, (kvh, err)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_kv_head_shard_reassembly(gh, oracle, cuda, world):
    """Config 4 sharded by kv head: rank r's pools hold kv heads
    [r*8/N, (r+1)*8/N) of the full pools; each rank runs its own plan over the same spans and
    block tables.  The concatenated head slices reproduce the unsharded output (bf16
    tolerance: a smaller shard may split decode spans differently) and the oracle."""
    torch = cuda
    from paper_2312_05516_b200.sharding import shard_shape
    w = config(4)
    q, k, v = gh.device_inputs(w)
    full, _ = gh.run_plan(w, q, k, v)
    d, nkv, g = w.head_size, w.n_kv_head, w.n_head // w.n_kv_head
    kk = k.view(w.n_slots * w.chunk, nkv, d)
    vv = v.view(w.n_slots * w.chunk, nkv, d)
    qq = q.view(w.total_tokens, w.n_head, d)
    parts = []
    for r in range(world):
        s = shard_shape(w.shape(), r, world)
        k0, k1 = r * s.n_kv_head, (r + 1) * s.n_kv_head
        ks = kk[:, k0:k1].contiguous()
        vs = vv[:, k0:k1].contiguous()
        qs = qq[:, k0 * g:k1 * g].contiguous()
        out, _ = gh.run_plan(w, qs, ks, vs, shape=s)
        parts.append(out.reshape(w.total_tokens, s.n_head, d))
    joined = np.concatenate(parts, axis=1).reshape(-1)
    ok, err = gh.bf16_close(joined, full)
    assert ok, err
    # oracle: the heaviest prefill span on the last rank's first kv head, plus two decode spans
    dec = [i for i, (_, _, ql) in enumerate(w.spans) if ql == 1][:2]
    heavy = _heaviest_prefill(w, 1)
    kvh = (world - 1) * (nkv // world)
    want = gh.group_oracle(oracle, w, heavy + dec, kvh)
    ok, err = gh.bf16_close(gh.group_rows(joined, w, heavy + dec, kvh).reshape(-1), want.reshape(-1))
    assert ok, err
