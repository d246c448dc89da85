"""Edge cases of the reference's batch contract (check_batch, /root/reference/proj/src/attention.cpp:
23-48) on the GPU path, each against the CPU oracle:

* zero-length spans (query_len 0, with or without cached context) between real spans;
* a batch whose spans are all zero-length, and an empty batch (no spans);
* contexts that end exactly on a page boundary, contexts of one token, one-token pages left
  over (context % 16 == 1);
* the highest slot of the pool in a block table;
* the widest GQA groups (64 query heads on one kv head) and an MHA layout;
* long contexts (16K tokens) for decode and prefill spans in one batch, both the fused schedule
  and the separate-decode schedule.
Tolerance (BASELINE.json north_star, bf16): |gpu - oracle| <= 2e-2 + 1e-2 * |oracle|."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, AttnShape, Batch  # noqa: E402
from paper_2312_05516_b200.workloads import SplitMix64, _build  # noqa: E402


@pytest.fixture(scope="module")
def gh(cuda):
    import gpu_helpers as gh
    return gh


def _check(gh, oracle, w, flags=0):
    q, k, v = gh.device_inputs(w)
    got, plan = gh.run_plan(w, q, k, v, flags=flags)
    st, want = oracle.attention(w.shape(), w.batch(), w.host_q(), w.host_pool("k"), w.host_pool("v"))
    assert st == 0
    if want.size:
        ok, err = gh.bf16_close(got, want)
        assert ok, (err, plan.stats())
    return plan


@pytest.mark.parametrize("n_head,n_kv", [(64, 8), (8, 8)])
def test_zero_length_spans_between_real_spans(gh, oracle, n_head, n_kv):
    convs = [[(0, 40)], [(37, 0)], [(500, 1)], [(0, 0)], [(128, 3)], [(16, 0)], [(1000, 1)], [(64, 65)]]
    w = _build("zlen", n_head, n_kv, 128, 16, PB_BF16, 3, convs, SplitMix64(3))
    _check(gh, oracle, w)


def test_all_zero_length_spans(gh, oracle):
    w = _build("allzero", 16, 4, 128, 16, PB_BF16, 4, [[(37, 0)], [(0, 0)], [(255, 0)]], SplitMix64(4))
    assert w.total_tokens == 0
    q, k, v = gh.device_inputs(w)
    out, plan = gh.run_plan(w, q, k, v)
    assert out.size == 0


def test_empty_batch_plans_and_runs():
    import torch
    shape = AttnShape(n_head=8, n_kv_head=2, head_size=128, chunk_size=16, n_slots=4, dtype=PB_BF16, scale=11.3)
    plan = abi.AttentionPlan(shape, Batch([], [], []))
    st = torch.cuda.current_stream().cuda_stream
    plan.upload(st)
    buf = torch.zeros(16, dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    plan.run(buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), ws.data_ptr(), st)
    torch.cuda.synchronize()
    assert plan.stats()["prefill_tiles"] == 0 and plan.stats()["decode_units"] == 0


def test_page_boundaries_and_single_tokens(gh, oracle):
    # contexts 16, 32, 1, 17, 129 (one row into a new page), 2048 (exact), prefill spans ending on
    # a page edge and one row past it
    convs = [[(15, 1)], [(31, 1)], [(0, 1)], [(16, 1)], [(128, 1)], [(2047, 1)], [(0, 32)], [(0, 33)], [(96, 33)]]
    w = _build("pages", 32, 4, 128, 16, PB_BF16, 5, convs, SplitMix64(5))
    _check(gh, oracle, w)


def test_highest_slot_in_use(gh, oracle):
    w = _build("topslot", 16, 2, 128, 16, PB_BF16, 6, [[(100, 20)], [(300, 1)]], SplitMix64(6))
    top = w.n_slots - 1
    for t in w.conv_tables:
        assert t.dtype == np.int32
    assert any(top in t for t in w.conv_tables)
    _check(gh, oracle, w)


@pytest.mark.parametrize("n_head,n_kv", [(64, 1), (40, 40)])
def test_extreme_group_sizes(gh, oracle, n_head, n_kv):
    convs = [[(0, 70)], [(200, 1)], [(33, 17)], [(900, 1)]]
    w = _build("groups", n_head, n_kv, 128, 16, PB_BF16, 7, convs, SplitMix64(7))
    _check(gh, oracle, w)


@pytest.mark.parametrize("flags", [0, abi.PB_PLAN_SEPARATE_DECODE])
def test_long_contexts(gh, oracle, flags):
    convs = [[(16383, 1)], [(16000, 100)], [(5000, 1)], [(0, 300)]]
    w = _build("long", 16, 2, 128, 16, PB_BF16, 8, convs, SplitMix64(8))
    _check(gh, oracle, w, flags)


@pytest.mark.parametrize("d,chunk", [(96, 16), (256, 16), (32, 8), (128, 24)])
def test_shapes_outside_the_tensor_core_paths(gh, oracle, d, chunk):
    """Head sizes other than 64 / 128 and pages that do not tile a 128-row kv tile run on the
    SIMT kernel (bf16 in, fp32 accumulation); same contract, same oracle."""
    convs = [[(0, 50)], [(300, 1)], [(77, 9)], [(1000, 1)]]
    w = _build(f"simt{d}", 8, 2, d, chunk, PB_BF16, 9, convs, SplitMix64(9))
    plan = _check(gh, oracle, w)
    assert plan.stats()["simt_tiles"] > 0
