"""Page gather / scatter / append kernels: bit-exact against the CPU restatement
(oracle/attn_oracle.c) and the reference's paged-write addressing (qkv_project,
proj/src/attention.cpp:315-327; KAT proj/tests/test_attention.cpp:465-483)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, PB_F32, AttnShape  # noqa: E402


@pytest.mark.parametrize("layer_major", [0, 1])
def test_gather_scatter_multi_layer_bit_exact(cuda, oracle, layer_major):
    torch = cuda
    n_layers, n_slots, page_bytes = 3, 37, 16 * 10 * 128 * 2  # Llama-2-13B page, bf16
    rng = np.random.default_rng(1)
    pool = rng.integers(0, 256, size=n_layers * n_slots * page_bytes, dtype=np.uint8)
    d_pool = torch.from_numpy(pool).cuda()
    slots = np.array([5, 0, 36, 17, 9, 22], np.int32)
    d_slots = torch.from_numpy(slots).cuda()
    stage = torch.zeros(n_layers * len(slots) * page_bytes, dtype=torch.uint8, device="cuda")
    abi.gather_pages(d_pool.data_ptr(), n_slots * page_bytes, n_layers, page_bytes, d_slots.data_ptr(),
                     len(slots), stage.data_ptr(), layer_major)
    torch.cuda.synchronize()
    got = stage.cpu().numpy().reshape(-1, page_bytes)
    for l in range(n_layers):
        want = oracle.gather(pool[l * n_slots * page_bytes:(l + 1) * n_slots * page_bytes], page_bytes, slots)
        want = want.reshape(len(slots), page_bytes)
        for i in range(len(slots)):
            row = l * len(slots) + i if layer_major else i * n_layers + l
            assert np.array_equal(got[row], want[i])
    # scatter into a zero pool at different slots == oracle scatter
    dst_slots = np.array([1, 2, 3, 30, 31, 32], np.int32)
    d_dst = torch.from_numpy(dst_slots).cuda()
    pool2 = torch.zeros_like(d_pool)
    abi.scatter_pages(stage.data_ptr(), n_slots * page_bytes, n_layers, page_bytes, d_dst.data_ptr(),
                      len(dst_slots), pool2.data_ptr(), layer_major)
    torch.cuda.synchronize()
    got_pool = pool2.cpu().numpy()
    for l in range(n_layers):
        ref = np.zeros(n_slots * page_bytes, np.uint8)
        st = np.concatenate([got[(l * len(slots) + i) if layer_major else (i * n_layers + l)]
                             for i in range(len(slots))])
        oracle.scatter(st, page_bytes, dst_slots, ref)
        assert np.array_equal(got_pool[l * n_slots * page_bytes:(l + 1) * n_slots * page_bytes], ref)


def _append(torch, shape, spans, k_rows, v_rows, k_pages, v_pages):
    """spans: list of (start_pos, n_rows, block_table)."""
    row_start = np.cumsum([0] + [n for _, n, _ in spans[:-1]]).astype(np.int64)
    n_rows = np.array([n for _, n, _ in spans], np.int64)
    start = np.array([s for s, _, _ in spans], np.int64)
    bt = np.concatenate([np.asarray(t, np.int32) for _, _, t in spans])
    bt_off = np.cumsum([0] + [len(t) for _, _, t in spans]).astype(np.int64)
    dev = [torch.from_numpy(a).cuda() for a in (row_start, n_rows, start, bt, bt_off)]
    p = lambda a: a.ctypes.data  # noqa: E731
    abi.check(abi.lib.pb_kv_append(
        abi.ctypes.byref(shape), len(spans), p(row_start), p(n_rows), p(start), p(bt), p(bt_off),
        *[d.data_ptr() for d in dev], k_rows.data_ptr(), v_rows.data_ptr(), k_pages.data_ptr(),
        v_pages.data_ptr(), None))
    torch.cuda.synchronize()


def test_append_matches_qkv_project_addressing(cuda, oracle):
    torch = cuda
    # proj/tests/test_attention.cpp:465-483: chunk 4, 2 kv heads x 4, table {0, 2, 1},
    # positions 6..9 -> pos 6 in slot 2 row 2, pos 9 in slot 1 row 1
    shape = AttnShape(2, 2, 4, 4, 3, PB_F32, 2.0)
    rows = np.arange(4 * 8, dtype=np.float32).reshape(4, 8) + 1
    k_pages = torch.zeros(3 * 4 * 8, device="cuda")
    v_pages = torch.zeros_like(k_pages)
    kr = torch.from_numpy(rows).cuda()
    _append(torch, shape, [(6, 4, [0, 2, 1])], kr, -kr, k_pages, v_pages)
    kp = k_pages.cpu().numpy()
    assert kp[(2 * 4 + 2) * 8 + 0] == rows[0, 0]
    assert v_pages.cpu().numpy()[(1 * 4 + 1) * 8 + 7] == -rows[3, 7]
    ref = np.zeros(3 * 4 * 8, np.float32)
    assert oracle.append(ref, 4, 3, 8, [0, 2, 1], 6, rows) == 0
    assert np.array_equal(kp, ref)


def test_append_ragged_bf16_and_errors(cuda, oracle):
    torch = cuda
    shape = AttnShape(8, 2, 128, 16, 40, PB_BF16, 1.0)
    row = 2 * 128
    spans = [(37, 20, [3, 7, 11, 12]), (0, 1, [0]), (100, 29, [20, 21, 22, 23, 24, 25, 26, 27, 28])]
    total = sum(n for _, n, _ in spans)
    kr = torch.randn(total, row, device="cuda").to(torch.bfloat16)
    vr = torch.randn(total, row, device="cuda").to(torch.bfloat16)
    kp = torch.zeros(40 * 16 * row, dtype=torch.bfloat16, device="cuda")
    vp = torch.zeros_like(kp)
    _append(torch, shape, spans, kr, vr, kp, vp)
    ref_k = np.zeros(40 * 16 * row, np.float32)
    r0 = 0
    krn = kr.float().cpu().numpy()
    for start, n, table in spans:
        assert oracle.append(ref_k, 16, 40, row, table, start, krn[r0:r0 + n]) == 0
        r0 += n
    assert np.array_equal(kp.float().cpu().numpy(), ref_k)
    with pytest.raises(abi.DimensionMismatch):  # table too short for the written positions
        _append(torch, shape, [(40, 20, [3, 7])], kr[:20], vr[:20], kp, vp)
    with pytest.raises(abi.Error):  # out-of-range slot
        _append(torch, shape, [(0, 2, [99])], kr[:2], vr[:2], kp, vp)
