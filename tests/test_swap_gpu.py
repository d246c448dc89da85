"""CPU-tier swap engine (pb_swap_step): bytes land where the bookkeeping's slot moves say,
bit-exact, with the reference's ordering contract (src/swap_engine.cpp:21-53) and the
same-step slot-reuse hazards of the LIFO reclaim (src/paged_kv_cache.cpp:28-37) handled."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200.abi import (PB_D2H_AFTER_SWAP_IN, PB_D2H_CONCURRENT,  # noqa: E402
                                       PB_D2H_ON_COPY_STREAM, PB_SWAP_IN_STAGED, PB_SWAP_IN_ZERO_COPY,
                                       KvCache, KvTier)

D2H_MODES = [PB_D2H_AFTER_SWAP_IN, PB_D2H_CONCURRENT, PB_D2H_ON_COPY_STREAM]
SWAP_IN = [PB_SWAP_IN_STAGED, PB_SWAP_IN_ZERO_COPY]


def _pools(torch, n_layer, n_slots, page_bytes, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    k = torch.randint(0, 256, (n_layer, n_slots, page_bytes), dtype=torch.uint8, device="cuda", generator=g)
    v = torch.randint(0, 256, (n_layer, n_slots, page_bytes), dtype=torch.uint8, device="cuda", generator=g)
    return k, v


def test_swap_out_then_in_roundtrip(cuda):
    torch = cuda
    L, n_slots, page = 3, 24, 16 * 2 * 128 * 2
    k, v = _pools(torch, L, n_slots, page, 1)
    k0, v0 = k.cpu().numpy().copy(), v.cpu().numpy().copy()
    tier = KvTier(L, 16, page, 8)
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    out = [(100, 3, 5), (101, 7, 0), (102, 20, 9)]  # chunk, device src -> host dst
    tier.step(k.data_ptr(), v.data_ptr(), n_slots * page, out, [], cs.cuda_stream, xs.cuda_stream)
    tier.sync()
    host = tier.host_view().reshape(16, L, 2, page)
    for _, d, h in out:
        for l in range(L):
            assert np.array_equal(host[h, l, 0], k0[l, d]) and np.array_equal(host[h, l, 1], v0[l, d])
    # swap back into different device slots, layer by layer
    back = [(100, 5, 11), (101, 0, 12), (102, 9, 13)]  # host src -> device dst
    tier.step(k.data_ptr(), v.data_ptr(), n_slots * page, [], back, cs.cuda_stream, xs.cuda_stream)
    for l in range(L):
        tier.wait_layer(l, cs.cuda_stream)
    torch.cuda.synchronize()
    kn, vn = k.cpu().numpy(), v.cpu().numpy()
    for (_, d, _h), (_, _h2, dd) in zip(out, back):
        for l in range(L):
            assert np.array_equal(kn[l, dd], k0[l, d]) and np.array_equal(vn[l, dd], v0[l, d])


@pytest.mark.parametrize("d2h_mode", D2H_MODES)  # D2H after / concurrent with / behind swap-ins
@pytest.mark.parametrize("swap_in", SWAP_IN)
def test_same_step_slot_reuse_hazard(cuda, d2h_mode, swap_in):
    """A device slot vacated by swap-out is refilled by a swap-in in the SAME step (the LIFO
    reclaim makes this common): the host must get the old bytes, the device the new ones."""
    torch = cuda
    L, n_slots, page = 4, 8, 4096
    k, v = _pools(torch, L, n_slots, page, 2)
    k0, v0 = k.cpu().numpy().copy(), v.cpu().numpy().copy()
    tier = KvTier(L, 4, page, 4)
    tier.set_policy(swap_in, d2h_mode)
    host = tier.host_view().reshape(4, L, 2, page)
    rng = np.random.default_rng(3)
    host[2] = rng.integers(0, 256, size=(L, 2, page), dtype=np.uint8)  # chunk resident on host slot 2
    incoming = host[2].copy()
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    # evict device slot 6 -> host slot 1, restore host slot 2 -> device slot 6 (same step)
    tier.step(k.data_ptr(), v.data_ptr(), n_slots * page, [(7, 6, 1)], [(9, 2, 6)], cs.cuda_stream, xs.cuda_stream)
    for l in range(L):
        tier.wait_layer(l, cs.cuda_stream)
    tier.sync()
    torch.cuda.synchronize()
    for l in range(L):
        assert np.array_equal(host[1, l, 0], k0[l, 6]) and np.array_equal(host[1, l, 1], v0[l, 6])
        assert np.array_equal(k.cpu().numpy()[l, 6], incoming[l, 0])
        assert np.array_equal(v.cpu().numpy()[l, 6], incoming[l, 1])


def test_cache_moves_drive_the_engine(cuda):
    """Bookkeeping -> bytes: moves reported by pb_cache_* are executed by pb_swap_step and
    every chunk's bytes follow it through evict -> restore cycles."""
    torch = cuda
    L, dev_slots, host_slots, page = 2, 12, 12, 2048
    cache = KvCache(16, dev_slots, host_slots)
    k, v = _pools(torch, L, dev_slots, page, 4)
    tier = KvTier(L, host_slots, page, dev_slots)
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    ids = cache.allocate(1, 16 * 6, 0.0) + cache.allocate(2, 16 * 4, 0.0)
    truth = {c: (k.cpu().numpy()[:, cache.chunk(c).slot].copy(), v.cpu().numpy()[:, cache.chunk(c).slot].copy())
             for c in ids}
    out = cache.apply_evictions(ids[:5], True)
    ids3 = cache.allocate(3, 16 * 5, 1.0)  # reuses the vacated slots (LIFO) in the same step
    tier.step(k.data_ptr(), v.data_ptr(), dev_slots * page, out, [], cs.cuda_stream, xs.cuda_stream)
    tier.sync()
    assert len(ids3) == 5
    cache.release_conversation(3)
    back = cache.restore(ids[:5])
    tier.step(k.data_ptr(), v.data_ptr(), dev_slots * page, [], back, cs.cuda_stream, xs.cuda_stream)
    tier.sync()
    torch.cuda.synchronize()
    kn, vn = k.cpu().numpy(), v.cpu().numpy()
    for c in ids[:5]:
        s = cache.chunk(c).slot
        assert np.array_equal(kn[:, s], truth[c][0]) and np.array_equal(vn[:, s], truth[c][1])


@pytest.mark.parametrize("d2h_mode", D2H_MODES)  # D2H after / concurrent with / behind swap-ins
@pytest.mark.parametrize("swap_in", SWAP_IN)
def test_host_slot_hazards_across_and_within_steps(cuda, d2h_mode, swap_in):
    """Host-side hazards of the double-buffered engine: (a) a swap-in in step s+1 from the host
    slot step s swapped out to (RAW across steps, without a host sync in between) gets the
    swapped-out bytes; (b) in one step, a swap-in reading host slot X and a swap-out writing X
    (restore frees X at once, src/paged_kv_cache.cpp:190) -- the swap-in gets the OLD bytes."""
    torch = cuda
    L, n_slots, page = 6, 16, 8192
    k, v = _pools(torch, L, n_slots, page, 4)
    k0, v0 = k.cpu().numpy().copy(), v.cpu().numpy().copy()
    tier = KvTier(L, 6, page, 4)
    tier.set_policy(swap_in, d2h_mode)
    host = tier.host_view().reshape(6, L, 2, page)
    rng = np.random.default_rng(5)
    host[3] = rng.integers(0, 256, size=(L, 2, page), dtype=np.uint8)
    old3 = host[3].copy()
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    stride = n_slots * page
    # step 1: device slot 2 -> host slot 0
    tier.step(k.data_ptr(), v.data_ptr(), stride, [(1, 2, 0)], [], cs.cuda_stream, xs.cuda_stream)
    # step 2 (issued immediately): host slot 0 -> device slot 9 (RAW on host slot 0), and in the
    # same step host slot 3 -> device slot 10 while device slot 4 -> host slot 3 (WAR on slot 3)
    tier.step(k.data_ptr(), v.data_ptr(), stride, [(2, 4, 3)], [(1, 0, 9), (3, 3, 10)], cs.cuda_stream,
              xs.cuda_stream)
    for l in range(L):
        tier.wait_layer(l, cs.cuda_stream)
    tier.sync()
    torch.cuda.synchronize()
    kn, vn = k.cpu().numpy(), v.cpu().numpy()
    for l in range(L):
        assert np.array_equal(kn[l, 9], k0[l, 2]) and np.array_equal(vn[l, 9], v0[l, 2])
        assert np.array_equal(kn[l, 10], old3[l, 0]) and np.array_equal(vn[l, 10], old3[l, 1])
        assert np.array_equal(host[3, l, 0], k0[l, 4]) and np.array_equal(host[3, l, 1], v0[l, 4])


@pytest.mark.parametrize("d2h_mode", D2H_MODES)  # D2H after / concurrent with / behind swap-ins
@pytest.mark.parametrize("swap_in", SWAP_IN)
def test_cross_step_war_on_a_freed_host_slot(cuda, d2h_mode, swap_in):
    """The D2H no longer joins the copy stream, so a step's swap-out could race the previous
    step's swap-in from the same host slot (restore frees it at once and the next eviction may
    reuse it).  Step 1 swaps host slot 5 in; step 2, issued right away with no layer wait on the
    compute stream, swaps a device slot out to host slot 5: step 1 must still read the OLD bytes."""
    torch = cuda
    L, n_slots, page = 8, 16, 1 << 16
    k, v = _pools(torch, L, n_slots, page, 6)
    k0, v0 = k.cpu().numpy().copy(), v.cpu().numpy().copy()
    tier = KvTier(L, 8, page, 8)
    tier.set_policy(swap_in, d2h_mode)
    host = tier.host_view().reshape(8, L, 2, page)
    rng = np.random.default_rng(7)
    host[:] = rng.integers(0, 256, size=host.shape, dtype=np.uint8)
    old = host.copy()
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    stride = n_slots * page
    ins = [(c, h, 8 + h) for c, h in enumerate(range(8))]  # every host slot -> device 8..15
    tier.step(k.data_ptr(), v.data_ptr(), stride, [], ins, cs.cuda_stream, xs.cuda_stream)
    tier.step(k.data_ptr(), v.data_ptr(), stride, [(9, 1, 5)], [], cs.cuda_stream, xs.cuda_stream)
    for l in range(L):
        tier.wait_layer(l, cs.cuda_stream)
    tier.sync()
    torch.cuda.synchronize()
    kn, vn = k.cpu().numpy(), v.cpu().numpy()
    for l in range(L):
        for h in range(8):
            assert np.array_equal(kn[l, 8 + h], old[h, l, 0]) and np.array_equal(vn[l, 8 + h], old[h, l, 1])
        assert np.array_equal(host[5, l, 0], k0[l, 1]) and np.array_equal(host[5, l, 1], v0[l, 1])


@pytest.mark.parametrize("d2h_mode", D2H_MODES)
@pytest.mark.parametrize("swap_in", SWAP_IN)
def test_evict_then_restore_same_chunk_in_one_step(cuda, d2h_mode, swap_in):
    """make_room can evict a queued conversation's chunk (device d -> host h) and a later
    admission in the SAME step restore it (host h -> device d').  The restore must get the
    evicted bytes (from the swap-out staging), not the stale host slot; the dead host copy is
    not written, so a later eviction into h in the same step owns it."""
    torch = cuda
    L, n_slots, page = 5, 16, 4096
    k, v = _pools(torch, L, n_slots, page, 8)
    k0, v0 = k.cpu().numpy().copy(), v.cpu().numpy().copy()
    tier = KvTier(L, 4, page, 4)
    tier.set_policy(swap_in, d2h_mode)
    host = tier.host_view().reshape(4, L, 2, page)
    host[:] = 7  # stale bytes
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    # chunk 5: device 3 -> host 1 -> device 12; then chunk 6: device 4 -> host 1 (slot reused)
    tier.step(k.data_ptr(), v.data_ptr(), n_slots * page, [(5, 3, 1), (6, 4, 1)], [(5, 1, 12)],
              cs.cuda_stream, xs.cuda_stream)
    for l in range(L):
        tier.wait_layer(l, cs.cuda_stream)
    tier.sync()
    torch.cuda.synchronize()
    kn, vn = k.cpu().numpy(), v.cpu().numpy()
    for l in range(L):
        assert np.array_equal(kn[l, 12], k0[l, 3]) and np.array_equal(vn[l, 12], v0[l, 3])
        assert np.array_equal(host[1, l, 0], k0[l, 4]) and np.array_equal(host[1, l, 1], v0[l, 4])


@pytest.mark.parametrize("d2h_mode", [PB_D2H_AFTER_SWAP_IN, PB_D2H_CONCURRENT])
@pytest.mark.parametrize("swap_in", SWAP_IN)
def test_raw_two_steps_back(cuda, d2h_mode, swap_in):
    """Step 1 swaps out to host slot h, step 2 moves nothing, step 3 restores from h with no
    swap-outs: the restore must wait for step 1's D2H (still in flight on the D2H stream),
    not only for the previous step's."""
    torch = cuda
    L, n_slots, page = 8, 16, 1 << 17  # 2 MiB per chunk: the D2H is still running at step 3
    k, v = _pools(torch, L, n_slots, page, 9)
    k0, v0 = k.cpu().numpy().copy(), v.cpu().numpy().copy()
    tier = KvTier(L, 4, page, 4)
    tier.set_policy(swap_in, d2h_mode)
    host = tier.host_view().reshape(4, L, 2, page)
    host[:] = 3
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    stride = n_slots * page
    tier.step(k.data_ptr(), v.data_ptr(), stride, [(1, 2, 0), (2, 5, 3)], [], cs.cuda_stream, xs.cuda_stream)
    tier.step(k.data_ptr(), v.data_ptr(), stride, [], [], cs.cuda_stream, xs.cuda_stream)
    tier.step(k.data_ptr(), v.data_ptr(), stride, [], [(1, 0, 9), (2, 3, 10)], cs.cuda_stream, xs.cuda_stream)
    for l in range(L):
        tier.wait_layer(l, cs.cuda_stream)
    tier.sync()
    torch.cuda.synchronize()
    kn, vn = k.cpu().numpy(), v.cpu().numpy()
    for l in range(L):
        assert np.array_equal(kn[l, 9], k0[l, 2]) and np.array_equal(vn[l, 9], v0[l, 2])
        assert np.array_equal(kn[l, 10], k0[l, 5]) and np.array_equal(vn[l, 10], v0[l, 5])


def test_policy_validation(cuda):
    from paper_2312_05516_b200.abi import ConfigError
    tier = KvTier(2, 2, 256, 2)
    with pytest.raises(ConfigError):
        tier.set_policy(5, PB_D2H_AFTER_SWAP_IN)
    with pytest.raises(ConfigError):
        tier.set_policy(PB_SWAP_IN_STAGED, 9)
    with pytest.raises(ConfigError):
        tier.set_policy(PB_SWAP_IN_STAGED, PB_D2H_AFTER_SWAP_IN, 3)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tier_chunk_bytes_is_model_chunk_bytes(cuda, world):
    """A rank's tier over its shard pages holds ModelConfig::chunk_bytes per chunk
    (/root/reference/proj/src/model_config.cpp:36-40, n_partitions = world)."""
    from paper_2312_05516_b200.abi import chunk_bytes, model_preset
    m = model_preset("llama2-70b")
    m.n_partitions = world
    page = 16 * (m.n_kv_head // world) * m.head_size * m.bytes_per_scalar
    tier = KvTier(m.n_layer, 1, page, 1)
    assert tier.chunk_bytes == chunk_bytes(m, 16)
