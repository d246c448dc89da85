"""KV page bookkeeping (pb_cache_*) against the reference PagedKvCache.

* the reference's own unit cases (proj/tests/test_paged_kv_cache.cpp) re-run on our cache;
* differential fuzz: the reference's two random-operation programs
  (proj/tests/test_paged_kv_cache.cpp:293-383 and proj/tests/acceptance.cpp:550-652) are
  replayed op for op on our cache and on the unmodified reference (oracle/_ref); after every
  op the dump(), the tier counters, every returned slot and every error class must be
  identical (bit-exact block tables and swap slot lists);
* the slot-pair (src, dst) triples our cache adds are checked for consistency.
"""
import pytest

from paper_2312_05516_b200 import abi
from paper_2312_05516_b200.abi import DEVICE, DROPPED, HOST, KvCache
from paper_2312_05516_b200.workloads import SplitMix64


def head(cache, conv, n):
    return [r.chunk_id for r in cache.conversation_chunks(conv)][:n]


def test_fill_partial_first():
    c = KvCache(32, 16, 16)
    created = c.allocate(1, 40, 0.0)
    assert [c.chunk(i).n_tokens for i in created] == [32, 8]
    assert [c.chunk(i).start_offset for i in created] == [0, 32]
    assert c.allocate(1, 24, 1.0) == []
    assert c.chunk(created[1]).n_tokens == 32 and c.chunk(created[1]).last_active == 1.0
    assert c.total_tokens(1) == 64
    c.verify()


def test_hundred_tokens_four_chunks_lowest_slots():
    c = KvCache(32, 8, 8)
    ids = c.allocate(5, 100, 0.0)
    assert [c.chunk(i).n_tokens for i in ids] == [32, 32, 32, 4]
    assert [c.chunk(i).slot for i in ids] == [0, 1, 2, 3]
    assert c.counts()["device_free"] == 4


def test_capacity_error_does_not_mutate():
    c = KvCache(32, 2, 2)
    c.allocate(1, 40, 0.0)
    before = (c.counts(), c.total_tokens(1))
    with pytest.raises(abi.InsufficientDeviceMemory):
        c.allocate(1, 64, 1.0)
    assert (c.counts(), c.total_tokens(1)) == before
    c.verify()


def test_layout_classifies_segments():
    c = KvCache(32, 16, 16)
    c.allocate(1, 320, 0.0)
    c.apply_evictions(head(c, 1, 5), True)
    c.apply_evictions(head(c, 1, 2), False)
    total, segs = c.layout(1)
    assert total == 320
    assert segs == [(DROPPED, 0, 64, 2), (HOST, 64, 160, 3), (DEVICE, 160, 320, 5)]
    with pytest.raises(abi.UnknownConversation):
        c.layout(99)


def test_lazy_reclaim_and_slot_pairs():
    c = KvCache(32, 8, 8)
    c.allocate(1, 96, 0.0)
    v = head(c, 1, 3)
    moves = c.apply_evictions(v, True)
    assert [(m[0], m[1]) for m in moves] == [(v[0], 0), (v[1], 1), (v[2], 2)]
    assert [m[2] for m in moves] == [0, 1, 2]  # host slots, lowest first
    cnt = c.counts()
    assert (cnt["device_reclaimable"], cnt["device_free"], cnt["host_free"], cnt["host_allocated"]) == (3, 5, 5, 3)
    with pytest.raises(abi.InvalidChunkState):
        c.apply_evictions([v[2]], True)
    c.apply_evictions(v[:2], False)
    with pytest.raises(abi.InvalidChunkState):
        c.apply_evictions([v[0]], False)
    # restore reuses the most recently vacated device slot first (LIFO lazy stack)
    back = c.restore([v[2]])
    assert back == [(v[2], 2, 2)]
    c.verify()


def test_host_overflow_throws_before_mutating():
    c = KvCache(32, 8, 1)
    c.allocate(1, 96, 0.0)
    with pytest.raises(abi.InsufficientHostMemory):
        c.apply_evictions(head(c, 1, 2), True)
    assert c.counts()["device_allocated"] == 3 and c.counts()["host_free"] == 1


def test_block_table_contract():
    c = KvCache(32, 8, 8)
    c.allocate(1, 100, 0.0)
    assert len(c.block_table(1, 100)) == 4 and len(c.block_table(1, 33)) == 2
    assert c.block_table(1, 0) == []
    with pytest.raises(abi.Error):
        c.block_table(1, 101)
    c.apply_evictions(head(c, 1, 1), True)
    with pytest.raises(abi.Error):
        c.block_table(1, 100)


def test_append_chunks_needed():
    c = KvCache(32, 8, 8)
    c.allocate(1, 40, 0.0)
    assert [c.append_chunks_needed(1, a) for a in (24, 25, 88)] == [0, 1, 2]
    assert c.append_chunks_needed(2, 1) == 1 and c.append_chunks_needed(2, 0) == 0


def test_release_frees_immediately():
    c = KvCache(32, 16, 16)
    c.allocate(1, 224, 0.0)
    c.retain_on_finish(1, 42.0)
    assert all(r.last_active == 42.0 for r in c.conversation_chunks(1))
    c.allocate(1, 50, 50.0)
    free_before = c.counts()["device_free"]
    c.release_conversation(1)
    assert c.counts()["device_allocated"] == 0 and c.counts()["device_free"] == free_before + 9
    assert c.total_tokens(1) == 0 and c.has_conversation(1)


class Pair:
    """Runs every op on ours and on the reference, asserting identical outcomes."""

    def __init__(self, reference, chunk, dev, host):
        from oracle.oracle import RefCache
        self.ours = KvCache(chunk, dev, host)
        self.ref = RefCache(reference, chunk, dev, host)
        self.ops = 0

    def call(self, name, *args):
        self.ops += 1
        res, err = {}, {}
        for tag, obj in (("ours", self.ours), ("ref", self.ref)):
            try:
                res[tag] = getattr(obj, name)(*args)
                err[tag] = 0
            except abi.PBError as e:
                err[tag] = e.code
            except Exception as e:  # RefCache.Err
                err[tag] = getattr(e, "code", -1)
        assert err["ours"] == err["ref"], (name, args, err)
        if not err["ours"]:
            a, b = res["ours"], res["ref"]
            if name in ("restore", "rematerialize"):
                a = [m[2] for m in a]  # device slots; the reference returns (chunk, slot)
            if name == "apply_evictions":
                a = b = None
            assert a == b, (name, args, a, b)
        return res.get("ours")

    def check(self):
        co, cr = self.ours.counts(), self.ref.counts()
        for k in ("device_free", "device_reclaimable", "device_allocated", "host_free", "host_allocated"):
            assert co[k] == cr[k], (k, co, cr)
        assert cr["verify_status"] == 0
        self.ours.verify()
        assert self.ours.dump() == self.ref.dump()


def conv_chunks(cache, conv, kind=None):
    return [r.chunk_id for r in cache.conversation_chunks(conv) if kind is None or r.location == kind]


def test_fuzz_unit_program_matches_reference(reference):
    """proj/tests/test_paged_kv_cache.cpp:293-383, replayed on both caches."""
    P = Pair(reference, 16, 48, 64)
    ours = P.ours
    rng = SplitMix64(20260814)
    now = 0.0
    convs = [1, 2, 3, 4, 5, 6, 7, 8]
    for _ in range(10000):
        now += 0.25
        conv = convs[rng.next() % len(convs)]
        op = rng.next() % 6
        if op == 0:
            add = rng.next() % 40 + 1
            if ours.append_chunks_needed(conv, add) <= ours.counts()["device_free"] + ours.counts()["device_reclaimable"]:
                P.call("allocate", conv, add, now)
        elif op == 1:
            if not ours.has_conversation(conv):
                continue
            dev = conv_chunks(ours, conv, DEVICE)
            if not dev:
                continue
            take = rng.next() % len(dev) + 1
            if take <= ours.counts()["host_free"]:
                P.call("apply_evictions", dev[:take], True)
        elif op == 2:
            host = ours.collect_chunks(HOST)
            if not host:
                continue
            P.call("apply_evictions", host[rng.next() % len(host):], False)
        elif op == 3:
            if not ours.has_conversation(conv):
                continue
            hosted = conv_chunks(ours, conv, HOST)
            avail = ours.counts()["device_free"] + ours.counts()["device_reclaimable"]
            if hosted and len(hosted) <= avail:
                P.call("restore", hosted)
        elif op == 4:
            if not ours.has_conversation(conv):
                continue
            dropped = conv_chunks(ours, conv, DROPPED)
            avail = ours.counts()["device_free"] + ours.counts()["device_reclaimable"]
            if dropped and len(dropped) <= avail:
                P.call("rematerialize", dropped)
        else:
            if not ours.has_conversation(conv):
                continue
            if rng.next() % 4 == 0:
                P.call("release_conversation", conv)
            else:
                P.call("retain_on_finish", conv, now)
        if P.ops % 50 == 0:
            P.check()
    P.check()
    assert P.ops > 5000


def test_fuzz_acceptance_program_matches_reference(reference):
    """proj/tests/acceptance.cpp:550-652 (criterion 10), errors included."""
    P = Pair(reference, 32, 48, 40)
    ours = P.ours
    rng = SplitMix64(4242)
    now = 0.0
    for _ in range(10000):
        now += 0.25
        conv = rng.next() % 8
        op = rng.next() % 6
        if op == 0:
            P.call("allocate", conv, 1 + rng.next() % 64, now)
        elif op == 1:
            if not ours.has_conversation(conv):
                continue
            prefix = []
            for r in ours.conversation_chunks(conv):
                if r.location != DEVICE:
                    break
                prefix.append(r.chunk_id)
                if len(prefix) >= 1 + rng.next() % 3:
                    break
            if prefix:
                P.call("apply_evictions", prefix, True)
        elif op == 2:
            if not ours.has_conversation(conv):
                continue
            hosted = conv_chunks(ours, conv, HOST)
            if len(hosted) > 1:
                hosted = hosted[: 1 + rng.next() % len(hosted)]
            if hosted:
                P.call("apply_evictions", hosted, False)
        elif op == 3:
            if not ours.has_conversation(conv):
                continue
            hosted = conv_chunks(ours, conv, HOST)
            if hosted:
                P.call("restore", hosted)
        elif op == 4:
            if not ours.has_conversation(conv):
                continue
            dropped = conv_chunks(ours, conv, DROPPED)
            if dropped:
                P.call("rematerialize", dropped)
        else:
            if not ours.has_conversation(conv):
                continue
            if rng.next() % 4 == 0:
                P.call("release_conversation", conv)
            else:
                P.call("retain_on_finish", conv, now)
        if P.ops % 50 == 0:
            P.check()
    P.check()


def test_block_tables_match_reference_after_churn(reference):
    P = Pair(reference, 16, 64, 64)
    rng = SplitMix64(77)
    now = 0.0
    for step in range(600):
        now += 1.0
        conv = rng.next() % 6
        P.call("allocate", conv, 1 + rng.next() % 50, now)
        if step % 7 == 3 and P.ours.has_conversation(conv):
            dev = conv_chunks(P.ours, conv, DEVICE)[:2]
            if dev:
                P.call("apply_evictions", dev, rng.next() % 2 == 0)
        if step % 11 == 5:
            for cv in range(6):
                if P.ours.has_conversation(cv):
                    hosted = conv_chunks(P.ours, cv, HOST)
                    if hosted:
                        P.call("restore", hosted)
                    dropped = conv_chunks(P.ours, cv, DROPPED)
                    if dropped:
                        P.call("rematerialize", dropped)
        for cv in range(6):
            if P.ours.has_conversation(cv):
                P.call("block_table", cv, P.ours.total_tokens(cv))
        if step % 97 == 96:
            for cv in range(6):
                if P.ours.has_conversation(cv) and rng.next() % 3 == 0:
                    P.call("release_conversation", cv)
    P.check()
