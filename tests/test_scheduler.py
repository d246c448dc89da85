"""Step planner (pb_sched_*): the reference Scheduler's span construction and batch assembly.

* the reference's own cases (proj/tests/test_scheduler.cpp:96-178, :393-462) re-run;
* differential simulation: a multi-turn workload under memory pressure is driven through our
  planner and through the UNMODIFIED reference Scheduler (oracle/_ref) step by step; every
  plan's spans, block tables, swap-in (chunk, slot) list, swap-out list and finished set, and
  the cache dump after every step, must be identical.
"""
import ctypes

import numpy as np
import pytest

from paper_2312_05516_b200.abi import KvCache
from paper_2312_05516_b200.planner import Scheduler, default_params
from paper_2312_05516_b200.workloads import SplitMix64


def rig(chunk=32, dev=64, host=32, **kw):
    cache = KvCache(chunk, dev, host)
    return cache, Scheduler(cache, params=default_params(**kw))


def test_plan_splits_returning_context_into_recompute_and_prompt():
    # proj/tests/test_scheduler.cpp:96-125 (also PAPER.md:654-660)
    cache, s = rig()
    cache.allocate(1, 320, 0.0)
    ids = [r.chunk_id for r in cache.conversation_chunks(1)]
    cache.apply_evictions(ids[:5], True)
    cache.apply_evictions(ids[:2], False)
    s.enqueue(999, 1, 0.0, 1, 1)  # registers the conversation (enqueue ensures it)
    s.append_history(1, 320)
    p = s.plan_request(10, 1, 40, 8)
    assert (p["input_tokens"], p["recompute_tokens"], p["pending_tokens"]) == (104, 64, 40)
    assert (p["n_rematerialize"], p["n_swap_in"]) == (2, 3)
    assert (p["device_hit_tokens"], p["host_hit_tokens"]) == (160, 96)
    assert p["spans"] == [(64, 64, 0), (40, 360, 320)]
    assert p["append_slots"] == 2


def test_plans_without_dropped_history_and_fresh_conversations():
    cache, s = rig()
    cache.allocate(1, 320, 0.0)
    s.enqueue(999, 1, 0.0, 1, 1)
    s.append_history(1, 320)
    assert s.plan_request(10, 1, 40, 8)["spans"] == [(40, 360, 320)]
    p = s.plan_request(10, 7, 40, 8)
    assert p["spans"] == [(40, 40, 0)] and p["append_slots"] == 2


def test_missing_suffix_merges_into_prompt_span():
    # proj/tests/test_scheduler.cpp:140-155
    cache, s = rig()
    cache.allocate(1, 64, 0.0)
    s.enqueue(999, 1, 0.0, 1, 1)
    s.append_history(1, 96)
    p = s.plan_request(11, 1, 40, 8)
    assert p["recompute_tokens"] == 32 and p["input_tokens"] == 72
    assert p["spans"] == [(72, 136, 64)] and p["append_slots"] == 3


def test_finish_bonus_preallocates_the_final_token():
    cache, s = rig()
    assert s.plan_request(10, 7, 32, 1)["append_slots"] == 2
    assert s.plan_request(11, 8, 32, 2)["append_slots"] == 1


def test_unified_build_batch_layout():
    # proj/tests/test_scheduler.cpp:393-432
    cache, s = rig()
    s.enqueue(1, 1, 0.0, 100, 50)
    s.enqueue(2, 2, 0.0, 200, 50)
    for i, _ in enumerate(s.step(0.5)):
        s.complete(i, 0.55)
    s.enqueue(3, 3, 1.0, 40, 50)
    plans = s.step(1.0)
    assert len(plans) == 1
    sp = plans[0].spans
    assert plans[0].total_tokens == 42
    assert [(x[0], x[1], x[2], x[4], len(x[5])) for x in sp] == [(3, 0, 40, 0, 2), (1, 40, 1, 100, 4), (2, 41, 1, 200, 7)]
    assert sp[1][3] == 101 and sp[2][3] == 201


def test_split_mode_two_plans():
    cache, s = rig(split_mode=1)
    s.enqueue(1, 1, 0.0, 100, 50)
    s.enqueue(2, 2, 0.0, 200, 50)
    for i, _ in enumerate(s.step(0.5)):
        s.complete(i, 0.55)
    s.enqueue(3, 3, 1.0, 40, 50)
    plans = s.step(1.0)
    assert [len(p.spans) for p in plans] == [1, 2]
    assert [p.total_tokens for p in plans] == [40, 2]


class RefSched:
    def __init__(self, reference, chunk, dev, host, split=0, lru=0, stateful=1, budget=4096, thr=0.25, res=0.10):
        L = reference.L
        P, I, LL, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double
        L.ref_sched_create.restype = P
        L.ref_sched_create.argtypes = [I, I, I, D, D, D, I, I, I, LL, D, D]
        L.ref_sched_destroy.argtypes = [P]
        L.ref_sched_enqueue.restype = I
        L.ref_sched_enqueue.argtypes = [P, LL, LL, I, D, LL, LL]
        L.ref_sched_step.restype = I
        L.ref_sched_step.argtypes = [P, D, ctypes.POINTER(I)]
        L.ref_sched_plan_info.argtypes = [P, I, P]
        L.ref_sched_plan_spans.argtypes = [P, I] + [P] * 10
        L.ref_sched_complete.restype = I
        L.ref_sched_complete.argtypes = [P, I, D, P, LL, ctypes.POINTER(LL)]
        L.ref_sched_dump.restype = I
        L.ref_sched_dump.argtypes = [P, ctypes.c_char_p, LL]
        self.L = L
        self.h = L.ref_sched_create(chunk, dev, host, 5e-7, 9.6e-4, 3e-5, split, lru, stateful, budget, thr, res)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_sched_destroy(self.h)

    def enqueue(self, req, conv, arrival, prompt, output, turn=0):
        assert self.L.ref_sched_enqueue(self.h, req, conv, turn, arrival, prompt, output) == 0

    def step(self, now):
        n = ctypes.c_int()
        st = self.L.ref_sched_step(self.h, now, ctypes.byref(n))
        if st:
            return st, None
        plans = []
        for i in range(n.value):
            info = np.zeros(6, np.int64)
            self.L.ref_sched_plan_info(self.h, i, info.ctypes.data)
            ns, ntok, nbt, nin, nout, rec = (int(x) for x in info)
            a = [np.zeros(max(1, ns), np.int64) for _ in range(5)]
            bt = np.zeros(max(1, nbt), np.int32)
            off = np.zeros(ns + 1, np.int64)
            sic = np.zeros(max(1, nin), np.int64)
            sis = np.zeros(max(1, nin), np.int32)
            so = np.zeros(max(1, nout), np.int64)
            self.L.ref_sched_plan_spans(self.h, i, *[x.ctypes.data for x in a], bt.ctypes.data, off.ctypes.data,
                                        sic.ctypes.data, sis.ctypes.data, so.ctypes.data)
            spans = [(int(a[0][k]), int(a[1][k]), int(a[2][k]), int(a[3][k]), int(a[4][k]), bt[off[k]:off[k + 1]].tolist())
                     for k in range(ns)]
            plans.append((spans, list(zip(sic[:nin].tolist(), sis[:nin].tolist())), so[:nout].tolist(), rec, ntok))
        return 0, plans

    def complete(self, i, t):
        out = np.zeros(4096, np.int64)
        n = ctypes.c_longlong()
        assert self.L.ref_sched_complete(self.h, i, t, out.ctypes.data, out.size, ctypes.byref(n)) == 0
        return out[: n.value].tolist()

    def dump(self):
        buf = ctypes.create_string_buffer(1 << 20)
        self.L.ref_sched_dump(self.h, buf, 1 << 20)
        return buf.value.decode()


@pytest.mark.parametrize("split,lru,stateful", [(0, 0, 1), (1, 0, 1), (0, 1, 1), (0, 0, 0)])
def test_differential_simulation_matches_reference(reference, split, lru, stateful):
    """Multi-turn conversations under device pressure (swap-outs, host overflow drops,
    prefix-drop recompute spans, suspensions): identical plans and cache state every step."""
    chunk, dev, host = 16, 96, 160
    cache = KvCache(chunk, dev, host)
    ours = Scheduler(cache, params=default_params(split_mode=split, policy=lru, stateful=stateful, token_budget=2048))
    ref = RefSched(reference, chunk, dev, host, split=split, lru=lru, stateful=stateful, budget=2048)
    rng = SplitMix64(777 + 10 * split + lru)
    n_conv = 24
    turns = {c: 2 + rng.next() % 3 for c in range(n_conv)}
    arrivals = sorted((0.05 * c + rng.u01() * 0.5, c) for c in range(n_conv))
    pending = [(t, c, 0) for t, c in arrivals]  # (arrival, conv, turn)
    req_conv, next_req = {}, 0
    now, steps, checked = 0.0, 0, 0
    while (pending or ours.queue_size or ours.running_size) and steps < 3000:
        steps += 1
        now += 0.05
        for item in sorted(p for p in pending if p[0] <= now):
            t, c, turn = item
            pending.remove(item)
            prompt = 8 + rng.next() % 120
            output = 2 + rng.next() % 24
            ours.enqueue(next_req, c, t, prompt, output, turn)
            ref.enqueue(next_req, c, t, prompt, output, turn)
            req_conv[next_req] = (c, turn)
            next_req += 1
        try:
            plans = ours.step(now)
            st = 0
        except Exception as e:  # CannotSuspendAll etc. must match the reference
            plans, st = None, getattr(e, "code", -1)
        rst, rplans = ref.step(now)
        assert st == rst, (steps, st, rst)
        if st:
            break
        assert len(plans) == len(rplans)
        for p, (rs, rin, rout, rrec, rtok) in zip(plans, rplans):
            assert p.spans == rs, steps
            assert [(m[0], m[2]) for m in p.in_moves] == rin
            assert [m[0] for m in p.out_moves] == rout
            assert (p.recompute_tokens, p.total_tokens) == (rrec, rtok)
            checked += 1
        for i in range(len(plans)):
            done = ours.complete(i, now + 0.01)
            assert done == ref.complete(i, now + 0.01)
            for rq in done:
                c, turn = req_conv[rq]
                if turn + 1 < turns[c]:
                    pending.append((now + 0.05 + rng.u01() * 0.3, c, turn + 1))
        assert cache.dump() == ref.dump(), steps
    assert checked > 50
