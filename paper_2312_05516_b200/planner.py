"""ctypes binding of the step planner (pb_sched_*), the reference Scheduler over pb_kv_cache."""
from __future__ import annotations

import ctypes
from typing import List

import numpy as np

from . import abi
from .abi import SlotMove, check, lib

_P, _I32, _I64, _D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class SchedParams(ctypes.Structure):
    _fields_ = [("split_mode", _I32), ("policy", _I32), ("stateful", _I32), ("token_budget", _I64),
                ("swap_threshold", _D), ("reserve_fraction", _D)]


_SIGS = {
    "pb_sched_default_params": (None, [ctypes.POINTER(SchedParams)]),
    "pb_sched_create_synthetic": (_I32, [_P, _D, _D, _D, ctypes.POINTER(SchedParams), ctypes.POINTER(_P)]),
    "pb_sched_destroy": (None, [_P]),
    "pb_sched_enqueue": (_I32, [_P, _I64, _I64, _I32, _D, _I64, _I64]),
    "pb_sched_append_history": (_I32, [_P, _I64, _I64]),
    "pb_sched_step": (_I32, [_P, _D, ctypes.POINTER(_I32)]),
    "pb_sched_plan_info": (_I32, [_P, _I32, _P]),
    "pb_sched_plan_spans": (_I32, [_P, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "pb_sched_plan_moves": (_I32, [_P, _I32, _P, _P]),
    "pb_sched_complete": (_I32, [_P, _I32, _D, _P, _I64, ctypes.POINTER(_I64)]),
    "pb_sched_plan_request": (_I32, [_P, _I64, _I64, _I64, _I64, _I64, _I32, _P, _P, _I64]),
    "pb_sched_queue_size": (_I64, [_P]),
    "pb_sched_running_size": (_I64, [_P]),
}
for _n, (_r, _a) in _SIGS.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a
abi._SIGS.update(_SIGS)


def default_params(**kw) -> SchedParams:
    p = SchedParams()
    lib.pb_sched_default_params(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class Plan:
    def __init__(self, spans, swap_in_moves, swap_out_moves, recompute_tokens, total_tokens):
        self.spans = spans  # list of (req_id, query_start, query_len, context_len, causal_offset, table)
        self.in_moves = swap_in_moves
        self.out_moves = swap_out_moves
        self.recompute_tokens = recompute_tokens
        self.total_tokens = total_tokens

    def batch(self) -> abi.Batch:
        return abi.Batch([s[2] for s in self.spans], [s[4] for s in self.spans], [s[5] for s in self.spans])


class Scheduler:
    """pb_scheduler over a KvCache; the cache object must outlive the scheduler."""

    def __init__(self, cache: abi.KvCache, k_attn=5e-7, c_other=9.6e-4, per_token_other=3e-5,
                 params: SchedParams = None):
        self.cache = cache
        h = _P()
        check(lib.pb_sched_create_synthetic(cache._h, k_attn, c_other, per_token_other,
                                            ctypes.byref(params or default_params()), ctypes.byref(h)))
        self._h = h
        self.n_plans = 0

    def __del__(self):
        if getattr(self, "_h", None):
            lib.pb_sched_destroy(self._h)
            self._h = None

    def enqueue(self, req_id, conv_id, arrival, prompt, output, turn=0):
        check(lib.pb_sched_enqueue(self._h, req_id, conv_id, turn, arrival, prompt, output))

    def append_history(self, conv, tokens):
        check(lib.pb_sched_append_history(self._h, conv, tokens))

    def step(self, now: float) -> List[Plan]:
        n = _I32()
        check(lib.pb_sched_step(self._h, now, ctypes.byref(n)))
        self.n_plans = n.value
        return [self._plan(i) for i in range(n.value)]

    def _plan(self, i) -> Plan:
        info = np.zeros(8, np.int64)
        check(lib.pb_sched_plan_info(self._h, i, info.ctypes.data))
        ns, ntok, nbt, _, _, rec, nin, nout = (int(x) for x in info)
        arrs = [np.zeros(max(1, ns), np.int64) for _ in range(5)]
        bt = np.zeros(max(1, nbt), np.int32)
        off = np.zeros(ns + 1, np.int64)
        check(lib.pb_sched_plan_spans(self._h, i, *[a.ctypes.data for a in arrs], bt.ctypes.data, off.ctypes.data))
        spans = [(int(arrs[0][k]), int(arrs[1][k]), int(arrs[2][k]), int(arrs[3][k]), int(arrs[4][k]),
                  bt[off[k]:off[k + 1]].tolist()) for k in range(ns)]
        mi = (SlotMove * max(1, nin))()
        mo = (SlotMove * max(1, nout))()
        check(lib.pb_sched_plan_moves(self._h, i, mi, mo))
        return Plan(spans, [(m.chunk, m.src_slot, m.dst_slot) for m in mi[:nin]],
                    [(m.chunk, m.src_slot, m.dst_slot) for m in mo[:nout]], rec, ntok)

    def complete(self, plan_index: int, end_time: float) -> List[int]:
        out = np.zeros(4096, np.int64)
        n = _I64()
        check(lib.pb_sched_complete(self._h, plan_index, end_time, out.ctypes.data, out.size, ctypes.byref(n)))
        return out[: n.value].tolist()

    def plan_request(self, req_id, conv_id, prompt, output, generated=0, suspended=False):
        info = np.zeros(9, np.int64)
        spans = np.zeros(3 * 64, np.int64)
        check(lib.pb_sched_plan_request(self._h, req_id, conv_id, prompt, output, generated, 1 if suspended else 0,
                                        info.ctypes.data, spans.ctypes.data, 64))
        keys = ("input_tokens", "recompute_tokens", "pending_tokens", "n_rematerialize", "n_swap_in",
                "append_slots", "device_hit_tokens", "host_hit_tokens", "n_spans")
        d = dict(zip(keys, (int(x) for x in info)))
        d["spans"] = [tuple(int(x) for x in spans[3 * k:3 * k + 3]) for k in range(d["n_spans"])]
        return d

    @property
    def queue_size(self):
        return int(lib.pb_sched_queue_size(self._h))

    @property
    def running_size(self):
        return int(lib.pb_sched_running_size(self._h))
