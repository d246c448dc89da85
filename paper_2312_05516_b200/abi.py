"""ctypes binding of include/pensieve_b200.h.

Every wrapper maps a non-OK ``pb_status`` onto the Python analogue of the reference's
exception class (include/kvsim/errors.hpp), so parity tests read like the reference's own
doctest cases (``CHECK_THROWS_AS(..., DimensionMismatch)``).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libpensieve_b200.so")

# descriptor types shared with the host-only modules (no library load there)
from .descriptors import PB_BF16, PB_F32, AttnShape, Batch, _ptr  # noqa: E402,F401

PB_PLAN_SINGLE_TOKEN = 1
PB_PLAN_FORCE_SIMT = 2
PB_PLAN_NO_SPLIT = 4
PB_PLAN_SEPARATE_DECODE = 8
PB_PLAN_LPT_ORDER = 16


class PBError(RuntimeError):
    code = -1


class DimensionMismatch(PBError):
    code = 1


class NumericError(PBError):
    code = 2


class Error(PBError):
    code = 3


class InsufficientDeviceMemory(PBError):
    code = 4


class InsufficientHostMemory(PBError):
    code = 5


class InvalidChunkState(PBError):
    code = 6


class UnknownConversation(PBError):
    code = 7


class ConfigError(PBError):
    code = 8


class NotEnoughEvictable(PBError):
    code = 9


class TraceMissing(PBError):
    code = 10


class CannotSuspendAll(PBError):
    code = 11


class CudaError(PBError):
    code = 20


class Unsupported(PBError):
    code = 21


_ERRORS = {c.code: c for c in (DimensionMismatch, NumericError, Error, InsufficientDeviceMemory,
                               InsufficientHostMemory, InvalidChunkState, UnknownConversation,
                               ConfigError, NotEnoughEvictable, TraceMissing, CannotSuspendAll,
                               CudaError, Unsupported)}


def _load() -> ctypes.CDLL:
    if not os.path.exists(SO_PATH):
        raise ImportError(
            f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    return ctypes.CDLL(SO_PATH)


lib = _load()

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_DP = ctypes.POINTER(ctypes.c_double)
_SHP = ctypes.POINTER(AttnShape)

_SIGS = {
    "pb_last_error": (ctypes.c_char_p, []),
    "pb_version": (ctypes.c_char_p, []),
    "pb_launch_count": (_U64, []),
    "pb_attn_plan_create": (_I32, [_SHP, _I32, _P, _P, _P, _P, _P, _P, _I64, _I32, ctypes.POINTER(_P)]),
    "pb_attn_plan_upload": (_I32, [_P, _P]),
    "pb_attn_plan_workspace_bytes": (ctypes.c_size_t, [_P]),
    "pb_attn_plan_stats": (None, [_P, _DP]),
    "pb_attn_run": (_I32, [_P, _P, _P, _P, _P, _P, _P]),
    "pb_attn_stage_bytes": (ctypes.c_size_t, [_P]),
    "pb_attn_run_append": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pb_attn_set_trace": (None, [_P, _P]),
    "pb_attn_run_layers_host": (_I32, [_P, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "pb_attn_run_layers": (_I32, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    "pb_attn_check_numerics": (_I32, [_P, _P, _P, _P, _P]),
    "pb_attn_plan_destroy": (None, [_P]),
    "pb_paged_multi_token_attention": (_I32, [_SHP, _I32, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P]),
    "pb_single_token_attention": (_I32, [_SHP, _I32, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P]),
    "pb_kv_gather_pages": (_I32, [_P, _I64, _I32, _I64, _P, _I64, _P, _I32, _P]),
    "pb_kv_scatter_pages": (_I32, [_P, _I64, _I32, _I64, _P, _I64, _P, _I32, _P]),
    "pb_kv_append": (_I32, [_SHP, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pb_fill_splitmix_unit": (_I32, [_P, _I32, _I64, _U64, _U64, _P]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def check(status: int) -> None:
    if status != 0:
        msg = lib.pb_last_error().decode(errors="replace")
        raise _ERRORS.get(status, PBError)(f"pb status {status}: {msg}")


def exported_symbols() -> Sequence[str]:
    return list(_SIGS)


def launch_count() -> int:
    return int(lib.pb_launch_count())


class AttentionPlan:
    """pb_attn_plan: validated batch + work list, reusable across layers."""

    def __init__(self, shape: AttnShape, batch: Batch, flags: int = 0):
        self.shape = shape
        self.batch = batch
        h = _P()
        check(lib.pb_attn_plan_create(ctypes.byref(shape), *batch.args(), batch.total_tokens, flags,
                                      ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def upload(self, stream: Optional[int] = None) -> None:
        check(lib.pb_attn_plan_upload(self._h, stream))

    def workspace_bytes(self) -> int:
        return int(lib.pb_attn_plan_workspace_bytes(self._h))

    def stats(self) -> dict:
        o = (ctypes.c_double * 8)()
        lib.pb_attn_plan_stats(self._h, o)
        return {"prefill_tiles": int(o[0]), "decode_units": int(o[1]), "split_spans": int(o[2]),
                "flops": o[3], "bytes": o[4], "total_tokens": int(o[5]), "simt_tiles": int(o[6]),
                "rows": int(o[7])}

    def run(self, q: int, k_pages: int, v_pages: int, out: int, workspace: Optional[int],
            stream: Optional[int] = None) -> None:
        check(lib.pb_attn_run(self._h, q, k_pages, v_pages, out, workspace, stream))

    def run_append(self, q: int, k_new: int, v_new: int, k_pages: int, v_pages: int, out: int,
                   workspace: Optional[int], stream: Optional[int] = None) -> None:
        """pb_attn_run_append: write the batch's new K/V rows into the pages, then attend."""
        check(lib.pb_attn_run_append(self._h, q, k_new, v_new, k_pages, v_pages, out, workspace, stream))

    def run_layers(self, q: Sequence[int], k_pages: Sequence[int], v_pages: Sequence[int],
                   out: Sequence[int], workspace: Optional[int], stream: Optional[int] = None) -> None:
        """pb_attn_run_layers: the layer loop as one CUDA graph launch (captured on first use,
        replayed while the pointers stay the same)."""
        n = len(q)
        if not (len(k_pages) == len(v_pages) == len(out) == n):
            raise DimensionMismatch("per-layer pointer lists differ in length")
        arr = ctypes.c_void_p * n
        keep = (arr(*q), arr(*k_pages), arr(*v_pages), arr(*out))
        check(lib.pb_attn_run_layers(self._h, n, *[ctypes.cast(a, _P) for a in keep], workspace, stream))

    def set_trace(self, d_trace: Optional[int]) -> None:
        lib.pb_attn_set_trace(self._h, d_trace)

    def stage_bytes(self) -> int:
        return int(lib.pb_attn_stage_bytes(self._h))

    def run_layers_host(self, q_host: Sequence[int], out_host: Sequence[int], k_pages: Sequence[int],
                        v_pages: Sequence[int], staging: int, workspace: Optional[int],
                        stream: Optional[int] = None) -> None:
        """pb_attn_run_layers_host: per-layer host q / out, copies overlapped with compute."""
        n = len(q_host)
        arr = ctypes.c_void_p * n
        self._io_keep = (arr(*q_host), arr(*out_host), arr(*k_pages), arr(*v_pages))
        check(lib.pb_attn_run_layers_host(self._h, n, *[ctypes.cast(a, _P) for a in self._io_keep], staging,
                                          workspace, stream))

    def check_numerics(self, q: int, k_pages: int, d_flag: int, stream: Optional[int] = None) -> None:
        check(lib.pb_attn_check_numerics(self._h, q, k_pages, d_flag, stream))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.pb_attn_plan_destroy(h)
            self._h = None


def _one_shot(fn, shape: AttnShape, batch: Batch, q: np.ndarray, keys: np.ndarray,
              values: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.float32)
    keys = np.ascontiguousarray(keys, dtype=np.float32)
    values = np.ascontiguousarray(values, dtype=np.float32)
    out = np.zeros_like(q)
    check(fn(ctypes.byref(shape), *batch.args(), _ptr(q), batch.total_tokens, _ptr(keys),
             _ptr(values), _ptr(out)))
    return out


def paged_multi_token_attention(shape: AttnShape, batch: Batch, q, keys, values) -> np.ndarray:
    """Host-buffer mirror of kvsim::paged_multi_token_attention (attention.hpp:71-72)."""
    return _one_shot(lib.pb_paged_multi_token_attention, shape, batch, q, keys, values)


def single_token_attention(shape: AttnShape, batch: Batch, q, keys, values) -> np.ndarray:
    """Host-buffer mirror of kvsim::single_token_attention (attention.hpp:76-77)."""
    return _one_shot(lib.pb_single_token_attention, shape, batch, q, keys, values)


def gather_pages(pool: int, layer_stride: int, n_layers: int, page_bytes: int, d_slots: int,
                 n: int, staging: int, layer_major: int = 0, stream: Optional[int] = None) -> None:
    check(lib.pb_kv_gather_pages(pool, layer_stride, n_layers, page_bytes, d_slots, n, staging,
                                 layer_major, stream))


def scatter_pages(staging: int, layer_stride: int, n_layers: int, page_bytes: int, d_slots: int,
                  n: int, pool: int, layer_major: int = 0, stream: Optional[int] = None) -> None:
    check(lib.pb_kv_scatter_pages(staging, layer_stride, n_layers, page_bytes, d_slots, n, pool,
                                  layer_major, stream))


def fill_unit(dst: int, dtype: int, n: int, seed: int, first_draw: int,
              stream: Optional[int] = None) -> None:
    check(lib.pb_fill_splitmix_unit(dst, dtype, n, seed, first_draw, stream))


# ============================================================================ model bytes, shards
class ModelConfig(ctypes.Structure):
    """pb_model_config: kvsim::ModelConfig's integer fields (include/kvsim/model_config.hpp)."""
    _fields_ = [("n_layer", _I32), ("hidden", _I32), ("n_head", _I32), ("n_kv_head", _I32),
                ("head_size", _I32), ("bytes_per_scalar", _I32), ("n_partitions", _I32)]


_MODEL_SIGS = {
    "pb_model_validate": (_I32, [ctypes.POINTER(ModelConfig)]),
    "pb_model_kv_token_bytes": (_I32, [ctypes.POINTER(ModelConfig), ctypes.POINTER(ctypes.c_uint64)]),
    "pb_model_chunk_bytes": (_I32, [ctypes.POINTER(ModelConfig), _I32, ctypes.POINTER(ctypes.c_uint64)]),
    "pb_model_preset": (_I32, [ctypes.c_char_p, ctypes.POINTER(ModelConfig)]),
    "pb_shard_shape": (_I32, [_SHP, _I32, _I32, _SHP, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
}
for _name, (_res, _args) in _MODEL_SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
_SIGS.update(_MODEL_SIGS)


def model_preset(name: str) -> ModelConfig:
    m = ModelConfig()
    check(lib.pb_model_preset(name.encode(), ctypes.byref(m)))
    return m


def model_validate(m: ModelConfig) -> None:
    check(lib.pb_model_validate(ctypes.byref(m)))


def kv_token_bytes(m: ModelConfig) -> int:
    out = ctypes.c_uint64()
    check(lib.pb_model_kv_token_bytes(ctypes.byref(m), ctypes.byref(out)))
    return int(out.value)


def chunk_bytes(m: ModelConfig, chunk_size: int) -> int:
    out = ctypes.c_uint64()
    check(lib.pb_model_chunk_bytes(ctypes.byref(m), chunk_size, ctypes.byref(out)))
    return int(out.value)


def shard_shape(shape: AttnShape, rank: int, world: int):
    """pb_shard_shape: (shard AttnShape, first query head, first kv head) of rank / world."""
    out, h0, k0 = AttnShape(), _I32(), _I32()
    check(lib.pb_shard_shape(ctypes.byref(shape), rank, world, ctypes.byref(out), ctypes.byref(h0),
                             ctypes.byref(k0)))
    return out, int(h0.value), int(k0.value)


# ============================================================================ KV bookkeeping
class SlotMove(ctypes.Structure):
    _fields_ = [("chunk", ctypes.c_int64), ("src_slot", ctypes.c_int32), ("dst_slot", ctypes.c_int32)]


class ChunkRecord(ctypes.Structure):
    _fields_ = [("chunk_id", ctypes.c_int64), ("conv_id", ctypes.c_int64), ("start_offset", ctypes.c_int64),
                ("n_tokens", ctypes.c_int64), ("location", ctypes.c_int32), ("slot", ctypes.c_int32),
                ("last_active", ctypes.c_double)]


class LayoutSegment(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_chunks", ctypes.c_int32), ("token_begin", ctypes.c_int64),
                ("token_end", ctypes.c_int64), ("first_chunk", ctypes.c_int64)]


DEVICE, HOST, DROPPED = 0, 1, 2

_I64P = ctypes.POINTER(_I64)
_CACHE_SIGS = {
    "pb_cache_create": (_I32, [_I32, _I32, _I32, ctypes.POINTER(_P)]),
    "pb_cache_destroy": (None, [_P]),
    "pb_cache_allocate": (_I32, [_P, _I64, _I64, ctypes.c_double, _P, _I64, _I64P]),
    "pb_cache_apply_evictions": (_I32, [_P, _P, _I64, _I32, _P]),
    "pb_cache_restore": (_I32, [_P, _P, _I64, _P]),
    "pb_cache_rematerialize": (_I32, [_P, _P, _I64, _P]),
    "pb_cache_release_conversation": (_I32, [_P, _I64]),
    "pb_cache_touch": (_I32, [_P, _I64, ctypes.c_double]),
    "pb_cache_block_table": (_I32, [_P, _I64, _I64, _P, _I64, _I64P]),
    "pb_cache_layout": (_I32, [_P, _I64, _P, _I64, _I64P, _I64P]),
    "pb_cache_conversation_chunks": (_I32, [_P, _I64, _P, _I64, _I64P]),
    "pb_cache_chunk": (_I32, [_P, _I64, _P]),
    "pb_cache_collect_chunks": (_I32, [_P, _I32, _P, _I64, _P, _I64, _I64P]),
    "pb_cache_counts": (None, [_P, _P]),
    "pb_cache_has_conversation": (_I32, [_P, _I64]),
    "pb_cache_total_tokens": (_I64, [_P, _I64]),
    "pb_cache_append_chunks_needed": (_I32, [_P, _I64, _I64]),
    "pb_cache_verify": (_I32, [_P]),
    "pb_cache_dump": (_I64, [_P, ctypes.c_char_p, _I64]),
}
for _name, (_res, _args) in _CACHE_SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
_SIGS.update(_CACHE_SIGS)


def _ids(ids) -> np.ndarray:
    return np.ascontiguousarray(ids, dtype=np.int64)


class KvCache:
    """pb_kv_cache: the two-tier page-slot allocator (kvsim::PagedKvCache semantics)."""

    def __init__(self, chunk_size: int, device_slots: int, host_slots: int):
        h = _P()
        check(lib.pb_cache_create(chunk_size, device_slots, host_slots, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.pb_cache_destroy(h)
            self._h = None

    def allocate(self, conv: int, n_tokens: int, now: float):
        cap = max(1, n_tokens // 1 + 1)
        out = np.zeros(min(cap, 1 << 20), np.int64)
        n = _I64()
        check(lib.pb_cache_allocate(self._h, conv, n_tokens, now, out.ctypes.data, out.size, ctypes.byref(n)))
        return out[: n.value].tolist()

    def _moves(self, fn, ids, *extra):
        ids = _ids(ids)
        moves = (SlotMove * max(1, len(ids)))()
        check(fn(self._h, ids.ctypes.data if len(ids) else None, len(ids), *extra, moves))
        return [(m.chunk, m.src_slot, m.dst_slot) for m in moves[: len(ids)]]

    def apply_evictions(self, ids, to_host: bool):
        ids = _ids(ids)
        moves = (SlotMove * max(1, len(ids)))()
        check(lib.pb_cache_apply_evictions(self._h, ids.ctypes.data if len(ids) else None, len(ids),
                                           1 if to_host else 0, moves))
        return [(m.chunk, m.src_slot, m.dst_slot) for m in moves[: len(ids)]]

    def restore(self, ids):
        return self._moves(lib.pb_cache_restore, ids)

    def rematerialize(self, ids):
        return self._moves(lib.pb_cache_rematerialize, ids)

    def release_conversation(self, conv):
        check(lib.pb_cache_release_conversation(self._h, conv))

    def touch(self, conv, now):
        check(lib.pb_cache_touch(self._h, conv, now))

    retain_on_finish = touch

    def block_table(self, conv, ctx):
        out = np.zeros(max(1, ctx // 1 + 1), np.int32)
        n = _I64()
        check(lib.pb_cache_block_table(self._h, conv, ctx, out.ctypes.data, out.size, ctypes.byref(n)))
        return out[: n.value].tolist()

    def layout(self, conv):
        segs = (LayoutSegment * 4096)()
        n, total = _I64(), _I64()
        check(lib.pb_cache_layout(self._h, conv, segs, 4096, ctypes.byref(n), ctypes.byref(total)))
        return total.value, [(s.kind, s.token_begin, s.token_end, s.n_chunks) for s in segs[: n.value]]

    def conversation_chunks(self, conv):
        n = _I64()
        check(lib.pb_cache_conversation_chunks(self._h, conv, None, 0, ctypes.byref(n)))
        recs = (ChunkRecord * max(1, n.value))()
        check(lib.pb_cache_conversation_chunks(self._h, conv, recs, n.value, ctypes.byref(n)))
        return list(recs[: n.value])

    def chunk(self, cid) -> ChunkRecord:
        r = ChunkRecord()
        check(lib.pb_cache_chunk(self._h, cid, ctypes.byref(r)))
        return r

    def collect_chunks(self, location, exclude=()):
        ex = _ids(list(exclude) or [0])
        out = np.zeros(1 << 16, np.int64)
        n = _I64()
        check(lib.pb_cache_collect_chunks(self._h, location, ex.ctypes.data, len(exclude), out.ctypes.data,
                                          out.size, ctypes.byref(n)))
        return out[: n.value].tolist()

    def counts(self):
        o = np.zeros(8, np.int64)
        lib.pb_cache_counts(self._h, o.ctypes.data)
        keys = ("device_capacity", "device_free", "device_reclaimable", "device_allocated", "host_capacity",
                "host_free", "host_allocated", "chunk_size")
        return dict(zip(keys, (int(x) for x in o)))

    def has_conversation(self, conv) -> bool:
        return bool(lib.pb_cache_has_conversation(self._h, conv))

    def total_tokens(self, conv) -> int:
        return int(lib.pb_cache_total_tokens(self._h, conv))

    def append_chunks_needed(self, conv, add) -> int:
        return int(lib.pb_cache_append_chunks_needed(self._h, conv, add))

    def verify(self):
        check(lib.pb_cache_verify(self._h))

    def dump(self) -> str:
        n = lib.pb_cache_dump(self._h, None, 0)
        buf = ctypes.create_string_buffer(int(n) + 1)
        lib.pb_cache_dump(self._h, buf, n + 1)
        return buf.value.decode()


# ============================================================================ swap engine
_TIER_SIGS = {
    "pb_tier_create": (_I32, [_I32, _I32, _I64, _I32, ctypes.POINTER(_P)]),
    "pb_tier_destroy": (None, [_P]),
    "pb_tier_host_base": (_P, [_P]),
    "pb_tier_chunk_bytes": (_I64, [_P]),
    "pb_swap_step": (_I32, [_P, _P, _P, _I64, _P, _I64, _P, _I64, _P, _P]),
    "pb_swap_wait_layer": (_I32, [_P, _I32, _P]),
    "pb_swap_sync": (_I32, [_P]),
    "pb_tier_set_event_log": (_I32, [_P, _P]),
    "pb_tier_set_policy": (_I32, [_P, _I32, _I32, _I32]),
    "pb_evlog_create": (_I32, [_I64, ctypes.POINTER(_P)]),
    "pb_evlog_destroy": (None, [_P]),
    "pb_evlog_mark": (_I32, [_P, _I32, _I32, _I64, _P]),
    "pb_evlog_read": (_I32, [_P, _P, _I64, ctypes.POINTER(_I64)]),
    "pb_evlog_reset": (_I32, [_P]),
    "pb_evlog_audit": (_I32, [_P, _I64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]),
    "pb_evlog_audit_steps": (_I32, [_P, _I64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]),
}
for _name, (_res, _args) in _TIER_SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
_SIGS.update(_TIER_SIGS)


def _moves_array(moves):
    arr = (SlotMove * max(1, len(moves)))()
    for i, (c, s, d) in enumerate(moves):
        arr[i].chunk, arr[i].src_slot, arr[i].dst_slot = c, s, d
    return arr


PB_EV_SWAP_IN_LAYER, PB_EV_SWAP_OUT, PB_EV_ATTN_START, PB_EV_STEP_END = 0, 1, 2, 3
EVENT_DTYPE = np.dtype([("t_ns", np.int64), ("kind", np.int32), ("layer", np.int32), ("req", np.int64)])


def audit_events(events: np.ndarray, per_step: bool = False):
    """pb_evlog_audit: LayerDependencyAuditor (src/event_log.cpp:90-118) over records of
    EVENT_DTYPE (per_step: pb_evlog_audit_steps).  Returns (violations, steps)."""
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    v, st = ctypes.c_uint64(), ctypes.c_uint64()
    fn = lib.pb_evlog_audit_steps if per_step else lib.pb_evlog_audit
    check(fn(ev.ctypes.data if len(ev) else None, len(ev), ctypes.byref(v), ctypes.byref(st)))
    return int(v.value), int(st.value)


class EventLog:
    """pb_event_log: device-timestamped pipeline events."""

    def __init__(self, capacity: int = 1 << 16):
        h = _P()
        check(lib.pb_evlog_create(capacity, ctypes.byref(h)))
        self._h = h
        self.capacity = capacity

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.pb_evlog_destroy(h)
            self._h = None

    def mark(self, kind: int, layer: int = -1, req: int = -1, stream: Optional[int] = None) -> None:
        check(lib.pb_evlog_mark(self._h, kind, layer, req, stream))

    def read(self) -> np.ndarray:
        n = ctypes.c_int64()
        out = np.zeros(self.capacity, dtype=EVENT_DTYPE)
        check(lib.pb_evlog_read(self._h, out.ctypes.data, self.capacity, ctypes.byref(n)))
        return out[: n.value]

    def reset(self) -> None:
        check(lib.pb_evlog_reset(self._h))


PB_SWAP_IN_STAGED, PB_SWAP_IN_ZERO_COPY = 0, 1
PB_D2H_ON_COPY_STREAM, PB_D2H_CONCURRENT, PB_D2H_AFTER_SWAP_IN = 0, 1, 2


class KvTier:
    """pb_kv_tier: pinned host tier + ordered, layer-pipelined swap copies."""

    def __init__(self, n_layer: int, host_slots: int, page_bytes: int, max_chunks_per_step: int):
        h = _P()
        check(lib.pb_tier_create(n_layer, host_slots, page_bytes, max_chunks_per_step, ctypes.byref(h)))
        self._h = h
        self.n_layer, self.host_slots, self.page_bytes = n_layer, host_slots, page_bytes

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.pb_tier_destroy(h)
            self._h = None

    @property
    def chunk_bytes(self) -> int:
        return int(lib.pb_tier_chunk_bytes(self._h))

    def host_view(self) -> np.ndarray:
        """The pinned host tier as a numpy byte array [host_slot][layer][K|V][page]."""
        base = lib.pb_tier_host_base(self._h)
        buf = (ctypes.c_uint8 * (self.host_slots * self.chunk_bytes)).from_address(base)
        return np.frombuffer(buf, dtype=np.uint8)

    def step(self, k_pool: int, v_pool: int, layer_stride: int, out_moves, in_moves,
             compute_stream: Optional[int] = None, copy_stream: Optional[int] = None) -> None:
        om, im = _moves_array(out_moves), _moves_array(in_moves)
        check(lib.pb_swap_step(self._h, k_pool, v_pool, layer_stride, om, len(out_moves), im, len(in_moves),
                               compute_stream, copy_stream))

    def set_policy(self, swap_in: int = PB_SWAP_IN_STAGED, d2h: int = PB_D2H_AFTER_SWAP_IN,
                   layers_per_piece: int = 0) -> None:
        """pb_tier_set_policy: transfer method / D2H ordering (defaults are the measured best)."""
        check(lib.pb_tier_set_policy(self._h, swap_in, d2h, layers_per_piece))

    def set_event_log(self, log: Optional["EventLog"]) -> None:
        self._log = log
        check(lib.pb_tier_set_event_log(self._h, log._h if log is not None else None))

    def wait_layer(self, layer: int, compute_stream: Optional[int] = None) -> None:
        check(lib.pb_swap_wait_layer(self._h, layer, compute_stream))

    def sync(self) -> None:
        check(lib.pb_swap_sync(self._h))
