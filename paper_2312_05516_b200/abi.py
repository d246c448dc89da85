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

PB_F32 = 0
PB_BF16 = 1

PB_PLAN_SINGLE_TOKEN = 1
PB_PLAN_FORCE_SIMT = 2
PB_PLAN_NO_SPLIT = 4


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


class AttnShape(ctypes.Structure):
    _fields_ = [
        ("n_head", ctypes.c_int32),
        ("n_kv_head", ctypes.c_int32),
        ("head_size", ctypes.c_int32),
        ("chunk_size", ctypes.c_int32),
        ("n_slots", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("scale", ctypes.c_double),
    ]


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


def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    if a is None:
        return None
    return a.ctypes.data


def launch_count() -> int:
    return int(lib.pb_launch_count())


class Batch:
    """Ragged query batch descriptors: the SubRequest list of include/kvsim/batch.hpp:17-24
    (query_start, query_len, context_len, causal_offset, block_table) as CSR arrays."""

    def __init__(self, query_len, causal_offset, block_tables: Sequence[Sequence[int]],
                 query_start=None, context_len=None):
        self.query_len = np.ascontiguousarray(query_len, dtype=np.int64)
        self.causal_offset = np.ascontiguousarray(causal_offset, dtype=np.int64)
        n = len(self.query_len)
        if query_start is None:
            query_start = np.zeros(n, dtype=np.int64)
            if n:
                query_start[1:] = np.cumsum(self.query_len)[:-1]
        self.query_start = np.ascontiguousarray(query_start, dtype=np.int64)
        if context_len is None:
            context_len = self.causal_offset + self.query_len
        self.context_len = np.ascontiguousarray(context_len, dtype=np.int64)
        tables = [np.asarray(t, dtype=np.int32) for t in block_tables]
        self.bt_off = np.zeros(n + 1, dtype=np.int64)
        for i, t in enumerate(tables):
            self.bt_off[i + 1] = self.bt_off[i] + len(t)
        self.bt = np.ascontiguousarray(np.concatenate(tables) if tables else np.zeros(0, np.int32),
                                       dtype=np.int32)
        if self.bt.size == 0:
            self.bt = np.zeros(1, dtype=np.int32)  # keep a valid pointer
        self.total_tokens = int(self.query_len.sum()) if n else 0

    @property
    def n_spans(self) -> int:
        return len(self.query_len)

    def table(self, i: int) -> np.ndarray:
        return self.bt[self.bt_off[i]:self.bt_off[i + 1]]

    def args(self):
        return (self.n_spans, _ptr(self.query_start), _ptr(self.query_len), _ptr(self.context_len),
                _ptr(self.causal_offset), _ptr(self.bt), _ptr(self.bt_off))


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

    def check_numerics(self, q: int, k_pages: int, d_flag: int, stream: Optional[int] = None) -> None:
        check(lib.pb_attn_check_numerics(self._h, q, k_pages, d_flag, stream))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
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
