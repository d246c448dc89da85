"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
import this module.  ``Oracle`` wraps our C restatement (liboracle.so, attn_oracle.c);
``Reference`` wraps the unmodified reference library built into _ref/ by the Makefile.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkvsim_ref.so")

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_D = ctypes.c_double


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    return None if a is None else a.ctypes.data


class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        L.oracle_splitmix_next.restype = _U64
        L.oracle_splitmix_next.argtypes = [ctypes.POINTER(_U64)]
        L.oracle_fill_unit.argtypes = [ctypes.POINTER(_U64), _P, _I64]
        L.oracle_paged_attention.restype = _I32
        L.oracle_paged_attention.argtypes = [_I32, _I32, _I32, _I32, _I32, _I32, _D, _P, _I64, _I32,
                                             _P, _P, _P, _P, _P, _P, _P, _P, _P]
        L.oracle_dense_attention.restype = _I32
        L.oracle_dense_attention.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _D, _P]
        L.oracle_gather_pages.argtypes = [_P, _I64, _P, _I64, _P]
        L.oracle_scatter_pages.argtypes = [_P, _I64, _P, _I64, _P]
        L.oracle_append_rows.restype = _I32
        L.oracle_append_rows.argtypes = [_P, _I32, _I32, _I32, _P, _I64, _I64, _P, _I64]
        self.L = L

    def attention(self, shape, batch, q, keys, values, single=False):
        """Returns (status, out) — status uses the PB_* codes."""
        q = np.ascontiguousarray(q, np.float32)
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        out = np.zeros_like(q)
        st = self.L.oracle_paged_attention(
            1 if single else 0, shape.n_head, shape.n_kv_head, shape.head_size, shape.chunk_size,
            shape.n_slots, shape.scale, _p(q), q.size, batch.n_spans, _p(batch.query_start),
            _p(batch.query_len), _p(batch.context_len), _p(batch.causal_offset), _p(batch.bt),
            _p(batch.bt_off), _p(keys), _p(values), _p(out))
        return st, out

    def dense(self, q, k, v, q_len, kv_len, causal_offset, n_head, n_kv, hs, scale):
        out = np.zeros(q_len * n_head * hs, np.float32)
        st = self.L.oracle_dense_attention(_p(np.ascontiguousarray(q, np.float32)),
                                           _p(np.ascontiguousarray(k, np.float32)),
                                           _p(np.ascontiguousarray(v, np.float32)), q_len, kv_len,
                                           causal_offset, n_head, n_kv, hs, scale, _p(out))
        return st, out

    def splitmix(self, seed, n):
        s = _U64(seed)
        return [self.L.oracle_splitmix_next(ctypes.byref(s)) for _ in range(n)]

    def fill_unit(self, seed, n):
        s = _U64(seed)
        out = np.empty(n, np.float32)
        self.L.oracle_fill_unit(ctypes.byref(s), _p(out), n)
        return out

    def gather(self, pool_bytes: np.ndarray, page_bytes: int, slots: np.ndarray) -> np.ndarray:
        slots = np.ascontiguousarray(slots, np.int32)
        out = np.empty(len(slots) * page_bytes, np.uint8)
        self.L.oracle_gather_pages(_p(pool_bytes), page_bytes, _p(slots), len(slots), _p(out))
        return out

    def scatter(self, staging: np.ndarray, page_bytes: int, slots: np.ndarray, pool: np.ndarray):
        slots = np.ascontiguousarray(slots, np.int32)
        self.L.oracle_scatter_pages(_p(staging), page_bytes, _p(slots), len(slots), _p(pool))

    def append(self, pool, chunk, n_slots, row_elems, bt, start_pos, rows):
        bt = np.ascontiguousarray(bt, np.int32)
        rows = np.ascontiguousarray(rows, np.float32)
        return self.L.oracle_append_rows(_p(pool), chunk, n_slots, row_elems, _p(bt), len(bt),
                                         start_pos, _p(rows), rows.size // row_elems)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference (kvsim) through oracle/ref_shim.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        L = ctypes.CDLL(REF_SO)
        L.ref_store_create.restype = _P
        L.ref_store_create.argtypes = [_I32, _I32, _I32, _I32, _P, _P]
        L.ref_store_destroy.argtypes = [_P]
        L.ref_attention.restype = _I32
        L.ref_attention.argtypes = [_P, _I32, _I32, _I32, _D, _P, _I64, _I32, _P, _P, _P, _P, _P, _P,
                                    _P, ctypes.POINTER(_U64)]
        L.ref_attention_mt.restype = _I32
        L.ref_attention_mt.argtypes = [_P, _I32, _I32, _I32, _D, _P, _I32, _P, _P, _P, _P, _P, _P, _P]
        L.ref_dense_attention.restype = _I32
        L.ref_dense_attention.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _D, _P]
        L.ref_qkv_project.restype = _I32
        L.ref_qkv_project.argtypes = [_P, _P, _I32, _I32, _P, _I32, _P, _P, _I32, _P, _I64, _I64, _P, _P, _P]
        L.ref_store_read.argtypes = [_P, _P, _P]
        L.ref_splitmix_next.restype = _U64
        L.ref_splitmix_next.argtypes = [ctypes.POINTER(_U64)]
        L.ref_model_bytes.restype = _I32
        L.ref_model_bytes.argtypes = [ctypes.c_char_p, _I32, _I32, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]
        L.ref_schedule_swap_in.restype = _I32
        L.ref_schedule_swap_in.argtypes = [_D, _U64, _I32, _D, _D, _P, _P, _P, _P]
        L.ref_transfer_time.restype = _I32
        L.ref_transfer_time.argtypes = [_U64, _D, _I32, _D, ctypes.POINTER(_D)]
        L.ref_swap_out_start.restype = _D
        L.ref_swap_out_start.argtypes = [_D, _D, _I32]
        L.ref_cache_create.restype = _P
        L.ref_cache_create.argtypes = [_I32, _I32, _I32]
        L.ref_cache_destroy.argtypes = [_P]
        L.ref_cache_allocate.restype = _I32
        L.ref_cache_allocate.argtypes = [_P, _I64, _I64, _D, _P, _I64, ctypes.POINTER(_I64)]
        L.ref_cache_evict.restype = _I32
        L.ref_cache_evict.argtypes = [_P, _P, _I64, _I32]
        L.ref_cache_bring_back.restype = _I32
        L.ref_cache_bring_back.argtypes = [_P, _I32, _P, _I64, _P]
        L.ref_cache_release.restype = _I32
        L.ref_cache_release.argtypes = [_P, _I64]
        L.ref_cache_retain.restype = _I32
        L.ref_cache_retain.argtypes = [_P, _I64, _D]
        L.ref_cache_block_table.restype = _I32
        L.ref_cache_block_table.argtypes = [_P, _I64, _I64, _P, _I64, ctypes.POINTER(_I64)]
        L.ref_cache_counts.argtypes = [_P, _P]
        L.ref_cache_has.restype = _I32
        L.ref_cache_has.argtypes = [_P, _I64]
        L.ref_cache_total_tokens.restype = _I64
        L.ref_cache_total_tokens.argtypes = [_P, _I64]
        L.ref_cache_append_needed.restype = _I32
        L.ref_cache_append_needed.argtypes = [_P, _I64, _I64]
        L.ref_cache_conv_chunks.restype = _I32
        L.ref_cache_conv_chunks.argtypes = [_P, _I64, _P, _P, _P, _I64, ctypes.POINTER(_I64)]
        L.ref_cache_dump.restype = _I64
        L.ref_cache_dump.argtypes = [_P, ctypes.c_char_p, _I64]
        L.ref_audit_layer_deps.argtypes = [_I32, _P, _P, _P, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]
        self.L = L

    # ---- event log -------------------------------------------------------------------
    def audit_layer_deps(self, kinds, layers, times_s):
        """kvsim::LayerDependencyAuditor fed these events in order -> (violations, steps)."""
        k = np.ascontiguousarray(kinds, np.int32)
        ly = np.ascontiguousarray(layers, np.int32)
        t = np.ascontiguousarray(times_s, np.float64)
        v, st = _U64(), _U64()
        self.L.ref_audit_layer_deps(len(k), k.ctypes.data, ly.ctypes.data, t.ctypes.data, ctypes.byref(v),
                                    ctypes.byref(st))
        return int(v.value), int(st.value)

    # ---- attention -------------------------------------------------------------------
    def store(self, chunk, n_kv, hs, n_slots, keys=None, values=None):
        keys = None if keys is None else np.ascontiguousarray(keys, np.float32)
        values = None if values is None else np.ascontiguousarray(values, np.float32)
        return self.L.ref_store_create(chunk, n_kv, hs, n_slots, _p(keys), _p(values))

    def attention(self, shape, batch, q, keys, values, mode=0):
        """mode 0 paged_multi_token, 1 single_token, 2 copyout_then_dense -> (status, out, gathered)."""
        h = self.store(shape.chunk_size, shape.n_kv_head, shape.head_size, shape.n_slots, keys, values)
        try:
            return self.attention_on(h, shape, batch, q, mode)
        finally:
            self.L.ref_store_destroy(h)

    def attention_on(self, store, shape, batch, q, mode=0):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros_like(q)
        g = _U64(0)
        st = self.L.ref_attention(store, mode, shape.n_head, shape.head_size, shape.scale, _p(q), q.size,
                                  batch.n_spans, _p(batch.query_start), _p(batch.query_len),
                                  _p(batch.context_len), _p(batch.causal_offset), _p(batch.bt),
                                  _p(batch.bt_off), _p(out), ctypes.byref(g))
        return st, out, g.value

    def attention_mt(self, store, shape, batch, q, n_threads):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros_like(q)
        st = self.L.ref_attention_mt(store, n_threads, shape.n_head, shape.head_size, shape.scale, _p(q),
                                     batch.n_spans, _p(batch.query_start), _p(batch.query_len),
                                     _p(batch.context_len), _p(batch.causal_offset), _p(batch.bt),
                                     _p(batch.bt_off), _p(out))
        return st, out

    def destroy_store(self, h):
        self.L.ref_store_destroy(h)

    def splitmix(self, seed, n):
        s = _U64(seed)
        return [self.L.ref_splitmix_next(ctypes.byref(s)) for _ in range(n)]

    def model_bytes(self, preset, chunk, n_kv_override=0):
        a, b = _U64(), _U64()
        st = self.L.ref_model_bytes(preset.encode(), n_kv_override, chunk, ctypes.byref(a), ctypes.byref(b))
        return st, a.value, b.value


class RefCache:
    """The reference kvsim::PagedKvCache through the shim (raises RuntimeError(code))."""

    class Err(RuntimeError):
        def __init__(self, code):
            super().__init__(f"reference status {code}")
            self.code = code

    def __init__(self, ref: "Reference", chunk, dev, host):
        self.L = ref.L
        self.h = self.L.ref_cache_create(chunk, dev, host)
        assert self.h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_cache_destroy(self.h)
            self.h = None

    def _chk(self, st):
        if st != 0:
            raise RefCache.Err(st)

    def allocate(self, conv, n, now):
        out = np.zeros(max(1, n + 1), np.int64)
        k = _I64()
        self._chk(self.L.ref_cache_allocate(self.h, conv, n, now, _p(out), out.size, ctypes.byref(k)))
        return out[: k.value].tolist()

    def apply_evictions(self, ids, to_host):
        ids = np.ascontiguousarray(ids, np.int64)
        self._chk(self.L.ref_cache_evict(self.h, _p(ids) if len(ids) else None, len(ids), 1 if to_host else 0))

    def _bring(self, kind, ids):
        ids = np.ascontiguousarray(ids, np.int64)
        slots = np.zeros(max(1, len(ids)), np.int32)
        self._chk(self.L.ref_cache_bring_back(self.h, kind, _p(ids) if len(ids) else None, len(ids), _p(slots)))
        return slots[: len(ids)].tolist()

    def restore(self, ids):
        return self._bring(0, ids)

    def rematerialize(self, ids):
        return self._bring(1, ids)

    def release_conversation(self, conv):
        self._chk(self.L.ref_cache_release(self.h, conv))

    def retain_on_finish(self, conv, now):
        self._chk(self.L.ref_cache_retain(self.h, conv, now))

    def block_table(self, conv, ctx):
        out = np.zeros(max(1, ctx + 1), np.int32)
        k = _I64()
        self._chk(self.L.ref_cache_block_table(self.h, conv, ctx, _p(out), out.size, ctypes.byref(k)))
        return out[: k.value].tolist()

    def counts(self):
        c = np.zeros(8, np.int64)
        self.L.ref_cache_counts(self.h, _p(c))
        keys = ("device_capacity", "device_free", "device_reclaimable", "device_allocated", "host_capacity",
                "host_free", "host_allocated", "verify_status")
        return dict(zip(keys, (int(x) for x in c)))

    def has_conversation(self, conv):
        return bool(self.L.ref_cache_has(self.h, conv))

    def total_tokens(self, conv):
        return int(self.L.ref_cache_total_tokens(self.h, conv))

    def append_chunks_needed(self, conv, add):
        return int(self.L.ref_cache_append_needed(self.h, conv, add))

    def conversation_chunks(self, conv):
        n = 1 << 14
        ids, kinds, slots = np.zeros(n, np.int64), np.zeros(n, np.int32), np.zeros(n, np.int32)
        k = _I64()
        self._chk(self.L.ref_cache_conv_chunks(self.h, conv, _p(ids), _p(kinds), _p(slots), n, ctypes.byref(k)))
        return list(zip(ids[: k.value].tolist(), kinds[: k.value].tolist(), slots[: k.value].tolist()))

    def dump(self):
        n = self.L.ref_cache_dump(self.h, None, 0)
        buf = ctypes.create_string_buffer(int(n) + 1)
        self.L.ref_cache_dump(self.h, buf, n + 1)
        return buf.value.decode()
