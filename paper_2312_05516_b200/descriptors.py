"""Batch descriptor types of the C-ABI (include/pensieve_b200.h) that host-only code needs
without loading the native library: the attention shape struct and the ragged batch (CSR
block tables).  The reference-arm benchmark and the workload generators import these; only
``abi`` loads libpensieve_b200.so."""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

PB_F32 = 0
PB_BF16 = 1


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



def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    if a is None:
        return None
    return a.ctypes.data


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
