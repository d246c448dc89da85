"""B200-native Pensieve hot path (arXiv 2312.05516): ragged paged attention + KV tier movement.

The product is the C-ABI library ``libpensieve_b200.so`` (include/pensieve_b200.h) built from
``csrc/`` for sm_100a.  This module is a thin ctypes binding used by the tests and bench; it
never computes anything itself and fails loudly when the native library is missing.
"""
from __future__ import annotations

from . import abi
from .abi import (  # noqa: F401
    PB_BF16,
    PB_F32,
    AttnShape,
    PBError,
    lib,
)

__all__ = ["abi", "lib", "AttnShape", "PBError", "PB_F32", "PB_BF16", "so_path"]


def so_path() -> str:
    return abi.SO_PATH
