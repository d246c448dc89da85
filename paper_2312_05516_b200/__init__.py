"""B200-native Pensieve hot path (arXiv 2312.05516): ragged paged attention + KV tier movement.

The product is the C-ABI library ``libpensieve_b200.so`` (include/pensieve_b200.h) built from
``csrc/`` for sm_100a.  ``abi`` is a thin ctypes binding used by the tests and bench; it never
computes anything itself and raises ImportError when the native library is missing.  The
library is loaded on first use of ``abi`` (not at package import), so host-only modules
(``descriptors``, ``workloads``) can be used by the reference-arm benchmark without it.
"""
from __future__ import annotations

from .descriptors import PB_BF16, PB_F32, AttnShape, Batch  # noqa: F401

__all__ = ["abi", "lib", "AttnShape", "Batch", "PBError", "PB_F32", "PB_BF16", "so_path"]


def __getattr__(name):
    if name in ("abi", "lib", "PBError"):
        import importlib
        abi = importlib.import_module(".abi", __name__)
        return abi if name == "abi" else getattr(abi, name)
    raise AttributeError(name)


def so_path() -> str:
    from . import abi
    return abi.SO_PATH
