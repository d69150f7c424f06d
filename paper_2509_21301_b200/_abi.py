"""ctypes declarations of the engine ABI (include/nova.h)."""
from __future__ import annotations

import ctypes as C

ENGINE_SIGNATURES: dict = {}


def declare(lb) -> None:
    for name, (res, args) in ENGINE_SIGNATURES.items():
        if hasattr(lb, name):
            fn = getattr(lb, name)
            fn.argtypes = args
            fn.restype = res
