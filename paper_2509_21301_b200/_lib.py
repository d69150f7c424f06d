"""ctypes loader for libnova.so (the C ABI in include/nova.h and include/nova_ops.h).

Fails loudly when the extension is missing: there is no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnova.so")
_lib = None

P = C.c_void_p
I = C.c_int
F = C.c_float
D = C.c_double
I64 = C.c_int64
U64 = C.c_uint64

OPS_SIGNATURES = {
    "nova_op_gemm": [P, I, P, I, P, I, P, I, I, I, I, I, P],
    "nova_op_gemm_fold": [P, I, P, I, P, I, P, I, I, I, I, I, P, P, I, P, I, P, P],
    "nova_op_fold_rows": [P, I, I, F, P, I, P],
    "nova_op_gemm_rope2d": [P, I, P, I, P, I, P, I, I, I, I, I, I, F, I, P],
    "nova_op_rms_prep": [P, I, P, P, I, P, I, I, I, P],
    "nova_op_gemm_mode": [I],
    "nova_op_gemm_config": [I, I, I],
    "nova_op_gemv": [P, I, I, P, I, I, P, I, P, I, I, P],
    "nova_op_gemv_tma": [P, I, P, I, I, P, I, P, I, I, P, P, I, P],
    "nova_op_flash_attn": [P, I, P, I, I, I, I, I, I, I, P],
    "nova_op_flash_attn_mma": [P, I, P, I, I, I, I, I, I, P],
    "nova_op_decode_attn": [P, I, P, I, P, I, I, I, I, I, P, I, P, I, I, P, P, I, P],
    "nova_op_gemv_fused": [P, I, I, P, I, I, P, I, P, I, I, P, F, I, I, I, F, P, P, I, I, P, I, P, P],
    "nova_op_argmax_finalize": [P, I, P, P, P, I, P],
    "nova_op_block_weights": [P, P, I, I, P],
    "nova_op_gemv_stream": [P, P, I, P, I, I, P, I, P, I, I, P, P, P, I, P],
    "nova_op_gemv_umma": [P, P, I, P, I, I, P, I, P, I, I, P, P, P, I, P, F, P, P, I, P],
    "nova_op_gemv_umma_splits": [I, I, I],
    "nova_op_gemv_umma_qkv": [P, I, P, I, I, P, I, P, I, P, F, I, I, I, F, P, P, I, I, P, I, P, P, I, P],
    "nova_op_scale_rows_bf16": [P, I, P, P, I, I, I, P],
    "nova_op_chunk_attn": [P, I, P, I, I, I, I, I, I, P, I, I, P, P],
    "nova_op_decode_attn_p": [P, I, P, I, P, I, I, I, I, I, P, I, P, I, I, P, P, I, I, P],
    "nova_op_layernorm": [P, I, P, P, P, I, I, I, F, P],
    "nova_op_rmsnorm": [P, I, P, P, I, I, I, I, F, P],
    "nova_op_patchify": [P, I, I, I, I, I, I, P, P],
    "nova_op_vit_rope": [P, I, I, I, I, I, F, P],
    "nova_op_llm_rope_kv": [P, I, I, I, I, I, F, I, I, P, I, P, I, I, P, I, I, P, I, P],
    "nova_op_embed": [P, I, P, P, P, P, I, I, P],
    "nova_op_argmax": [P, I, I, I, P, P, P, I, P],
}


def lib():
    """Load libnova.so once; raise if it was not built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing; build it with `python -m paper_2509_21301_b200.build` "
                               "(the CUDA path has no fallback)")
        lb = C.CDLL(LIB_PATH)
        for name, args in OPS_SIGNATURES.items():
            fn = getattr(lb, name)
            fn.argtypes = args
            fn.restype = I
        from . import _abi
        _abi.declare(lb)
        _lib = lb
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        raise RuntimeError(f"libnova call {what} failed with status {rc}")
