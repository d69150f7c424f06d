"""Seeded random-init weights as bf16 bit patterns (uint16).

Shared input generator (no method arithmetic).  Per tensor the stream is
PCG64 seeded with (seed, crc32(name)) so any tensor can be regenerated on its
own.  Values are drawn in float32 and rounded to
bf16 with round-to-nearest-even; both the oracle and the engine consume the
*same* bf16 bits.

`device_tensor` is the fast path the benchmark uses at full model size: the
same distributions drawn with torch's CUDA generator.  Those values differ
from the host stream (timing does not depend on them) and never feed a
parity check.
"""
from __future__ import annotations

import zlib

import numpy as np

from .models import ModelShape, weight_specs


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern, round-to-nearest-even (NaN-free inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def _rng(seed: int, name: str) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed), zlib.crc32(name.encode())]))


def gen_tensor(name: str, shape: tuple, init: tuple, seed: int) -> np.ndarray:
    """One tensor as bf16 bits (uint16, C-contiguous, `shape`)."""
    rng = _rng(seed, name)
    kind, a = init
    n = int(np.prod(shape))
    if kind == "normal":
        v = rng.standard_normal(n, dtype=np.float32) * np.float32(a)
    elif kind == "uniform":
        v = rng.uniform(-a, a, n).astype(np.float32)
    elif kind == "gamma":
        v = (1.0 + rng.uniform(-a, a, n)).astype(np.float32)
    else:
        raise ValueError(kind)
    return f32_to_bf16_bits(v).reshape(shape)


def gen_weights(shape: ModelShape, seed: int) -> dict[str, np.ndarray]:
    """All tensors of `shape` as {name: uint16 array}."""
    return {n: gen_tensor(n, shp, init, seed) for n, shp, init in weight_specs(shape)}


def device_tensor(name: str, shp: tuple, init: tuple, seed: int, device="cuda"):
    """Same distribution drawn on the GPU by torch (bench only; never a parity input)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) << 32) ^ zlib.crc32(name.encode()))
    kind, a = init
    if kind == "normal":
        t = torch.randn(shp, generator=g, device=device, dtype=torch.float32).mul_(a)
    elif kind == "uniform":
        t = torch.rand(shp, generator=g, device=device, dtype=torch.float32).mul_(2 * a).sub_(a)
    else:
        t = torch.rand(shp, generator=g, device=device, dtype=torch.float32).mul_(2 * a).add_(1 - a)
    return t.to(torch.bfloat16)
