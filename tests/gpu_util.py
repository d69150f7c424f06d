"""Helpers for GPU parity tests: move bf16 bit patterns between numpy and torch."""
import numpy as np
import torch

from synth.weights import f32_to_bf16_bits, bf16_bits_to_f32


def bf16_dev(bits_or_f32: np.ndarray) -> torch.Tensor:
    a = np.asarray(bits_or_f32)
    if a.dtype != np.uint16:
        a = f32_to_bf16_bits(a.astype(np.float32))
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def bf16_host(t: torch.Tensor) -> np.ndarray:
    """bf16 device tensor -> float32 numpy (exact)."""
    return bf16_bits_to_f32(t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16))


def rand_bf16(rng, shape, scale=1.0) -> np.ndarray:
    """Random values already rounded to bf16 (returned as float32)."""
    return bf16_bits_to_f32(f32_to_bf16_bits((rng.standard_normal(shape) * scale).astype(np.float32)))


def rel_inf(a, ref) -> float:
    return float(np.abs(np.asarray(a, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))
