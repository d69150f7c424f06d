"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds shapes, weight schema, random weights, request inputs and arrival
traces -- and none of the method's arithmetic.
"""
from .models import ModelShape, TINY, Q2B, Q7B, PRESETS, weight_specs, reduced_depth, param_count  # noqa: F401
from .weights import gen_weights, gen_tensor, f32_to_bf16_bits, bf16_bits_to_f32  # noqa: F401
from .inputs import RequestInput, make_request, tiny_request, poisson_trace, mmpp2_trace  # noqa: F401
