"""Nova (arXiv 2509.21301) on B200: cross-stage co-execution of a VLM's vision
encode, LLM prefill and LLM decode on disjoint, elastically resized SM partitions
of one GPU, behind the C ABI in include/nova.h (libnova.so).

The package holds only the path: csrc/ (sm_100a kernels, stage programs,
partition executor, Algorithm 1 controller, C ABI) and its Python binding.
"""
from ._lib import lib, LIB_PATH  # noqa: F401
