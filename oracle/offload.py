"""ORACLE (test infrastructure only) -- layer-wise ViT weight offload (§III-E).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline leg may
import this.  Shares no code with the CUDA path.

  Eq. 7  nxt_layer = (cur_layer + K) mod L
  Eq. 8  B >= (S/T) (L-K)/(L-2)   (zero-stall bandwidth)
Swap-in starts after layer 0 finishes and wraps into the next pass
(reading R20).  `simulate` is the two-timeline model: one compute
timeline, one copy engine doing one DMA at a time.
"""
from __future__ import annotations


def next_logical_layer(cur: int, K: int, L: int) -> int:
    """Eq. 7."""
    return (cur + K) % L


def load_schedule(K: int, L: int, passes: int = 1) -> list[tuple[int, int, int]]:
    """(pass, logical layer just finished, logical layer loaded into its slot)."""
    out = []
    for p in range(passes):
        for l in range(L):
            out.append((p, l, next_logical_layer(l, K, L)))
    return out


def required_bandwidth(S: float, T: float, L: int, K: int) -> float:
    """Eq. 8: minimum bandwidth for zero stall, S bytes of weights, T forward time."""
    return S / T * (L - K) / (L - 2)


def simulate(compute: list[float], layer_bytes: float, bw: float, K: int, passes: int = 1):
    """Two timelines (compute, copy).  Layers 0..K-1 resident at t=0.

    After layer l of a pass finishes, its slot (l mod K) is refilled with layer
    (l+K) mod L (which belongs to the same pass if l+K < L, else to the next).
    Returns (total time, total stall) where stall = time the compute timeline
    waited for a load."""
    L = len(compute)
    t_copy = 0.0
    ready = {}                       # (pass, layer) -> load completion time
    for l in range(min(K, L)):
        ready[(0, l)] = 0.0
    t = 0.0
    stall = 0.0
    for p in range(passes):
        for l in range(L):
            start = max(t, ready[(p, l)])
            stall += start - t
            t = start + compute[l]
            nxt = l + K
            key = (p, nxt) if nxt < L else (p + 1, nxt - L)
            t_copy = max(t_copy, t) + layer_bytes / bw
            ready[key] = t_copy
    return t, stall
