"""Seeded request inputs (screenshot pixels, prompt ids) and arrival traces.

Shared input generator (no method arithmetic).  Shapes follow the paper's
workload: GUI screenshots (§II-C), short instructions, 30-80
output tokens (§V-A) and Poisson arrivals; the
bursty MMPP-2 variant and the 1080p grids are the recipe of SURVEY.md §8(d) d1'.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .models import ModelShape
from .weights import f32_to_bf16_bits

# 1920x1080 screenshot resized by Qwen2-VL smart_resize (factor 28):
# max_pixels 1280*28^2 -> 728x1316 (grid 52x94, N=4888); 2048*28^2 -> 924x1680 (66x120, N=7920)
GRID_1080P_A = (52, 94)
GRID_1080P_B = (66, 120)


@dataclass
class RequestInput:
    pixels: np.ndarray      # uint16 bf16 bits, [3][H][W]
    prompt_ids: np.ndarray  # int32 [n_prompt]
    gen_len: int

    @property
    def height(self) -> int:
        return int(self.pixels.shape[1])

    @property
    def width(self) -> int:
        return int(self.pixels.shape[2])


def make_request(shape: ModelShape, grid_hw: tuple[int, int], n_prompt: int, gen_len: int,
                 seed: int) -> RequestInput:
    """Image of grid_hw patches (H = gh*patch, W = gw*patch), U(-1,1) pixels, uniform ids."""
    gh, gw = grid_hw
    assert gh % shape.merge == 0 and gw % shape.merge == 0
    rng = np.random.Generator(np.random.PCG64([int(seed), 0x5EED]))
    H, W = gh * shape.patch, gw * shape.patch
    pix = rng.uniform(-1.0, 1.0, (shape.in_ch, H, W)).astype(np.float32)
    ids = rng.integers(0, shape.vocab, n_prompt, dtype=np.int64).astype(np.int32)
    return RequestInput(f32_to_bf16_bits(pix), ids, int(gen_len))


def tiny_request(shape: ModelShape, seed: int) -> RequestInput:
    """cfg 1: one 56x56 image (16 patches), 8 prompt ids, 8 greedy tokens."""
    return make_request(shape, (4, 4), 8, 8, seed)


# ------------------------------------------------------------------ traces
@dataclass
class TraceRow:
    arrival_s: float
    grid_h: int
    grid_w: int
    prompt_tokens: int
    gen_len: int


def poisson_trace(n: int, lam: float, seed: int, grids=(GRID_1080P_A,), prompt=(64, 64),
                  gen=(48, 48)) -> list[TraceRow]:
    """Poisson arrivals at rate lam (req/s); first arrival at t=0 (SURVEY d1')."""
    rng = np.random.Generator(np.random.PCG64([int(seed), 0x7AACE]))
    t, rows = 0.0, []
    for i in range(n):
        if i > 0:
            t += rng.exponential(1.0 / lam)
        rows.append(_row(rng, t, grids, prompt, gen))
    return rows


def mmpp2_trace(n: int, rho: float, t_front_s: float, seed: int,
                grids=(GRID_1080P_A, GRID_1080P_B), prompt=(32, 128), gen=(32, 64),
                burst_ratio: float = 4.0, calm_dwell: float = 40.0,
                burst_dwell: float = 10.0) -> list[TraceRow]:
    """Bursty 2-state MMPP: calm rate lc, burst rate 4*lc, dwell Exp(40 T) / Exp(10 T).

    Mean rate = lc*(40 + 4*10)/50 = 1.6*lc, so lc = rho / (1.6 * T_front).
    """
    rng = np.random.Generator(np.random.PCG64([int(seed), 0xB0057]))
    frac_burst = burst_dwell / (calm_dwell + burst_dwell)
    lc = rho / (t_front_s * ((1 - frac_burst) + frac_burst * burst_ratio))
    state, t = 0, 0.0
    state_end = rng.exponential(calm_dwell * t_front_s)
    rows = [_row(rng, 0.0, grids, prompt, gen)]
    while len(rows) < n:
        rate = lc * (burst_ratio if state else 1.0)
        dt = rng.exponential(1.0 / rate)
        if t + dt > state_end:          # memoryless: restart the clock at the switch
            t = state_end
            state ^= 1
            state_end = t + rng.exponential((burst_dwell if state else calm_dwell) * t_front_s)
            continue
        t += dt
        rows.append(_row(rng, t, grids, prompt, gen))
    return rows


def _row(rng, t, grids, prompt, gen) -> TraceRow:
    g = grids[int(rng.integers(0, len(grids)))] if len(grids) > 1 else grids[0]
    return TraceRow(float(t), int(g[0]), int(g[1]),
                    int(rng.integers(prompt[0], prompt[1] + 1)),
                    int(rng.integers(gen[0], gen[1] + 1)))


def write_csv(rows: list[TraceRow], path: str) -> None:
    with open(path, "w") as f:
        f.write("arrival_s,grid_h,grid_w,prompt_tokens,gen_len\n")
        for r in rows:
            f.write(f"{r.arrival_s:.6f},{r.grid_h},{r.grid_w},{r.prompt_tokens},{r.gen_len}\n")
