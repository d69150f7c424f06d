"""Per-CTA streaming rate of the tcgen05 decode GEMV (2B gate|up, 55 MB) on small grids (one CTA per SM:
max_ctas budget x 4 CTAs spread over the GPU), with timing-only variants (env NOVA_UMMA_DBG)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from kbench import timeit, rnd  # noqa: E402
from paper_2509_21301_b200 import ops as O  # noqa: E402

N, K = 17920, 1536
rot = 6
Wbs = []
for _ in range(rot):
    W = rnd((N, K), scale=K ** -0.5)
    Wb = torch.empty_like(W)
    O.nova_op_block_weights(W, Wb, N, K)
    Wbs.append(Wb)
X = rnd((16, K))
Y = torch.zeros(16, N // 2, dtype=torch.bfloat16, device="cuda")
for B in (2,):
    for ctas in (2, 8, 16, 32, 148):
        def call(i):
            O.nova_op_gemv_umma(X[:B], Wbs[i], Y, None, N, K, B, O.EPI_BF16_SILUMUL, max_ctas=ctas)
        ms = timeit(call, 10, rot)
        grid = min(4 * ctas, N // 128)
        gbs = N * K * 2 / (ms / 1e3) / 1e9
        print(json.dumps({"dbg": os.environ.get("NOVA_UMMA_DBG", "0"), "B": B, "ctas_budget": ctas, "grid": grid,
                          "us": round(ms * 1e3, 1), "GBs": round(gbs, 1), "GBs_per_cta": round(gbs / grid, 1)}),
              flush=True)
