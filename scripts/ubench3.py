"""Per-CTA timeline of one tcgen05 decode GEMV launch (env NOVA_UMMA_TDBG=1): 2B gate|up, B = 2."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NOVA_UMMA_TDBG"] = "1"
from paper_2509_21301_b200 import ops as O  # noqa: E402

N, K, B = 17920, 1536, 2
W = (torch.randn(N, K, device="cuda") * K ** -0.5).bfloat16()
Wb = torch.empty_like(W)
O.nova_op_block_weights(W, Wb, N, K)
X = torch.randn(16, K, device="cuda").bfloat16()
Y = torch.zeros(16, N // 2, dtype=torch.bfloat16, device="cuda")
for ctas in (148, 64):
    for it in range(3):
        O.nova_op_gemv_umma(X[:B], Wb, Y, None, N, K, B, O.EPI_BF16_SILUMUL, max_ctas=ctas)
    torch.cuda.synchronize()
    ws, _ = O._ws_cache[X.device]
    grid = 4 * ctas
    t = ws.view(torch.int64)[16 * 1024 * 1024: 16 * 1024 * 1024 + grid * 16].view(grid, 16).cpu().numpy()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    names = ["start", "prod_pdl", "mma_full0", "mma_lastcommit", "epi_tfull0", "epi_fence", "epi_ticket",
             "epi_done", "prod_done", "exit"]
    out = {n: [round(float(np.percentile(rel[:, i], q)), 2) for q in (0, 50, 90, 100)] for i, n in enumerate(names)
           if (t[:, i] > 0).any()}
    print(json.dumps({"ctas_budget": ctas, "grid": grid, "pct_0_50_90_100_us": out}))
