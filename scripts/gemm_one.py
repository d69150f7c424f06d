"""Run one GEMM shape through the op ABI a few times (for ncu captures).

    python scripts/gemm_one.py M N K EPI [MODE] [ITERS]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21301_b200 import ops as O  # noqa: E402

M, N, K, epi = (int(x) for x in sys.argv[1:5])
mode = int(sys.argv[5]) if len(sys.argv) > 5 else 0
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 5
O.nova_op_gemm_mode(mode)
A = (torch.randn(M, K, device="cuda")).bfloat16()
W = (torch.randn(N, K, device="cuda") * K ** -0.5).bfloat16()
bias = (torch.randn(N, device="cuda") * 0.1).bfloat16() if epi != O.EPI_BF16_SILUMUL else None
nout = N // 2 if epi == O.EPI_BF16_SILUMUL else N
C = torch.zeros(M, nout, device="cuda", dtype=torch.float32 if epi in (O.EPI_F32_RESID, O.EPI_F32_STORE) else torch.bfloat16)
for _ in range(iters):
    O.nova_op_gemm(A, W, C, bias, M, N, K, epi)
torch.cuda.synchronize()
print("tile", O.nova_op_gemm_config(M, N, K))
