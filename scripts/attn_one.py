"""Run one flash-attention shape through the op ABI a few times (for ncu captures).

    python scripts/attn_one.py S H KV hd causal [ITERS]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21301_b200 import ops as O  # noqa: E402

S, H, KV, hd, causal = (int(x) for x in sys.argv[1:6])
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 5
qkv = torch.randn(S, (H + 2 * KV) * hd, device="cuda").bfloat16()
out = torch.empty(S, H * hd, device="cuda", dtype=torch.bfloat16)
for _ in range(iters):
    O.nova_op_flash_attn(qkv, out, S, H, KV, hd, causal)
torch.cuda.synchronize()
