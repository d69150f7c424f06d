"""Persistent paged decode attention (csrc/decode_attn_p.cu, include/nova_ops.h
nova_op_decode_attn_p) vs the oracle's causal GQA attention (oracle/vlm.py attention_causal_gqa) on
the same bf16 q / cached K / V: 7B / 2B / tiny head shapes, ragged contexts (1 key .. 2048 keys,
chunk edges), scattered pages; bf16 rel-inf <= 8e-3; bitwise invariance to the SM budget and to
the rest of the batch (the partition-invariance that co-execution relies on)."""
import numpy as np
import pytest
import torch

from oracle import vlm as V
from tests.gpu_util import bf16_dev, bf16_host, rand_bf16, rel_inf

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2509_21301_b200 import ops as O


@pytest.mark.parametrize("H,KV,hd,ctxs", [(28, 4, 128, [1333, 17, 640, 2047]), (12, 2, 128, [1334, 0, 127, 128, 255]),
                                          (4, 2, 32, [11, 63, 64, 200]),
                                          (12, 2, 128, [1300 + 7 * b for b in range(16)])])
def test_decode_attn_p_matches_oracle_and_is_grid_invariant(H, KV, hd, ctxs):
    rng = np.random.default_rng(H + len(ctxs))
    B = len(ctxs)
    per = (max(ctxs) + 1 + 63) // 64
    n_pages = B * per + 3
    pool_np = rand_bf16(rng, (1, n_pages, 2, KV, 64, hd))
    pool = bf16_dev(pool_np)
    perm = rng.permutation(n_pages)[: B * per].astype(np.int32)
    bt = torch.from_numpy(perm.reshape(B, per).copy()).cuda()
    qd = rand_bf16(rng, (B, (H + 2 * KV) * hd))
    rows = torch.tensor([[b, ctxs[b], 0, 0] for b in range(B)], dtype=torch.int32, device="cuda")
    mch = (max(ctxs) + 1 + 127) // 128
    ws = torch.empty(B * KV * mch * (32 + (H // KV) * hd), dtype=torch.float32, device="cuda")
    tk = torch.zeros(B * KV, dtype=torch.int32, device="cuda")
    dq = bf16_dev(qd)
    outs = []
    for ctas in (0, 32, 8, 1):
        out = torch.empty(B, H * hd, dtype=torch.bfloat16, device="cuda")
        O.nova_op_decode_attn_p(dq, out, pool, 0, n_pages, H, KV, hd, bt, rows, B, max(ctxs), ws, tk, mch, ctas)
        torch.cuda.synchronize()
        outs.append(out)
    assert int(tk.abs().sum().item()) == 0
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    btn = bt.cpu().numpy()
    for b, ctx in enumerate(ctxs):
        kc = np.stack([pool_np[0, btn[b, t // 64], 0, :, t % 64] for t in range(ctx + 1)]).astype(np.float64)
        vc = np.stack([pool_np[0, btn[b, t // 64], 1, :, t % 64] for t in range(ctx + 1)]).astype(np.float64)
        ref = V.attention_causal_gqa(qd[b:b + 1, :H * hd].reshape(1, H, hd).astype(np.float64), kc, vc, hd ** -0.5, ctx)
        assert rel_inf(bf16_host(outs[0][b:b + 1]).reshape(1, H, hd), ref) <= 8e-3, b
    # batch invariance: request 0 alone == request 0 in the batch
    out1 = torch.empty(1, H * hd, dtype=torch.bfloat16, device="cuda")
    O.nova_op_decode_attn_p(dq[:1], out1, pool, 0, n_pages, H, KV, hd, bt, rows[:1], 1, ctxs[0], ws, tk, mch, 16)
    torch.cuda.synchronize()
    assert torch.equal(out1[0], outs[0][0])
