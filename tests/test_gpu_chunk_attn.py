"""Chunked-prefill attention (csrc/attn.cu chunk_attn, include/nova_ops.h nova_op_chunk_attn) vs
the oracle's causal GQA attention (oracle/vlm.py attention_causal_gqa) on the same bf16 q / k / v:
a chunk of C query rows at cache offset c0 over a paged cache whose pages are scattered in the pool
(block table), at the 2B / 7B / tiny head shapes, ragged chunk and prefix lengths.  bf16 output
rel-inf <= 2e-2 (P rounded to bf16 before P.V, as in every FMHA here)."""
import numpy as np
import pytest
import torch

from oracle import vlm as V
from tests.gpu_util import bf16_dev, bf16_host, rand_bf16, rel_inf

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2509_21301_b200 import ops as O


@pytest.mark.parametrize("H,KV,hd,c0,C", [(12, 2, 128, 1160, 126), (12, 2, 128, 0, 128), (28, 4, 128, 1900, 100),
                                          (4, 2, 32, 5, 7), (12, 2, 128, 64, 1), (28, 4, 128, 333, 77)])
def test_chunk_attn_matches_oracle(H, KV, hd, c0, C):
    rng = np.random.default_rng(H + c0 + C)
    T = c0 + C
    n_pages, layers, layer = (T + 63) // 64 + 5, 2, 1
    q = rand_bf16(rng, (C, H, hd))
    k = rand_bf16(rng, (T, KV, hd))
    v = rand_bf16(rng, (T, KV, hd))
    pages = rng.permutation(n_pages)[: (T + 63) // 64].astype(np.int32)       # scattered pages
    pool = np.zeros((layers, n_pages, 2, KV, 64, hd), dtype=np.float32)
    for j in range(T):
        pool[layer, pages[j // 64], 0, :, j % 64] = k[j]
        pool[layer, pages[j // 64], 1, :, j % 64] = v[j]
    ldq = (H + 2 * KV) * hd
    qkv = np.zeros((C, ldq), dtype=np.float32)
    qkv[:, : H * hd] = q.reshape(C, H * hd)
    d_qkv, d_pool = bf16_dev(qkv), bf16_dev(pool.reshape(-1, hd))
    out = torch.zeros(C, H * hd, dtype=torch.bfloat16, device="cuda")
    bt = torch.from_numpy(pages).cuda()
    O.nova_op_chunk_attn(d_qkv, out, C, c0, H, KV, hd, d_pool, layer, n_pages, bt)
    torch.cuda.synchronize()
    ref = V.attention_causal_gqa(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), hd ** -0.5, c0)
    assert rel_inf(bf16_host(out), ref.reshape(C, H * hd)) <= 2e-2
