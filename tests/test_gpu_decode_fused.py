"""Fused decode kernels (GPU) through the C ABI (include/nova_ops.h nova_op_gemv_fused,
nova_op_argmax_finalize, nova_op_decode_attn) vs the oracle's ops (oracle/vlm.py
rms_norm / linear / mrope_tables / apply_rope / attention_causal_gqa / argmax_lowest):

* RMSNorm applied on load == rmsnorm kernel + plain GEMV, bitwise (same statistics order);
* qkv GEMV + bias + RoPE + paged-KV append epilogue vs oracle (bf16 rel-inf <= 8e-3), and
  bitwise batch invariance of row 0;
* lm_head with the fused argmax: logits bitwise == the f32-store epilogue, token == oracle
  argmax_lowest (ties -> lowest index), keys reset to zero.
"""
import numpy as np
import pytest
import torch

from oracle import vlm as V
from tests.gpu_util import bf16_dev, bf16_host, rand_bf16, rel_inf

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2509_21301_b200 import ops as O


def _gamma(rng, d):
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    return bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (d,), 0.1) + 1.0))   # exactly representable


@pytest.mark.parametrize("N,K,epi", [(4608, 3584, "bf16"), (512, 128, "silu"), (37888, 3584, "silu"),
                                     (2048, 1536, "bf16")])
def test_norm_on_load_is_bitwise_rmsnorm_then_gemv(N, K, epi):
    rng = np.random.default_rng(N + K)
    W = bf16_dev(rand_bf16(rng, (N, K), K ** -0.5))
    g = bf16_dev(_gamma(rng, K))
    e = O.EPI_BF16 if epi == "bf16" else O.EPI_BF16_SILUMUL
    nout = N if epi == "bf16" else N // 2
    for B in (1, 5, 16):
        X = torch.from_numpy((rng.standard_normal((B, K)) * 3).astype(np.float32)).cuda()
        xb = torch.empty(B, K, dtype=torch.bfloat16, device="cuda")
        O.nova_op_rmsnorm(X, g, xb, B, K, 1e-6)
        Y0 = torch.empty(B, nout, dtype=torch.bfloat16, device="cuda")
        O.nova_op_gemv(xb, W, Y0, None, N, K, B, e)
        Y1 = torch.empty_like(Y0)
        O.nova_op_gemv_fused(X, O.XM_NORM_BF16, W, Y1, None, N, K, B, e, gamma=g, eps=1e-6)
        torch.cuda.synchronize()
        assert torch.equal(Y0.view(torch.int16), Y1.view(torch.int16)), B


@pytest.mark.parametrize("H,KV,hd,D,tma", [(4, 2, 32, 128, 0), (28, 4, 128, 3584, 0), (28, 4, 128, 3584, 1),
                                           (12, 2, 128, 1536, 1)])
def test_qkv_rope_kv_append_matches_oracle(H, KV, hd, D, tma):
    """tma = 0: register GEMV with RMSNorm on load; tma = 1: persistent TMA kernel on the
    bf16-normalized rows (rmsnorm kernel first)."""
    rng = np.random.default_rng(H * 7 + D)
    N = (H + 2 * KV) * hd
    W = rand_bf16(rng, (N, D), D ** -0.5)
    bias = rand_bf16(rng, (N,), 0.05)
    gam = _gamma(rng, D)
    n_pages, max_pages, theta, eps = 64, 8, 1e6, 1e-6
    bt = torch.from_numpy(rng.permutation(n_pages)[:4 * max_pages].reshape(4, max_pages).astype(np.int32)).cuda()
    dW, db, dg = bf16_dev(W), bf16_dev(bias), bf16_dev(gam)
    Xh = (rng.standard_normal((16, D)) * 2).astype(np.float32)
    rows_np = np.array([[b % 4, int(rng.integers(0, 500)), int(rng.integers(0, 3000)), 0] for b in range(16)],
                       np.int32)
    rows_np[:4, 0] = [0, 1, 2, 3]
    rows_np[:4, 1] = [0, 63, 64, 300]   # page boundaries
    got0 = None
    for B in (1, 4, 16):
        # rows beyond 4 reuse slots with distinct ctx (different cache cells)
        r = rows_np[:B].copy()
        for b in range(4, B):
            r[b, 1] = 320 + b
        pool = torch.zeros(2, n_pages, 2, KV, 64, hd, dtype=torch.bfloat16, device="cuda")
        rows = torch.from_numpy(r).cuda()
        Q = torch.zeros(B, N, dtype=torch.bfloat16, device="cuda")
        Xd = torch.from_numpy(Xh[:B]).cuda()
        if tma:
            xb = torch.empty(B, D, dtype=torch.bfloat16, device="cuda")
            O.nova_op_rmsnorm(Xd, dg, xb, B, D, eps)
            O.nova_op_gemv_fused(xb, O.XM_BF16, dW, Q, db, N, D, B, O.EPI_QKV_ROPE_KV, H=H, KV=KV, hd=hd,
                                 theta=theta, rows=rows, kv_pool=pool, layer=1, n_pages=n_pages, block_tables=bt)
        else:
            O.nova_op_gemv_fused(Xd, O.XM_NORM_BF16, dW, Q, db, N, D, B, O.EPI_QKV_ROPE_KV,
                                 gamma=dg, eps=eps, H=H, KV=KV, hd=hd, theta=theta, rows=rows, kv_pool=pool, layer=1,
                                 n_pages=n_pages, block_tables=bt)
        torch.cuda.synchronize()
        # oracle: bf16-rounded normalized input (the GEMV operand), f64 linear + bias, RoPE at pos
        from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
        a = bf16_bits_to_f32(f32_to_bf16_bits(V.rms_norm(Xh[:B].astype(np.float32), gam, eps).astype(np.float32)))
        y = V.linear(a.astype(np.float64), W.astype(np.float64), bias.astype(np.float64))
        pos3 = np.tile(r[:, 2], (3, 1))
        c, s = V.mrope_tables(pos3, hd, theta, (hd // 2, 0, 0), np.float64)   # t = h = w: any sections
        q = V.apply_rope(y[:, :H * hd].reshape(B, H, hd), c, s)
        k = V.apply_rope(y[:, H * hd:(H + KV) * hd].reshape(B, KV, hd), c, s)
        v = y[:, (H + KV) * hd:].reshape(B, KV, hd)
        assert rel_inf(bf16_host(Q[:, :H * hd]).reshape(B, H, hd), q) <= 8e-3
        P = bf16_host(pool[1])
        btn = bt.cpu().numpy()
        for b in range(B):
            pg, off = btn[r[b, 0], r[b, 1] // 64], r[b, 1] % 64
            assert rel_inf(P[pg, 0, :, off], k[b]) <= 8e-3
            assert rel_inf(P[pg, 1, :, off], v[b]) <= 8e-3
        assert float(np.abs(bf16_host(pool[0])).max()) == 0.0     # other layers untouched
        row0 = Q[0].view(torch.int16).cpu()
        if got0 is None:
            got0 = row0
        assert torch.equal(row0, got0)                            # bitwise batch invariance


@pytest.mark.parametrize("V_,D", [(512, 128), (152064, 3584)])
def test_lm_head_fused_argmax(V_, D):
    rng = np.random.default_rng(V_ + D)
    W = rand_bf16(rng, (V_, D), 2 * D ** -0.5)
    gam = _gamma(rng, D)
    B = 5
    Xh = (rng.standard_normal((B, D)) * 2).astype(np.float32)
    # an exact tie at the top for row 0: two identical weight rows aligned with the normalized input
    xn0 = V.rms_norm(Xh[:1].astype(np.float64), gam, 1e-6)[0]
    top = np.sign(xn0).astype(np.float32) * 0.25
    i, j = 7, V_ - 3
    W[i] = W[j] = top
    dW, dg = bf16_dev(W), bf16_dev(gam)
    X = torch.from_numpy(Xh).cuda()
    L0 = torch.empty(B, V_, dtype=torch.float32, device="cuda")
    O.nova_op_gemv_fused(X, O.XM_NORM_F32, dW, L0, None, V_, D, B, O.EPI_F32_STORE, gamma=dg, eps=1e-6)
    keys = torch.zeros(B, dtype=torch.int64, device="cuda")
    L1 = torch.empty_like(L0)
    O.nova_op_gemv_fused(X, O.XM_NORM_F32, dW, L1, None, V_, D, B, O.EPI_F32_ARGMAX, gamma=dg, eps=1e-6, keys=keys)
    tok = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    last = torch.full((8,), -1, dtype=torch.int32, device="cuda")
    rows = torch.tensor([[6 - b, 0, 0, 0] for b in range(B)], dtype=torch.int32, device="cuda")
    O.nova_op_argmax_finalize(keys, B, tok, rows, last)
    torch.cuda.synchronize()
    assert torch.equal(L0, L1)
    lg = L1.cpu().numpy()
    ref = V.linear(V.rms_norm(Xh.astype(np.float64), gam, 1e-6), W.astype(np.float64))
    assert rel_inf(lg, ref) <= 1e-4
    toks = tok.cpu().numpy()
    for b in range(B):
        assert toks[b] == V.argmax_lowest(lg[b])
        assert last.cpu().numpy()[6 - b] == toks[b]
    assert lg[0, i] == lg[0, j] and toks[0] == i              # exact tie -> lowest index
    assert int(keys.abs().sum().item()) == 0                  # finalize leaves the keys zeroed


@pytest.mark.parametrize("N,K", [(4608, 3584), (3584, 18944), (37888, 3584), (256, 128), (17920, 1536)])
def test_streaming_layout_gemv_bitwise_equals_rowmajor_and_is_grid_invariant(N, K):
    """block_weights + bulk-copy tiles == tensor-map tiles of the row-major weight (bitwise),
    on every SM budget, and both match the oracle linear."""
    rng = np.random.default_rng(N + 2 * K)
    W = rand_bf16(rng, (N, K), K ** -0.5)
    X = rand_bf16(rng, (16, K))
    dW, dX = bf16_dev(W), bf16_dev(X)
    Wb = torch.empty_like(dW)
    O.nova_op_block_weights(dW, Wb, N, K)
    ref = V.linear(X.astype(np.float64), W.astype(np.float64))
    for B in (1, 7, 16):
        Y0 = torch.empty(B, N, dtype=torch.float32, device="cuda")
        O.nova_op_gemv_tma(dX[:B], dW, Y0, None, N, K, B, O.EPI_F32_STORE)
        torch.cuda.synchronize()
        assert rel_inf(Y0.cpu().numpy(), ref[:B]) <= 1e-4
        # 148: split units only; 24 / 32 / 8: whole-row-block units first, split units for the rest
        for ctas in (148, 32, 24, 8):
            Y1 = torch.empty_like(Y0)
            O.nova_op_gemv_stream(dX[:B], Wb, Y1, None, N, K, B, O.EPI_F32_STORE, max_ctas=ctas)
            torch.cuda.synchronize()
            assert torch.equal(Y0, Y1), (B, ctas)


def test_streaming_lm_head_hi_lo_argmax():
    """Decode lm_head: RMSNorm -> bf16 hi/lo rows -> streaming GEMV with two products ->
    f32 logits within 1e-4 of the oracle and the exact greedy argmax."""
    rng = np.random.default_rng(77)
    V_, D, B = 152064, 3584, 3
    W = rand_bf16(rng, (V_, D), 2 * D ** -0.5)
    gam = _gamma(rng, D)
    Xh = (rng.standard_normal((B, D)) * 2).astype(np.float32)
    dW, dg = bf16_dev(W), bf16_dev(gam)
    Wb = torch.empty_like(dW)
    O.nova_op_block_weights(dW, Wb, V_, D)
    hl = torch.empty(2 * B, D, dtype=torch.bfloat16, device="cuda")
    O.nova_op_rmsnorm(torch.from_numpy(Xh).cuda(), dg, hl, B, D, 1e-6, y_mode=2)
    keys = torch.zeros(B, dtype=torch.int64, device="cuda")
    L = torch.empty(B, V_, dtype=torch.float32, device="cuda")
    O.nova_op_gemv_stream(hl[:B], Wb, L, None, V_, D, B, O.EPI_F32_ARGMAX, X_lo=hl[B:], keys=keys, max_ctas=40)
    tok = torch.empty(B, dtype=torch.int32, device="cuda")
    O.nova_op_argmax_finalize(keys, B, tok)
    torch.cuda.synchronize()
    lg = L.cpu().numpy()
    ref = V.linear(V.rms_norm(Xh.astype(np.float64), gam, 1e-6), W.astype(np.float64))
    assert rel_inf(lg, ref) <= 1e-4
    assert tok.cpu().numpy().tolist() == [V.argmax_lowest(lg[b]) for b in range(B)]
