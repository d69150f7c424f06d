"""Decode GEMV on tcgen05 (csrc/gemv_umma.cu) through the C ABI (include/nova_ops.h
nova_op_gemv_umma) vs the oracle's ops (oracle/vlm.py linear / rms_norm / silu / argmax_lowest):

* f32-store epilogue within 1e-4 (rel-inf) of the fp64 oracle linear on the same bf16 inputs, at
  the 2B / 7B decode shapes and a tiny one (split and unsplit K plans);
* bitwise invariance to the SM budget (the partition) -- whole-block and split units alike -- and
  to the batch composition (row 0 alone == row 0 of a batch of 16);
* SiLU(gate) * up over the interleaved gate|up rows, residual add, and the hi/lo lm_head with
  the fused greedy argmax (exact token, keys left zero).
"""
import numpy as np
import pytest
import torch

from oracle import vlm as V
from tests.gpu_util import bf16_dev, bf16_host, rand_bf16, rel_inf

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2509_21301_b200 import ops as O


def _blocked(W, N, K):
    dW = bf16_dev(W)
    Wb = torch.empty_like(dW)
    O.nova_op_block_weights(dW, Wb, N, K)
    return Wb


@pytest.mark.parametrize("N,K", [(17920, 1536), (1536, 8960), (2048, 1536), (37888, 3584), (3584, 18944),
                                 (256, 128), (768, 128), (384, 320), (1280, 2240)])
def test_umma_gemv_matches_oracle_and_is_grid_and_batch_invariant(N, K):
    rng = np.random.default_rng(3 * N + K)
    W = rand_bf16(rng, (N, K), K ** -0.5)
    X = rand_bf16(rng, (16, K))
    Wb = _blocked(W, N, K)
    dX = bf16_dev(X)
    ref = V.linear(X.astype(np.float64), W.astype(np.float64))
    Y16 = None
    for B in (16, 1, 9):
        Y0 = torch.empty(B, N, dtype=torch.float32, device="cuda")
        O.nova_op_gemv_umma(dX[:B], Wb, Y0, None, N, K, B, O.EPI_F32_STORE)
        torch.cuda.synchronize()
        assert rel_inf(Y0.cpu().numpy(), ref[:B]) <= 1e-4, B
        if Y16 is None:
            Y16 = Y0
        else:
            assert torch.equal(Y0[0], Y16[0]), B          # batch invariance of row 0
        for ctas in (148, 40, 24, 8, 1):                    # stream-K ranges: blocks shared across CTAs
            Y1 = torch.empty_like(Y0)
            O.nova_op_gemv_umma(dX[:B], Wb, Y1, None, N, K, B, O.EPI_F32_STORE, max_ctas=ctas)
            torch.cuda.synchronize()
            assert torch.equal(Y0, Y1), (B, ctas)


def test_umma_stream_k_ranges_any_grid():
    """Item ranges cut blocks at every position (1..37 CTAs of 3 per SM budget unit): the left fold of
    the chunk partials is completed by whichever CTA arrives last -- bitwise the same result."""
    N, K = 640, 1600                                      # 5 blocks x P chunks (25 k-steps, short last chunk)
    P = O.nova_op_gemv_umma_splits(N, K, O.EPI_F32_STORE)
    assert P > 1
    rng = np.random.default_rng(5)
    W = rand_bf16(rng, (N, K), K ** -0.5)
    X = rand_bf16(rng, (3, K))
    Wb, dX = _blocked(W, N, K), bf16_dev(X)
    ref = V.linear(X.astype(np.float64), W.astype(np.float64))
    Y0 = None
    for ctas in (1, 2, 3, 5, 7, 11, 37):
        Y = torch.empty(3, N, dtype=torch.float32, device="cuda")
        O.nova_op_gemv_umma(dX, Wb, Y, None, N, K, 3, O.EPI_F32_STORE, max_ctas=ctas)
        torch.cuda.synchronize()
        assert rel_inf(Y.cpu().numpy(), ref) <= 1e-4, ctas
        if Y0 is None:
            Y0 = Y
        assert torch.equal(Y, Y0), ctas


def test_umma_gemv_silu_and_residual_epilogues():
    rng = np.random.default_rng(11)
    F, D, B = 8960, 1536, 5
    G = rand_bf16(rng, (F, D), D ** -0.5)
    U = rand_bf16(rng, (F, D), D ** -0.5)
    Wgu = np.empty((2 * F, D), dtype=np.float32)         # interleave 16 gate | 16 up rows (engine layout)
    for i in range(F // 16):
        Wgu[32 * i:32 * i + 16] = G[16 * i:16 * i + 16]
        Wgu[32 * i + 16:32 * i + 32] = U[16 * i:16 * i + 16]
    X = rand_bf16(rng, (B, D))
    Wb = _blocked(Wgu, 2 * F, D)
    act = torch.empty(B, F, dtype=torch.bfloat16, device="cuda")
    O.nova_op_gemv_umma(bf16_dev(X), Wb, act, None, 2 * F, D, B, O.EPI_BF16_SILUMUL, max_ctas=32)
    torch.cuda.synchronize()
    x64 = X.astype(np.float64)
    ref = V.silu(V.linear(x64, G.astype(np.float64))) * V.linear(x64, U.astype(np.float64))
    assert rel_inf(bf16_host(act), ref) <= 8e-3
    # residual: Y += X W^T (f32)
    Wd = rand_bf16(rng, (D, F), F ** -0.5)
    Xa = rand_bf16(rng, (B, F))
    base = rng.standard_normal((B, D)).astype(np.float32)
    Y = torch.from_numpy(base.copy()).cuda()
    O.nova_op_gemv_umma(bf16_dev(Xa), _blocked(Wd, D, F), Y, None, D, F, B, O.EPI_F32_RESID, max_ctas=24)
    torch.cuda.synchronize()
    ref2 = base.astype(np.float64) + V.linear(Xa.astype(np.float64), Wd.astype(np.float64))
    assert rel_inf(Y.cpu().numpy(), ref2) <= 1e-4


def test_umma_lm_head_hi_lo_argmax():
    rng = np.random.default_rng(78)
    V_, D, B = 151936, 1536, 3
    W = rand_bf16(rng, (V_, D), 2 * D ** -0.5)
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    gam = bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (D,), 0.1) + 1.0))
    Xh = (rng.standard_normal((B, D)) * 2).astype(np.float32)
    Wb = _blocked(W, V_, D)
    hl = torch.empty(2 * B, D, dtype=torch.bfloat16, device="cuda")
    O.nova_op_rmsnorm(torch.from_numpy(Xh).cuda(), bf16_dev(gam), hl, B, D, 1e-6, y_mode=2)
    keys = torch.zeros(B, dtype=torch.int64, device="cuda")
    L = torch.empty(B, V_, dtype=torch.float32, device="cuda")
    O.nova_op_gemv_umma(hl[:B], Wb, L, None, V_, D, B, O.EPI_F32_ARGMAX, X_lo=hl[B:], keys=keys, max_ctas=32)
    tok = torch.empty(B, dtype=torch.int32, device="cuda")
    O.nova_op_argmax_finalize(keys, B, tok)
    torch.cuda.synchronize()
    lg = L.cpu().numpy()
    ref = V.linear(V.rms_norm(Xh.astype(np.float64), gam, 1e-6), W.astype(np.float64))
    assert rel_inf(lg, ref) <= 1e-4
    assert tok.cpu().numpy().tolist() == [V.argmax_lowest(lg[b]) for b in range(B)]
    assert int(keys.abs().sum().item()) == 0


@pytest.mark.parametrize("F,D,B", [(8960, 1536, 2), (8960, 1536, 16), (192, 128, 3)])
def test_umma_gate_up_with_folded_rmsnorm(F, D, B):
    """DESIGN R25: x~ = bf16(h * gamma) through the GEMV, rows scaled by rsqrt(mean h^2 + eps) after it
    == RMSNorm(h) then gate|up (oracle rms_norm / linear / silu), bf16 rel-inf <= 8e-3; and bitwise
    invariant to the SM budget."""
    rng = np.random.default_rng(F + B)
    G = rand_bf16(rng, (F, D), D ** -0.5)
    U = rand_bf16(rng, (F, D), D ** -0.5)
    Wgu = np.empty((2 * F, D), dtype=np.float32)
    for i in range(F // 16):
        Wgu[32 * i:32 * i + 16] = G[16 * i:16 * i + 16]
        Wgu[32 * i + 16:32 * i + 32] = U[16 * i:16 * i + 16]
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    gam = bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (D,), 0.1) + 1.0))
    h = (rng.standard_normal((B, D)) * 3).astype(np.float32)
    xt = bf16_bits_to_f32(f32_to_bf16_bits(h * gam))                      # x~ = bf16(h * gamma)
    Wb = _blocked(Wgu, 2 * F, D)
    dh, dx = torch.from_numpy(h).cuda(), bf16_dev(xt)
    outs = []
    for ctas in (0, 24):
        act = torch.empty(B, F, dtype=torch.bfloat16, device="cuda")
        O.nova_op_gemv_umma(dx, Wb, act, None, 2 * F, D, B, O.EPI_BF16_SILUMUL, max_ctas=ctas, norm_hid=dh,
                            norm_eps=1e-6)
        torch.cuda.synchronize()
        outs.append(act)
    assert torch.equal(outs[0], outs[1])
    xn = V.rms_norm(h.astype(np.float64), gam, 1e-6)
    ref = V.silu(V.linear(xn, G.astype(np.float64))) * V.linear(xn, U.astype(np.float64))
    assert rel_inf(bf16_host(outs[0]), ref) <= 8e-3


@pytest.mark.parametrize("D,F,B", [(1536, 8960, 2), (3584, 3584, 16), (128, 256, 3)])
def test_umma_resid_writes_next_norm_input(D, F, B):
    """DESIGN R25, the o-proj half of the fold: Y += X W^T (f32, oracle linear) and nxout = bf16(Y_new * gamma),
    bitwise against the host rounding of the GPU's own Y_new; bitwise invariant to the SM budget."""
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    rng = np.random.default_rng(D + F + B)
    Wd = rand_bf16(rng, (D, F), F ** -0.5)
    Xa = rand_bf16(rng, (B, F))
    gam = bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (D,), 0.1) + 1.0))
    base = rng.standard_normal((B, D)).astype(np.float32)
    Wb = _blocked(Wd, D, F)
    got = []
    for ctas in (0, 24):
        Y = torch.from_numpy(base.copy()).cuda()
        nx = torch.zeros(B, D, dtype=torch.bfloat16, device="cuda")
        O.nova_op_gemv_umma(bf16_dev(Xa), Wb, Y, None, D, F, B, O.EPI_F32_RESID, max_ctas=ctas,
                            ngamma=bf16_dev(gam), nxout=nx)
        torch.cuda.synchronize()
        got.append((Y, nx))
    assert torch.equal(got[0][0], got[1][0]) and torch.equal(got[0][1], got[1][1])
    Y, nx = got[0][0].cpu().numpy(), got[0][1]
    ref = base.astype(np.float64) + V.linear(Xa.astype(np.float64), Wd.astype(np.float64))
    assert rel_inf(Y, ref) <= 1e-4
    want = f32_to_bf16_bits((Y * gam).astype(np.float32))
    assert np.array_equal(nx.view(torch.int16).cpu().numpy().view(np.uint16), want)


@pytest.mark.parametrize("H,KV,D", [(12, 2, 1536), (28, 4, 3584), (2, 1, 256)])
def test_umma_qkv_folded_rmsnorm_rope_kv_append(H, KV, D):
    """Decode qkv on tcgen05: x~ = bf16(h * ln1) (scale_rows_bf16), the RMSNorm row scale
    folded after the GEMV (R25), + bias, RoPE at pos on q / k, k / v appended to the paged cache -- vs the
    oracle (rms_norm, linear, mrope_tables / apply_rope at t = h = w), bf16 rel-inf <= 8e-3; bitwise
    invariant to the SM budget and to the batch composition (row 0)."""
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    hd, n_pages, max_pages, theta, eps = 128, 64, 8, 1e6, 1e-6
    rng = np.random.default_rng(H * 11 + D)
    N = (H + 2 * KV) * hd
    W = rand_bf16(rng, (N, D), D ** -0.5)
    bias = rand_bf16(rng, (N,), 0.05)
    gam = bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (D,), 0.1) + 1.0))
    bt = torch.from_numpy(rng.permutation(n_pages)[:4 * max_pages].reshape(4, max_pages).astype(np.int32)).cuda()
    Wb, db, dg = _blocked(W, N, D), bf16_dev(bias), bf16_dev(gam)
    Xh = (rng.standard_normal((16, D)) * 2).astype(np.float32)
    got0 = None
    for B, ctas in ((1, 0), (4, 24), (16, 0), (16, 40)):
        r = np.array([[b % 4, 320 + b, int(rng.integers(0, 3000)), 0] for b in range(B)], np.int32)
        r[:min(B, 4), 1] = [0, 63, 64, 300][:min(B, 4)]    # page boundaries
        r[0, 2] = 1234
        pool = torch.zeros(2, n_pages, 2, KV, 64, hd, dtype=torch.bfloat16, device="cuda")
        rows = torch.from_numpy(r).cuda()
        Q = torch.zeros(B, N, dtype=torch.bfloat16, device="cuda")
        hd_ = torch.from_numpy(Xh[:B]).cuda()
        xt = torch.empty(B, D, dtype=torch.bfloat16, device="cuda")
        O.nova_op_scale_rows_bf16(hd_, dg, xt, B, D)
        O.nova_op_gemv_umma_qkv(xt, Wb, Q, db, N, D, B, hd_, eps, H, KV, hd, theta, rows, pool, 1, n_pages, bt,
                                max_ctas=ctas)
        torch.cuda.synchronize()
        assert np.array_equal(xt.view(torch.int16).cpu().numpy().view(np.uint16),
                              f32_to_bf16_bits((Xh[:B] * gam).astype(np.float32)))
        xn = V.rms_norm(Xh[:B].astype(np.float64), gam, eps)
        y = V.linear(xn, W.astype(np.float64), bias.astype(np.float64))
        pos3 = np.tile(r[:, 2], (3, 1))
        c, s = V.mrope_tables(pos3, hd, theta, (hd // 2, 0, 0), np.float64)
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
        assert torch.equal(row0, got0)
