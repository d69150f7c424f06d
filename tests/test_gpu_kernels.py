"""Per-kernel parity (GPU): each libnova kernel vs the oracle's op on the same bf16
inputs, through the C ABI (include/nova_ops.h).  Tolerances (SURVEY.md §8(c) c6,
DESIGN.md "Tolerances"): bf16 outputs rel-inf <= 8e-3 (~2 output ulps), f32
outputs rel-inf <= 1e-4 (accumulation-order only); argmax/indices exact; grid
and batch invariance bitwise."""
import numpy as np
import pytest
import torch

from oracle import vlm as V
from tests.gpu_util import bf16_dev, bf16_host, rand_bf16, rel_inf

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2509_21301_b200 import ops as O


def interleave_gate_up(wg: np.ndarray, wu: np.ndarray, blk: int = 16) -> np.ndarray:
    F, K = wg.shape
    out = np.empty((2 * F, K), wg.dtype)
    for b in range(F // blk):
        out[2 * b * blk:(2 * b + 1) * blk] = wg[b * blk:(b + 1) * blk]
        out[(2 * b + 1) * blk:(2 * b + 2) * blk] = wu[b * blk:(b + 1) * blk]
    return out


GEMM_SHAPES = [(16, 64, 64), (12, 256, 128), (200, 384, 1176), (1286, 4608, 3584), (777, 1280, 5120), (4888, 3840, 1280),
               (300, 1216, 200), (513, 448, 64)]


@pytest.fixture(params=[0, 1, 2], ids=["auto", "cta1", "pair"])
def gemm_mode(request):
    """Tile family: automatic, single-CTA 128 x BN only, CTA-pair (cta_group::2) 256 x BN only."""
    prev = O.nova_op_gemm_mode(request.param)
    yield request.param
    O.nova_op_gemm_mode(prev)


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_tc_epilogues(M, N, K, gemm_mode):
    if gemm_mode == 1 and N % 64:
        pytest.skip("single-CTA tiles need N % 64 == 0")
    rng = np.random.default_rng(M + N + K)
    A = rand_bf16(rng, (M, K))
    W = rand_bf16(rng, (N, K), K ** -0.5)
    b = rand_bf16(rng, (N,), 0.1)
    ref = V.linear(A.astype(np.float64), W.astype(np.float64), b.astype(np.float64))
    dA, dW, db = bf16_dev(A), bf16_dev(W), bf16_dev(b)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    for epi, f in [(O.EPI_BF16, lambda z: z), (O.EPI_BF16_QGELU, V.quick_gelu), (O.EPI_BF16_GELU, V.gelu_erf)]:
        O.nova_op_gemm(dA, dW, C, db, M, N, K, epi)
        torch.cuda.synchronize()
        assert rel_inf(bf16_host(C), f(ref)) <= 8e-3, epi
    R0 = torch.from_numpy(rng.standard_normal((M, N)).astype(np.float32)).cuda()
    R = R0.clone()
    O.nova_op_gemm(dA, dW, R, db, M, N, K, O.EPI_F32_RESID)
    torch.cuda.synchronize()
    assert rel_inf(R.cpu().numpy(), R0.cpu().numpy() + ref) <= 1e-4
    Fo = torch.empty(M, N, dtype=torch.float32, device="cuda")
    O.nova_op_gemm(dA, dW, Fo, None, M, N, K, O.EPI_F32_STORE)
    torch.cuda.synchronize()
    ref_nb = V.linear(A.astype(np.float64), W.astype(np.float64))
    assert rel_inf(Fo.cpu().numpy(), ref_nb) <= 1e-4


@pytest.mark.parametrize("M,F,K", [(300, 512, 384), (1286, 1216, 448)])
def test_gemm_silu_mul_and_grid_invariance(M, F, K, gemm_mode):
    rng = np.random.default_rng(7)
    A = rand_bf16(rng, (M, K))
    Wg, Wu = rand_bf16(rng, (F, K), K ** -0.5), rand_bf16(rng, (F, K), K ** -0.5)
    Wi = interleave_gate_up(Wg, Wu)
    a64 = A.astype(np.float64)
    ref = V.silu(a64 @ Wg.T.astype(np.float64)) * (a64 @ Wu.T.astype(np.float64))
    dA, dW = bf16_dev(A), bf16_dev(Wi)
    outs = []
    for ctas in (148, 37, 5, 1):
        C = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
        O.nova_op_gemm(dA, dW, C, None, M, 2 * F, K, O.EPI_BF16_SILUMUL, max_ctas=ctas)
        torch.cuda.synchronize()
        outs.append(C.view(torch.int16).cpu())
    assert rel_inf(bf16_host(C), ref) <= 8e-3
    for o in outs[1:]:
        assert torch.equal(o, outs[0])           # bitwise SM-budget invariance


@pytest.mark.parametrize("N,K", [(256, 128), (4608, 3584), (3584, 18944), (512, 128), (2048, 1536)])
def test_gemv_and_batch_invariance(N, K):
    rng = np.random.default_rng(N + K)
    W = rand_bf16(rng, (N, K), K ** -0.5)
    b = rand_bf16(rng, (N,), 0.1)
    X = rand_bf16(rng, (16, K))
    dW, db, dX = bf16_dev(W), bf16_dev(b), bf16_dev(X)
    ref = V.linear(X.astype(np.float64), W.astype(np.float64), b.astype(np.float64))
    rows = {}
    for B in (1, 3, 8, 11, 16):
        Y = torch.empty(B, N, dtype=torch.float32, device="cuda")
        O.nova_op_gemv(dX[:B], dW, Y, db, N, K, B, O.EPI_F32_STORE)
        torch.cuda.synchronize()
        y = Y.cpu().numpy()
        assert rel_inf(y, ref[:B]) <= 1e-4
        rows[B] = y
    for B in (3, 8, 11, 16):
        assert np.array_equal(rows[B][0], rows[1][0])   # bitwise batch invariance
    Yb = torch.empty(5, N, dtype=torch.bfloat16, device="cuda")
    O.nova_op_gemv(dX[:5], dW, Yb, db, N, K, 5, O.EPI_BF16)
    torch.cuda.synchronize()
    assert rel_inf(bf16_host(Yb), ref[:5]) <= 8e-3
    R0 = torch.randn(5, N, device="cuda")
    R = R0.clone()
    O.nova_op_gemv(dX[:5], dW, R, db, N, K, 5, O.EPI_F32_RESID)
    torch.cuda.synchronize()
    assert rel_inf(R.cpu().numpy(), R0.cpu().numpy() + ref[:5]) <= 1e-4


@pytest.mark.parametrize("N,K", [(256, 128), (4608, 3584), (3584, 18944), (2048, 1536), (37888, 3584)])
def test_gemv_tma_matches_oracle_and_is_invariant(N, K):
    rng = np.random.default_rng(N * 3 + K)
    W = rand_bf16(rng, (N, K), K ** -0.5)
    b = rand_bf16(rng, (N,), 0.1)
    X = rand_bf16(rng, (16, K))
    dW, db, dX = bf16_dev(W), bf16_dev(b), bf16_dev(X)
    ref = V.linear(X.astype(np.float64), W.astype(np.float64), b.astype(np.float64))
    rows = {}
    for B in (1, 5, 8, 9, 16):
        Y = torch.empty(B, N, dtype=torch.float32, device="cuda")
        O.nova_op_gemv_tma(dX[:B], dW, Y, db, N, K, B, O.EPI_F32_STORE)
        torch.cuda.synchronize()
        rows[B] = Y.cpu().numpy()
        assert rel_inf(rows[B], ref[:B]) <= 1e-4
    for B in (5, 8, 9, 16):
        assert np.array_equal(rows[B][0], rows[1][0])      # bitwise batch invariance
    for ctas in (148, 37, 8):   # deterministic re-run on any SM budget (persistent grid)
        Y2 = torch.empty(16, N, dtype=torch.float32, device="cuda")
        O.nova_op_gemv_tma(dX, dW, Y2, db, N, K, 16, O.EPI_F32_STORE, max_ctas=ctas)
        torch.cuda.synchronize()
        assert np.array_equal(Y2.cpu().numpy(), rows[16]), ctas
    R0 = torch.randn(3, N, device="cuda")
    R = R0.clone()
    O.nova_op_gemv_tma(dX[:3], dW, R, db, N, K, 3, O.EPI_F32_RESID)
    Yb = torch.empty(3, N, dtype=torch.bfloat16, device="cuda")
    O.nova_op_gemv_tma(dX[:3], dW, Yb, db, N, K, 3, O.EPI_BF16)
    torch.cuda.synchronize()
    assert rel_inf(R.cpu().numpy(), R0.cpu().numpy() + ref[:3]) <= 1e-4
    assert rel_inf(bf16_host(Yb), ref[:3]) <= 8e-3
    if N % 64 == 0 and N >= 256:
        F = N // 2
        Wg, Wu = W[:F], W[F:]
        Yg = torch.empty(4, F, dtype=torch.bfloat16, device="cuda")
        O.nova_op_gemv_tma(dX[:4], bf16_dev(interleave_gate_up(Wg, Wu)), Yg, None, N, K, 4, O.EPI_BF16_SILUMUL)
        torch.cuda.synchronize()
        x64 = X[:4].astype(np.float64)
        refg = V.silu(x64 @ Wg.T.astype(np.float64)) * (x64 @ Wu.T.astype(np.float64))
        assert rel_inf(bf16_host(Yg), refg) <= 8e-3


def test_gemv_f32_input_and_silu():
    rng = np.random.default_rng(3)
    N, K = 512, 256
    W = rand_bf16(rng, (N, K), K ** -0.5)
    Xf = rng.standard_normal((4, K)).astype(np.float32)     # f32 activations (lm_head input)
    Y = torch.empty(4, N, dtype=torch.float32, device="cuda")
    O.nova_op_gemv(torch.from_numpy(Xf).cuda(), bf16_dev(W), Y, None, N, K, 4, O.EPI_F32_STORE)
    torch.cuda.synchronize()
    ref = Xf.astype(np.float64) @ W.T.astype(np.float64)
    assert rel_inf(Y.cpu().numpy(), ref) <= 2e-4             # hi/lo split keeps ~16 bits of x
    F = 256
    Wg, Wu = rand_bf16(rng, (F, K), K ** -0.5), rand_bf16(rng, (F, K), K ** -0.5)
    X = rand_bf16(rng, (9, K))
    Yb = torch.empty(9, F, dtype=torch.bfloat16, device="cuda")
    O.nova_op_gemv(bf16_dev(X), bf16_dev(interleave_gate_up(Wg, Wu)), Yb, None, 2 * F, K, 9, O.EPI_BF16_SILUMUL)
    torch.cuda.synchronize()
    x64 = X.astype(np.float64)
    ref = V.silu(x64 @ Wg.T.astype(np.float64)) * (x64 @ Wu.T.astype(np.float64))
    assert rel_inf(bf16_host(Yb), ref) <= 8e-3


@pytest.mark.parametrize("S,H,KV,hd,causal", [(16, 4, 4, 16, 0), (300, 4, 4, 16, 0), (12, 4, 2, 32, 1),
                                               (1286, 12, 2, 128, 1), (777, 16, 16, 80, 0), (130, 28, 4, 128, 1),
                                               (4888, 2, 2, 80, 0), (500, 4, 4, 128, 0), (100, 3, 3, 80, 0)])
def test_flash_attn(S, H, KV, hd, causal):
    rng = np.random.default_rng(S + hd)
    qkv = rand_bf16(rng, (S, (H + 2 * KV) * hd))
    d = bf16_dev(qkv)
    out = torch.empty(S, H * hd, dtype=torch.bfloat16, device="cuda")
    O.nova_op_flash_attn(d, out, S, H, KV, hd, causal)
    torch.cuda.synchronize()
    q = qkv[:, :H * hd].reshape(S, H, hd).astype(np.float64)
    k = qkv[:, H * hd:(H + KV) * hd].reshape(S, KV, hd).astype(np.float64)
    v = qkv[:, (H + KV) * hd:].reshape(S, KV, hd).astype(np.float64)
    if causal:
        ref = V.attention_causal_gqa(q, k, v, hd ** -0.5, 0)
    else:
        ref = V.attention_full(q, np.repeat(k, H // KV, 1), np.repeat(v, H // KV, 1), hd ** -0.5)
    assert rel_inf(bf16_host(out).reshape(S, H, hd), ref) <= 2e-2   # P rounded to bf16 before PV


@pytest.mark.parametrize("S,H,KV,hd,causal", [(300, 2, 2, 80, 0), (131, 4, 2, 128, 1), (1286, 28, 4, 128, 1)])
def test_flash_attn_mma_baseline_matches_oracle(S, H, KV, hd, causal):
    """The legacy mma.sync kernel (kept as the measured baseline) on the tcgen05 head dims."""
    rng = np.random.default_rng(S * 7 + hd)
    qkv = rand_bf16(rng, (S, (H + 2 * KV) * hd))
    out = torch.empty(S, H * hd, dtype=torch.bfloat16, device="cuda")
    O.nova_op_flash_attn_mma(bf16_dev(qkv), out, S, H, KV, hd, causal)
    torch.cuda.synchronize()
    q = qkv[:, :H * hd].reshape(S, H, hd).astype(np.float64)
    k = qkv[:, H * hd:(H + KV) * hd].reshape(S, KV, hd).astype(np.float64)
    v = qkv[:, (H + KV) * hd:].reshape(S, KV, hd).astype(np.float64)
    ref = V.attention_causal_gqa(q, k, v, hd ** -0.5, 0) if causal else \
        V.attention_full(q, np.repeat(k, H // KV, 1), np.repeat(v, H // KV, 1), hd ** -0.5)
    assert rel_inf(bf16_host(out).reshape(S, H, hd), ref) <= 2e-2


def test_flash_attn_tc_large_logits_rescale():
    """Row maxima that grow along the key axis force the lazy O rescaling path (> 2^8)."""
    rng = np.random.default_rng(99)
    S, H, hd = 700, 2, 80
    qkv = rand_bf16(rng, (S, 3 * H * hd))
    ramp = np.linspace(0, 6, S)[:, None]                    # later keys have larger logits
    qkv[:, H * hd:2 * H * hd] = rand_bf16(rng, (S, H * hd)) + ramp
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    qkv = bf16_bits_to_f32(f32_to_bf16_bits(qkv.astype(np.float32)))
    out = torch.empty(S, H * hd, dtype=torch.bfloat16, device="cuda")
    O.nova_op_flash_attn(bf16_dev(qkv), out, S, H, H, hd, 0)
    torch.cuda.synchronize()
    t = qkv.reshape(S, 3, H, hd).astype(np.float64)
    ref = V.attention_full(t[:, 0] * 3, t[:, 1], t[:, 2], hd ** -0.5) if False else \
        V.attention_full(t[:, 0], t[:, 1], t[:, 2], hd ** -0.5)
    assert rel_inf(bf16_host(out).reshape(S, H, hd), ref) <= 2e-2


def _pool_setup(rng, L, n_pages, KV, hd):
    return torch.zeros(L, n_pages, 2, KV, 64, hd, dtype=torch.bfloat16, device="cuda")


def test_llm_rope_kv_and_decode_attention():
    rng = np.random.default_rng(11)
    H, KV, hd, L, n_pages = 8, 2, 32, 2, 16
    sec = (4, 6, 6)
    S = 150
    qkv = rand_bf16(rng, (S, (H + 2 * KV) * hd))
    pos3 = V.mrope_positions(8, 6, S - 12, 2)          # 12 vision tokens + text
    bt = torch.tensor([[5, 9, 2, 7], [1, 3, 11, 0]], dtype=torch.int32, device="cuda")
    pool = _pool_setup(rng, L, n_pages, KV, hd)
    d = bf16_dev(qkv)
    O.nova_op_llm_rope_kv(d, S, H, KV, hd, 1e6, sec[0], sec[1], torch.from_numpy(pos3.astype(np.int32)).cuda(),
                          None, 0, 0, pool, 1, n_pages, bt)
    torch.cuda.synchronize()
    c, s = V.mrope_tables(pos3, hd, 1e6, sec, np.float64)
    q = qkv[:, :H * hd].reshape(S, H, hd).astype(np.float64)
    k = qkv[:, H * hd:(H + KV) * hd].reshape(S, KV, hd).astype(np.float64)
    v = qkv[:, (H + KV) * hd:].reshape(S, KV, hd)
    qr, kr = V.apply_rope(q, c, s), V.apply_rope(k, c, s)
    got = bf16_host(d)
    assert rel_inf(got[:, :H * hd].reshape(S, H, hd), qr) <= 8e-3
    assert rel_inf(got[:, H * hd:(H + KV) * hd].reshape(S, KV, hd), kr) <= 8e-3
    P = bf16_host(pool[1])                              # [pages][2][KV][64][hd]
    btn = bt.cpu().numpy()[0]
    kc = np.stack([P[btn[t // 64], 0, :, t % 64] for t in range(S)])
    vc = np.stack([P[btn[t // 64], 1, :, t % 64] for t in range(S)])
    assert np.array_equal(kc, got[:, H * hd:(H + KV) * hd].reshape(S, KV, hd))
    assert np.array_equal(vc, v)
    # one decode step for slot 0 at cache index S-1 (keys 0..S-1) using the cached K/V
    qd = rand_bf16(rng, (1, (H + 2 * KV) * hd))
    rows = torch.tensor([[0, S - 1, 0, 0]], dtype=torch.int32, device="cuda")
    out = torch.empty(1, H * hd, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(64 * H * (hd + 2), dtype=torch.float32, device="cuda")
    O.nova_op_decode_attn(bf16_dev(qd), out, pool, 1, n_pages, H, KV, hd, bt, rows, 1, S - 1, ws)
    torch.cuda.synchronize()
    ref = V.attention_causal_gqa(qd[:, :H * hd].reshape(1, H, hd).astype(np.float64), kc.astype(np.float64),
                                 vc.astype(np.float64), hd ** -0.5, S - 1)
    assert rel_inf(bf16_host(out).reshape(1, H, hd), ref) <= 8e-3


@pytest.mark.parametrize("H,KV", [(28, 4), (12, 2)])
def test_decode_attention_long_context_7b_shape(H, KV):
    """7B / 2B head shapes vs the oracle; bitwise equal on the whole GPU (cluster kernel, 2-stage ring) and
    on 8- / 24- / 40-SM budgets (1-stage ring, two CTAs per SM; the virtual-CTA kernel with fewer physical
    CTAs per (request, KV head) and the workspace merge)."""
    rng = np.random.default_rng(12)
    hd, n_pages = 128, 128
    ctxs = [1333, 17, 640, 2047]
    B = len(ctxs)
    pool_np = rand_bf16(rng, (1, n_pages, 2, KV, 64, hd))
    pool = bf16_dev(pool_np)
    perm = rng.permutation(n_pages).astype(np.int32)
    bt = torch.from_numpy(perm.reshape(4, 32).copy()).cuda()
    qd = rand_bf16(rng, (B, (H + 2 * KV) * hd))
    rows = torch.tensor([[b, ctxs[b], 0, 0] for b in range(B)], dtype=torch.int32, device="cuda")
    out = torch.empty(B, H * hd, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(B * H * 80 * (hd + 2), dtype=torch.float32, device="cuda")
    O.nova_op_decode_attn(bf16_dev(qd), out, pool, 0, n_pages, H, KV, hd, bt, rows, B, max(ctxs), ws)
    for ctas in (4, 8, 24, 40):   # virtual-CTA kernel (1 / 2 physical CTAs per (request, KV head)); 1-stage ring
        out8 = torch.empty_like(out)
        O.nova_op_decode_attn(bf16_dev(qd), out8, pool, 0, n_pages, H, KV, hd, bt, rows, B, max(ctxs), ws,
                              max_ctas=ctas)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), out8.view(torch.int16)), ctas
    btn = bt.cpu().numpy()
    for b, ctx in enumerate(ctxs):
        kc = np.stack([pool_np[0, btn[b, t // 64], 0, :, t % 64] for t in range(ctx + 1)]).astype(np.float64)
        vc = np.stack([pool_np[0, btn[b, t // 64], 1, :, t % 64] for t in range(ctx + 1)]).astype(np.float64)
        ref = V.attention_causal_gqa(qd[b:b + 1, :H * hd].reshape(1, H, hd).astype(np.float64), kc, vc,
                                     hd ** -0.5, ctx)
        assert rel_inf(bf16_host(out[b:b + 1]).reshape(1, H, hd), ref) <= 8e-3


def test_norms_patchify_vitrope_embed_argmax():
    rng = np.random.default_rng(5)
    M, d = 37, 1280
    x = rng.standard_normal((M, d)).astype(np.float32) * 3
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    g = bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (d,), 0.1) + 1))   # gamma exactly representable
    b = rand_bf16(rng, (d,), 0.05)
    y = torch.empty(M, d, dtype=torch.bfloat16, device="cuda")
    O.nova_op_layernorm(torch.from_numpy(x).cuda(), bf16_dev(g), bf16_dev(b), y, M, d, 1e-6)
    torch.cuda.synchronize()
    assert rel_inf(bf16_host(y), V.layer_norm(x.astype(np.float64), g, b, 1e-6)) <= 8e-3
    yf = torch.empty(M, d, dtype=torch.float32, device="cuda")
    O.nova_op_rmsnorm(torch.from_numpy(x).cuda(), bf16_dev(g), yf, M, d, 1e-6)
    torch.cuda.synchronize()
    assert rel_inf(yf.cpu().numpy(), V.rms_norm(x.astype(np.float64), g, 1e-6)) <= 1e-5
    # patchify: grid 6 x 8 patches of 14 px
    from synth import TINY
    pix = rand_bf16(rng, (3, 6 * 14, 8 * 14))
    X0 = torch.empty(48, 1176, dtype=torch.bfloat16, device="cuda")
    O.nova_op_patchify(bf16_dev(pix), 14, 2, 2, X0)
    torch.cuda.synchronize()
    ref, _, hp, wp = V.patchify(pix, TINY)
    assert np.array_equal(bf16_host(X0), ref)
    # ViT rope on qkv [48][3][4][16]
    qkv = rand_bf16(rng, (48, 3 * 4 * 16))
    dq = bf16_dev(qkv)
    O.nova_op_vit_rope(dq, 48, 4, 16, 8, 2, 1e4)
    torch.cuda.synchronize()
    c, s = V.vit_rope_tables(hp, wp, 16, 1e4, np.float64)
    t = qkv.reshape(48, 3, 4, 16).astype(np.float64)
    got = bf16_host(dq).reshape(48, 3, 4, 16)
    assert rel_inf(got[:, 0], V.apply_rope(t[:, 0], c, s)) <= 8e-3
    assert rel_inf(got[:, 1], V.apply_rope(t[:, 1], c, s)) <= 8e-3
    assert np.array_equal(got[:, 2], t[:, 2])
    # embedding + argmax (ties -> lowest index)
    table = rand_bf16(rng, (100, 64))
    ids = torch.tensor([3, 99, 0, 3], dtype=torch.int32, device="cuda")
    out = torch.empty(4, 64, dtype=torch.float32, device="cuda")
    O.nova_op_embed(bf16_dev(table), 64, ids, None, None, out, 4)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), table[[3, 99, 0, 3]])
    lg = rng.standard_normal((3, 152064)).astype(np.float32)
    lg[1, 7] = lg[1, 150000] = lg[1].max() + 1       # tie
    tok = torch.empty(3, dtype=torch.int32, device="cuda")
    O.nova_op_argmax(torch.from_numpy(lg).cuda(), 152064, 3, tok)
    torch.cuda.synchronize()
    assert tok.cpu().tolist() == [V.argmax_lowest(r) for r in lg]
    assert tok.cpu().tolist()[1] == 7


def test_flash_attn_vit_shape_grid_invariant():
    """ViT shape (N = 4888, 16 heads, hd 80): the persistent kernel's tail units are split along
    keys and merged; output must not depend on the SM budget, and matches the oracle on the
    heads that take the split path (head 15) and the whole-range path (head 0)."""
    rng = np.random.default_rng(4888)
    S, H, hd = 4888, 16, 80
    qkv = rand_bf16(rng, (S, 3 * H * hd))
    d = bf16_dev(qkv)
    outs = []
    for ctas in (148, 100, 37):
        out = torch.empty(S, H * hd, dtype=torch.bfloat16, device="cuda")
        O.nova_op_flash_attn(d, out, S, H, H, hd, 0, max_ctas=ctas)
        torch.cuda.synchronize()
        outs.append(out)
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16))
    t = qkv.reshape(S, 3, H, hd)
    got = bf16_host(outs[0]).reshape(S, H, hd)
    for h in (0, 15):
        ref = V.attention_full(t[:, 0, h:h + 1].astype(np.float64), t[:, 1, h:h + 1].astype(np.float64),
                               t[:, 2, h:h + 1].astype(np.float64), hd ** -0.5)
        assert rel_inf(got[:, h:h + 1], ref) <= 2e-2, h


@pytest.mark.parametrize("S,H,KV", [(1286, 28, 4), (2044, 28, 4), (257, 28, 4), (1286, 12, 2), (700, 12, 2)])
def test_flash_attn_prefill_causal_grid_invariant(S, H, KV):
    """7B / 2B prefill shapes (hd 128, causal): the persistent tcgen05 kernel runs the Q-tile pairs
    longest first in a snake order over the CTAs, the longest cut into key chunks merged in chunk
    order (shape-only plan); output must not depend on the SM budget and matches the oracle on the
    first and last head of two KV groups."""
    rng = np.random.default_rng(S + H)
    hd = 128
    qkv = rand_bf16(rng, (S, (H + 2 * KV) * hd))
    d = bf16_dev(qkv)
    outs = []
    for ctas in (148, 100, 37, 8):
        out = torch.empty(S, H * hd, dtype=torch.bfloat16, device="cuda")
        O.nova_op_flash_attn(d, out, S, H, KV, hd, 1, max_ctas=ctas)
        torch.cuda.synchronize()
        outs.append(out)
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16))
    got = bf16_host(outs[0]).reshape(S, H, hd)
    q = qkv[:, :H * hd].reshape(S, H, hd).astype(np.float64)
    k = qkv[:, H * hd:(H + KV) * hd].reshape(S, KV, hd).astype(np.float64)
    v = qkv[:, (H + KV) * hd:].reshape(S, KV, hd).astype(np.float64)
    for h in (0, H // KV - 1, H // KV, H - 1):
        g = h // (H // KV)
        ref = V.attention_causal_gqa(q[:, h:h + 1], k[:, g:g + 1], v[:, g:g + 1], hd ** -0.5, 0)
        assert rel_inf(got[:, h:h + 1], ref) <= 2e-2, h


@pytest.mark.parametrize("M,D,F,ctas", [(1286, 1536, 8960, 148), (300, 3584, 18944, 40), (12, 128, 384, 148)])
def test_prefill_rmsnorm_fold_gemms(M, D, F, ctas):
    """DESIGN R25 on the prefill GEMMs: (1) rms_prep: x~ = bf16(h * ln1) bitwise, 32-column sums of squares;
    (2) a residual GEMM (o-proj shape) writing h_new, the next x~ = bf16(h_new * ln2) (bitwise vs the host
    rounding of the GPU's h_new) and its chunk sums; (3) qkv (bias) and gate|up (SiLU * up) GEMMs on x~ with
    the row scale folded after the GEMM vs the oracle's rms_norm -> linear (bf16 rel-inf <= 8e-3); and the
    results bitwise independent of the SM budget."""
    from synth.weights import bf16_bits_to_f32, f32_to_bf16_bits
    rng = np.random.default_rng(M + D)
    eps = 1e-6
    g1 = bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (D,), 0.1) + 1.0))
    g2 = bf16_bits_to_f32(f32_to_bf16_bits(rand_bf16(rng, (D,), 0.1) + 1.0))
    h = (rng.standard_normal((M, D)) * 2).astype(np.float32)
    nt = D // 32
    dh = torch.from_numpy(h).cuda()
    xt = torch.empty(M, D, dtype=torch.bfloat16, device="cuda")
    ss = torch.empty(M, nt, dtype=torch.float32, device="cuda")
    O.nova_op_rms_prep(dh, bf16_dev(g1), xt, ss, M, D)
    torch.cuda.synchronize()
    assert np.array_equal(xt.view(torch.int16).cpu().numpy().view(np.uint16), f32_to_bf16_bits(h * g1))
    ref_ss = (h.astype(np.float64) ** 2).reshape(M, nt, 32).sum(-1)
    assert np.abs(ss.cpu().numpy() - ref_ss).max() <= 1e-5 * ref_ss.max()
    # (2) residual GEMM + next-norm outputs
    Wo = rand_bf16(rng, (D, D), D ** -0.5)
    Xa = rand_bf16(rng, (M, D))
    outs = []
    for c in (ctas, 24):
        Y = dh.clone()
        nx = torch.empty(M, D, dtype=torch.bfloat16, device="cuda")
        nss = torch.empty(M, nt, dtype=torch.float32, device="cuda")
        O.nova_op_gemm_fold(bf16_dev(Xa), bf16_dev(Wo), Y, None, M, D, D, O.EPI_F32_RESID, ngamma=bf16_dev(g2),
                            nxout=nx, nss=nss, max_ctas=c)
        torch.cuda.synchronize()
        outs.append((Y, nx, nss))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    Y, nx, nss = outs[0]
    hn = Y.cpu().numpy()
    ref = h.astype(np.float64) + V.linear(Xa.astype(np.float64), Wo.astype(np.float64))
    assert rel_inf(hn, ref) <= 1e-4
    assert np.array_equal(nx.view(torch.int16).cpu().numpy().view(np.uint16), f32_to_bf16_bits(hn * g2))
    ref_ss = (hn.astype(np.float64) ** 2).reshape(M, nt, 32).sum(-1)
    assert np.abs(nss.cpu().numpy() - ref_ss).max() <= 1e-5 * ref_ss.max()
    # (3) consumers with the folded row scale (fold_rows: rsqrt(sum of the chunk sums / D + eps))
    rsc = torch.empty(M, dtype=torch.float32, device="cuda")
    O.nova_op_fold_rows(nss, D, eps, rsc, M)
    torch.cuda.synchronize()
    ref_rs = 1.0 / np.sqrt((hn.astype(np.float64) ** 2).mean(-1) + eps)
    assert np.abs(rsc.cpu().numpy() / ref_rs - 1).max() <= 1e-5
    xn = V.rms_norm(hn.astype(np.float64), g2, eps)
    Wq = rand_bf16(rng, (256, D), D ** -0.5)
    bq = rand_bf16(rng, (256,), 0.05)
    q = torch.empty(M, 256, dtype=torch.bfloat16, device="cuda")
    O.nova_op_gemm_fold(nx, bf16_dev(Wq), q, bf16_dev(bq), M, 256, D, O.EPI_BF16, rscale=rsc, max_ctas=ctas)
    G = rand_bf16(rng, (F, D), D ** -0.5)
    U = rand_bf16(rng, (F, D), D ** -0.5)
    Wgu = np.empty((2 * F, D), dtype=np.float32)
    for i in range(F // 16):
        Wgu[32 * i:32 * i + 16] = G[16 * i:16 * i + 16]
        Wgu[32 * i + 16:32 * i + 32] = U[16 * i:16 * i + 16]
    act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    O.nova_op_gemm_fold(nx, bf16_dev(Wgu), act, None, M, 2 * F, D, O.EPI_BF16_SILUMUL, rscale=rsc, max_ctas=ctas)
    torch.cuda.synchronize()
    assert rel_inf(bf16_host(q), V.linear(xn, Wq.astype(np.float64), bq.astype(np.float64))) <= 8e-3
    ref_act = V.silu(V.linear(xn, G.astype(np.float64))) * V.linear(xn, U.astype(np.float64))
    assert rel_inf(bf16_host(act), ref_act) <= 8e-3


@pytest.mark.parametrize("gh,gw", [(52, 94), (6, 10)])
def test_vit_qkv_gemm_with_fused_2d_rope(gh, gw):
    """ViT qkv GEMM with the 2D RoPE in its epilogue (hd 80, Qwen2-VL ViT width): q / k heads rotated by
    their patch's (row, col) angles (oracle patchify positions + vit_rope_tables / apply_rope), v untouched,
    bias added before the rotation; bf16 rel-inf <= 8e-3 against the f64 oracle; bitwise independent of the
    SM budget."""
    from synth import Q2B
    rng = np.random.default_rng(gh * gw)
    Dv, heads, hd, theta = 1280, 16, 80, 1e4
    M, N = gh * gw, 3 * Dv
    X = rand_bf16(rng, (M, Dv))
    Wq = rand_bf16(rng, (N, Dv), Dv ** -0.5)
    b = rand_bf16(rng, (N,), 0.05)
    dX, dW, db = bf16_dev(X), bf16_dev(Wq), bf16_dev(b)
    outs = []
    for ctas in (148, 40):
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        O.nova_op_gemm_rope2d(dX, dW, C, db, M, N, Dv, 2 * Dv, gw, 2, theta, max_ctas=ctas)
        torch.cuda.synchronize()
        outs.append(C)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    _, _, hp, wp = V.patchify(np.zeros((3, gh * 14, gw * 14), np.float32), Q2B)
    c, s = V.vit_rope_tables(hp, wp, hd, theta, np.float64)
    y = V.linear(X.astype(np.float64), Wq.astype(np.float64), b.astype(np.float64)).reshape(M, 3, heads, hd)
    got = bf16_host(outs[0]).reshape(M, 3, heads, hd)
    assert rel_inf(got[:, 0], V.apply_rope(y[:, 0], c, s)) <= 8e-3
    assert rel_inf(got[:, 1], V.apply_rope(y[:, 1], c, s)) <= 8e-3
    assert rel_inf(got[:, 2], y[:, 2]) <= 8e-3
