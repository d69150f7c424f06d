"""Pins for oracle/vlm.py against things other than itself (CPU only).

- library routine: HF transformers Qwen2-VL in float64 (tests/hf_ref.py);
- library routines: torch SDPA (GQA attention), conv3d (patch embed), torch GELU/SiLU;
- invariants: KV-cached decode == full recompute, softmax rows sum to 1, RoPE
  identity at 0 and norm preservation, M-RoPE with t=h=w == 1D RoPE (complex
  rotation), LN of a constant row == beta, RMSNorm closed form, causal prefix
  independence.
"""
import json
import os
from dataclasses import replace

import numpy as np
import pytest
import torch

from synth import TINY, gen_weights, tiny_request, make_request, bf16_bits_to_f32
from oracle import vlm as V

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def tiny():
    seed = json.load(open(os.path.join(GOLD, "tiny_seed.json")))["seed"]
    bits = gen_weights(TINY, seed)
    req = tiny_request(TINY, seed)
    return bits, req


def _hf_compare(s, bits, req):
    from tests import hf_ref
    W64 = V.OracleWeights(bits, np.float64)
    out = V.generate(W64, req.pixels, req.prompt_ids, req.gen_len, s)
    m = hf_ref.build(s, bits)
    X0, grid, _, _ = V.patchify(bf16_bits_to_f32(req.pixels).astype(np.float64), s)
    pos3 = V.mrope_positions(*grid, len(req.prompt_ids) + req.gen_len - 1, s.merge)
    ev, lg = hf_ref.hf_logits(m, X0, grid, req.prompt_ids, out["tokens"], pos3)
    return out, ev, lg


def test_hf_library_pin_fp64(tiny):
    bits, req = tiny
    out, ev, lg = _hf_compare(TINY, bits, req)
    assert np.abs(ev - out["e_vis"]).max() <= 1e-9
    assert np.abs(lg - out["logits"]).max() <= 1e-9
    W32 = V.OracleWeights(bits, np.float32)
    o32 = V.generate(W32, req.pixels, req.prompt_ids, req.gen_len, TINY)
    assert np.abs(o32["logits"] - lg).max() <= 1e-4
    assert (o32["tokens"] == out["tokens"]).all()


def test_hf_library_pin_tied_mha_rect():
    """Other code paths: tied lm_head, kv_heads == heads, non-square image grid."""
    s = replace(TINY, name="tiny-tied", llm_kv_heads=4, tie_embed=True, vit_heads=2)
    bits = gen_weights(s, 3)
    req = make_request(s, (4, 6), 5, 4, 3)
    out, ev, lg = _hf_compare(s, bits, req)
    assert np.abs(ev - out["e_vis"]).max() <= 1e-9
    assert np.abs(lg - out["logits"]).max() <= 1e-9


def test_golden_tiny_tokens(tiny):
    bits, req = tiny
    g = json.load(open(os.path.join(GOLD, "tiny_seed.json")))
    out = V.generate(V.OracleWeights(bits, np.float64), req.pixels, req.prompt_ids, req.gen_len, TINY)
    assert out["tokens"].tolist() == g["tokens"]
    assert out["margins"].min() >= 0.1


def test_kv_cache_equals_full_recompute(tiny):
    bits, req = tiny
    W = V.OracleWeights(bits, np.float64)
    out = V.generate(W, req.pixels, req.prompt_ids, req.gen_len, TINY)
    fr = V.full_recompute_logits(W, req.pixels, req.prompt_ids, out["tokens"], TINY)
    assert np.abs(fr - out["logits"]).max() <= 1e-9


def test_causal_prefix_independence(tiny):
    bits, req = tiny
    W = V.OracleWeights(bits, np.float64)
    out = V.generate(W, req.pixels, req.prompt_ids, req.gen_len, TINY)
    alt = out["tokens"].copy()
    alt[4:] = (alt[4:] + 17) % TINY.vocab      # change the suffix
    fr = V.full_recompute_logits(W, req.pixels, req.prompt_ids, alt, TINY)
    assert np.abs(fr[:5] - out["logits"][:5]).max() <= 1e-9


def test_softmax_rows_sum_to_one():
    rng = np.random.default_rng(0)
    p = V.softmax_rows(rng.standard_normal((7, 33)) * 10)
    assert np.abs(p.sum(-1) - 1).max() <= 1e-12
    assert (p >= 0).all()


def test_rope_identity_at_zero_and_norm():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((5, 3, 32))
    pos = np.zeros((3, 5), dtype=np.int64)
    c, s = V.mrope_tables(pos, 32, 1e6, (4, 6, 6), np.float64)
    assert np.abs(V.apply_rope(x, c, s) - x).max() == 0
    pos = np.tile(np.arange(5) * 37, (3, 1))
    c, s = V.mrope_tables(pos, 32, 1e6, (4, 6, 6), np.float64)
    y = V.apply_rope(x, c, s)
    assert np.allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), atol=1e-12)


def test_mrope_equal_components_is_1d_rope():
    """Textbook RoPE as complex rotation of pairs (x_i, x_{i+d/2}) by pos*base^(-2i/d)."""
    d, base = 32, 1e6
    rng = np.random.default_rng(2)
    x = rng.standard_normal((6, 2, d))
    pos = np.arange(6) * 11 + 3
    c, s = V.mrope_tables(np.tile(pos, (3, 1)), d, base, (4, 6, 6), np.float64)
    y = V.apply_rope(x, c, s)
    z = x[..., : d // 2] + 1j * x[..., d // 2:]
    ang = pos[:, None] * base ** (-2.0 * np.arange(d // 2) / d)
    zr = z * np.exp(1j * ang)[:, None, :]
    ref = np.concatenate([zr.real, zr.imag], axis=-1)
    assert np.abs(y - ref).max() <= 1e-12


def test_vit_rope_tables_2d():
    """h and w halves rotate with their own coordinate (complex form)."""
    hd, th = 16, 1e4
    h, w = np.array([0, 3, 5]), np.array([0, 2, 7])
    c, s = V.vit_rope_tables(h, w, hd, th, np.float64)
    inv = th ** (-4.0 * np.arange(hd // 4) / hd)
    ang = np.concatenate([np.outer(h, inv), np.outer(w, inv)], axis=1)
    assert np.allclose(c[:, : hd // 2], np.cos(ang)) and np.allclose(s[:, hd // 2:], np.sin(ang))
    assert np.abs(c[0] - 1).max() == 0 and np.abs(s[0]).max() == 0


def test_gqa_attention_vs_torch_sdpa():
    rng = np.random.default_rng(3)
    Sq, Sk, H, KV, hd = 5, 9, 6, 2, 16
    q = rng.standard_normal((Sq, H, hd))
    k = rng.standard_normal((Sk, KV, hd))
    v = rng.standard_normal((Sk, KV, hd))
    off = Sk - Sq
    o = V.attention_causal_gqa(q, k, v, hd ** -0.5, off)
    tq = torch.from_numpy(q).permute(1, 0, 2)[None]
    tk = torch.from_numpy(np.repeat(k, H // KV, axis=1)).permute(1, 0, 2)[None]
    tv = torch.from_numpy(np.repeat(v, H // KV, axis=1)).permute(1, 0, 2)[None]
    mask = torch.from_numpy(np.arange(Sk)[None, :] <= (off + np.arange(Sq))[:, None])
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask)[0].permute(1, 0, 2)
    assert np.abs(o - ref.numpy()).max() <= 1e-12
    of = V.attention_full(q[:, :2], k[:5, :], v[:5, :], 0.3) if False else None  # noqa


def test_full_attention_vs_torch_sdpa():
    rng = np.random.default_rng(4)
    q, k, v = (rng.standard_normal((11, 3, 8)) for _ in range(3))
    o = V.attention_full(q, k, v, 8 ** -0.5)
    t = [torch.from_numpy(a).permute(1, 0, 2)[None] for a in (q, k, v)]
    ref = torch.nn.functional.scaled_dot_product_attention(*t)[0].permute(1, 0, 2)
    assert np.abs(o - ref.numpy()).max() <= 1e-12


def test_norms_closed_forms():
    g = np.linspace(0.5, 1.5, 8)
    b = np.linspace(-0.1, 0.1, 8)
    row = np.full((1, 8), 3.25)
    assert np.abs(V.layer_norm(row, g, b, 1e-6) - b).max() <= 1e-12
    c = -2.0
    r = V.rms_norm(np.full((1, 8), c), g, 1e-6)
    assert np.abs(r - g * c / np.sqrt(c * c + 1e-6)).max() <= 1e-12
    x = np.random.default_rng(5).standard_normal((4, 8))
    ref = torch.nn.functional.layer_norm(torch.from_numpy(x), (8,), torch.from_numpy(g), torch.from_numpy(b), 1e-6)
    assert np.abs(V.layer_norm(x, g, b, 1e-6) - ref.numpy()).max() <= 1e-12


def test_activations_vs_torch():
    z = np.linspace(-6, 6, 101)
    tz = torch.from_numpy(z)
    assert np.abs(V.gelu_erf(z) - torch.nn.functional.gelu(tz).numpy()).max() <= 1e-12
    assert np.abs(V.silu(z) - torch.nn.functional.silu(tz).numpy()).max() <= 1e-12
    assert np.abs(V.quick_gelu(z) - (tz * torch.sigmoid(1.702 * tz)).numpy()).max() <= 1e-12


def test_patchify_patch_embed_vs_conv3d():
    s = TINY
    bits = gen_weights(s, 0)
    req = make_request(s, (4, 6), 2, 2, 9)
    pix = bf16_bits_to_f32(req.pixels).astype(np.float64)
    X0, (gh, gw), hp, wp = V.patchify(pix, s)
    Wpe = bf16_bits_to_f32(bits["model.visual.patch_embed.proj.weight"]).astype(np.float64)
    ours = X0 @ Wpe.reshape(s.vit_dim, -1).T
    vid = torch.from_numpy(np.stack([pix] * s.temporal_patch, axis=1))[None]   # [1][C][T][H][W]
    conv = torch.nn.functional.conv3d(vid, torch.from_numpy(Wpe), stride=(s.temporal_patch, s.patch, s.patch))
    conv = conv[0, :, 0].numpy()                                                # [d][gh][gw]
    ref = conv[:, hp, wp].T
    assert np.abs(ours - ref).max() <= 1e-10
    # merge-group-major order: rows 4g..4g+3 form one 2x2 group
    assert list(zip(hp[:4], wp[:4])) == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert list(zip(hp[4:8], wp[4:8])) == [(0, 2), (0, 3), (1, 2), (1, 3)]


def test_mrope_positions_layout():
    p = V.mrope_positions(4, 6, 3, 2)       # LLM grid 2x3, 3 text tokens
    assert p[:, :6].T.tolist() == [[0, 0, 0], [0, 0, 1], [0, 0, 2], [0, 1, 0], [0, 1, 1], [0, 1, 2]]
    assert p[:, 6:].tolist() == [[3, 4, 5]] * 3
    assert V.text_start(52, 94, 2) == 47
