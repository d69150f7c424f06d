"""ORACLE (test infrastructure only) -- plain NumPy forward of the Qwen2-VL-shaped VLM.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline leg may
import this.  It shares no code with the CUDA path.

What it computes: the three stages of an agentic VLM request (PAPER.md:94-97,
§II-A "VLM inference ... vision encoder ... adapter ... LLM"; Table
`stage_duration` P:80-91): vision encode -> LLM prefill (builds the KV cache)
-> autoregressive greedy decode.  The paper's model (CogAgent) is
replaced by Qwen2-VL math (reading R1), written
out step by step in the order of SURVEY.md §8(c) c1 steps 1-11.  No blocking,
fusion or reordering: each step is its textbook definition, numpy matmul
being the only library primitive.

Precision: float32 by default (BASELINE.json "fp32 CPU oracle"), float64 via
``dtype=np.float64``; weights are the bf16 values of the file, upcast exactly.
Pins: tests/test_oracle_vlm.py (HF library model in fp64, invariants).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

from synth.models import ModelShape
from synth.weights import bf16_bits_to_f32


class OracleWeights:
    """bf16 bit patterns -> float arrays of the oracle's dtype (exact upcast)."""

    def __init__(self, bits: dict, dtype=np.float32):
        self.dtype = dtype
        self.w = {k: bf16_bits_to_f32(v).astype(dtype) for k, v in bits.items()}

    def __getitem__(self, k):
        return self.w[k]


# ---------------------------------------------------------------- step 1: patchify
def patchify(pixels: np.ndarray, s: ModelShape):
    """Image [C][H][W] -> patch rows X0[N][C*T*P*P] in merge-group-major order.

    Patch (i, j) vector = [c][t][py][px] with the frame duplicated over t
    (Qwen2-VL Conv3d kernel (T, P, P), image tiled T times).  Row order: 2x2
    merge groups row-major, then (di, dj) row-major inside the group, so the
    merger is a plain reshape (HF `rot_pos_emb` permutation).
    Returns X0, (gh, gw), hpos[N], wpos[N].
    """
    C, H, W = pixels.shape
    p, T, m = s.patch, s.temporal_patch, s.merge
    gh, gw = H // p, W // p
    rows, hpos, wpos = [], [], []
    for gi in range(gh // m):
        for gj in range(gw // m):
            for di in range(m):
                for dj in range(m):
                    i, j = gi * m + di, gj * m + dj
                    patch = pixels[:, i * p:(i + 1) * p, j * p:(j + 1) * p]   # [C][P][P]
                    vec = np.stack([patch] * T, axis=1)                    # [C][T][P][P]
                    rows.append(vec.reshape(-1))
                    hpos.append(i)
                    wpos.append(j)
    return np.stack(rows), (gh, gw), np.array(hpos), np.array(wpos)


# ---------------------------------------------------------------- primitives
def layer_norm(x, g, b, eps):
    """LayerNorm: mean, biased variance, eps inside the sqrt."""
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def rms_norm(x, g, eps):
    """RMSNorm: x / sqrt(mean(x^2) + eps) * g."""
    return x / np.sqrt((x * x).mean(-1, keepdims=True) + eps) * g


def linear(x, w, b=None):
    """y = x W^T (+ b), W stored [out][in]."""
    y = x @ w.T
    return y + b if b is not None else y


def quick_gelu(z):
    return z * (1.0 / (1.0 + np.exp(-1.702 * z)))


def gelu_erf(z):
    return 0.5 * z * (1.0 + erf(z / math.sqrt(2.0)))


def silu(z):
    return z / (1.0 + np.exp(-z))


def softmax_rows(s):
    """Row softmax with row-max subtraction."""
    s = s - s.max(-1, keepdims=True)
    e = np.exp(s)
    return e / e.sum(-1, keepdims=True)


def rotate_half(x):
    h = x.shape[-1] // 2
    return np.concatenate([-x[..., h:], x[..., :h]], axis=-1)


def apply_rope(x, cos, sin):
    """x [N][heads][hd]; cos/sin [N][hd]:  x*cos + rotate_half(x)*sin."""
    return x * cos[:, None, :] + rotate_half(x) * sin[:, None, :]


# ---------------------------------------------------------------- step 3: ViT 2D RoPE
def vit_rope_tables(hpos, wpos, hd, theta, dtype):
    """inv_freq[j] = theta^(-4j/hd), j < hd/4; angle = [h*inv | w*inv]; emb = [angle | angle]."""
    j = np.arange(hd // 4, dtype=np.float64)
    inv = 1.0 / theta ** (4.0 * j / hd)
    ang = np.concatenate([np.outer(hpos, inv), np.outer(wpos, inv)], axis=1)
    emb = np.concatenate([ang, ang], axis=1)
    return np.cos(emb).astype(dtype), np.sin(emb).astype(dtype)


# ---------------------------------------------------------------- steps 2-5: encode
def attention_full(q, k, v, scale):
    """Bidirectional MHA per head: softmax(q k^T * scale) v.  q,k,v [N][h][hd]."""
    out = np.empty_like(q)
    for h in range(q.shape[1]):
        p = softmax_rows((q[:, h, :] @ k[:, h, :].T) * scale)
        out[:, h, :] = p @ v[:, h, :]
    return out


def vit_block(x, W, i, s: ModelShape, cos, sin):
    p = f"model.visual.blocks.{i}."
    d, nh = s.vit_dim, s.vit_heads
    hd = d // nh
    a = layer_norm(x, W[p + "norm1.weight"], W[p + "norm1.bias"], s.ln_eps)
    qkv = linear(a, W[p + "attn.qkv.weight"], W[p + "attn.qkv.bias"])
    N = x.shape[0]
    q = qkv[:, 0:d].reshape(N, nh, hd)
    k = qkv[:, d:2 * d].reshape(N, nh, hd)
    v = qkv[:, 2 * d:3 * d].reshape(N, nh, hd)
    q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
    o = attention_full(q, k, v, hd ** -0.5).reshape(N, d)
    x = x + linear(o, W[p + "attn.proj.weight"], W[p + "attn.proj.bias"])
    m = layer_norm(x, W[p + "norm2.weight"], W[p + "norm2.bias"], s.ln_eps)
    h = quick_gelu(linear(m, W[p + "mlp.fc1.weight"], W[p + "mlp.fc1.bias"]))
    return x + linear(h, W[p + "mlp.fc2.weight"], W[p + "mlp.fc2.bias"])


def encode(W: OracleWeights, pixels_f: np.ndarray, s: ModelShape, taps: dict | None = None):
    """Vision encode: patchify -> patch embed -> depth x ViT block -> merger -> E_vis[N/4][d_llm]."""
    X0, (gh, gw), hpos, wpos = patchify(pixels_f.astype(W.dtype), s)
    x = X0 @ W["model.visual.patch_embed.proj.weight"].reshape(s.vit_dim, -1).T
    cos, sin = vit_rope_tables(hpos, wpos, s.vit_head_dim, s.vit_theta, W.dtype)
    for i in range(s.vit_depth):
        x = vit_block(x, W, i, s, cos, sin)
        if taps is not None:
            taps[f"vit{i}"] = x.copy()
    y = layer_norm(x, W["model.visual.merger.ln_q.weight"], W["model.visual.merger.ln_q.bias"], s.ln_eps)
    y = y.reshape(-1, s.merge_dim)
    y = gelu_erf(linear(y, W["model.visual.merger.mlp.0.weight"], W["model.visual.merger.mlp.0.bias"]))
    e = linear(y, W["model.visual.merger.mlp.2.weight"], W["model.visual.merger.mlp.2.bias"])
    return e, (gh, gw)


# ---------------------------------------------------------------- step 7: M-RoPE
def mrope_positions(gh: int, gw: int, n_text: int, merge: int):
    """3 x S positions (HF get_rope_index, image first): vision token j at LLM grid
    (r, c) -> (0, r, c); text token i -> all three = max_vision_pos + 1 + i."""
    lh, lw = gh // merge, gw // merge
    r, c = np.divmod(np.arange(lh * lw), lw)
    vis = np.stack([np.zeros_like(r), r, c])
    st = max(lh, lw)   # max vision position + 1
    txt = np.tile(st + np.arange(n_text), (3, 1))
    return np.concatenate([vis, txt], axis=1)


def text_start(gh: int, gw: int, merge: int) -> int:
    return max(gh // merge, gw // merge)


def mrope_tables(pos3: np.ndarray, hd: int, theta: float, section, dtype):
    """inv_freq[i] = theta^(-2i/hd); frequency index i takes its position from
    t (i < s0), h (i < s0+s1) or w; the second half mirrors the first."""
    i = np.arange(hd // 2, dtype=np.float64)
    inv = 1.0 / theta ** (2.0 * i / hd)
    comp = np.where(i < section[0], 0, np.where(i < section[0] + section[1], 1, 2))
    pos = pos3[comp, :].T.astype(np.float64)          # [S][hd/2]
    ang = pos * inv[None, :]
    emb = np.concatenate([ang, ang], axis=1)
    return np.cos(emb).astype(dtype), np.sin(emb).astype(dtype)


# ---------------------------------------------------------------- step 8: LLM block
def attention_causal_gqa(q, k, v, scale, q_offset):
    """q [Sq][H][hd], k/v [Sk][KV][hd]; query i (absolute q_offset+i) sees keys j <= q_offset+i;
    query head h uses KV head h // (H/KV)."""
    Sq, H, hd = q.shape
    Sk, KV, _ = k.shape
    g = H // KV
    out = np.empty_like(q)
    mask = np.arange(Sk)[None, :] > (q_offset + np.arange(Sq))[:, None]
    for h in range(H):
        sc = (q[:, h, :] @ k[:, h // g, :].T) * scale
        sc = np.where(mask, -np.inf, sc)
        out[:, h, :] = softmax_rows(sc) @ v[:, h // g, :]
    return out


def llm_layer(x, W, i, s: ModelShape, cos, sin, cache: dict, q_offset: int):
    """One decoder layer over rows x (absolute positions q_offset..), appending k, v to cache."""
    p = f"model.language_model.layers.{i}."
    H, KV, hd = s.llm_heads, s.llm_kv_heads, s.head_dim
    n = x.shape[0]
    a = rms_norm(x, W[p + "input_layernorm.weight"], s.rms_eps)
    q = linear(a, W[p + "self_attn.q_proj.weight"], W[p + "self_attn.q_proj.bias"]).reshape(n, H, hd)
    k = linear(a, W[p + "self_attn.k_proj.weight"], W[p + "self_attn.k_proj.bias"]).reshape(n, KV, hd)
    v = linear(a, W[p + "self_attn.v_proj.weight"], W[p + "self_attn.v_proj.bias"]).reshape(n, KV, hd)
    q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
    kc = np.concatenate([cache["k"][i], k]) if i in cache["k"] else k
    vc = np.concatenate([cache["v"][i], v]) if i in cache["v"] else v
    cache["k"][i], cache["v"][i] = kc, vc
    o = attention_causal_gqa(q, kc, vc, hd ** -0.5, q_offset).reshape(n, H * hd)
    x = x + linear(o, W[p + "self_attn.o_proj.weight"])
    m = rms_norm(x, W[p + "post_attention_layernorm.weight"], s.rms_eps)
    h = silu(linear(m, W[p + "mlp.gate_proj.weight"])) * linear(m, W[p + "mlp.up_proj.weight"])
    return x + linear(h, W[p + "mlp.down_proj.weight"])


def lm_head_weight(W, s: ModelShape):
    return W["model.language_model.embed_tokens.weight"] if s.tie_embed else W["lm_head.weight"]


def final_logits(x_row, W, s: ModelShape):
    """logits = RMSNorm(x) * g_f . W_lm^T (step 9)."""
    h = rms_norm(x_row, W["model.language_model.norm.weight"], s.rms_eps)
    return h @ lm_head_weight(W, s).T


def argmax_lowest(v: np.ndarray) -> int:
    """Greedy pick, ties -> lowest index (reading R6)."""
    return int(np.flatnonzero(v == v.max())[0])


def llm_forward_rows(x, pos3, W, s: ModelShape, cache: dict, q_offset: int, taps=None, tap_prefix=""):
    cos, sin = mrope_tables(pos3, s.head_dim, s.llm_theta, s.mrope_section, W.dtype)
    for i in range(s.llm_layers):
        x = llm_layer(x, W, i, s, cos, sin, cache, q_offset)
        if taps is not None:
            taps[f"{tap_prefix}llm{i}"] = x.copy()
    return x


# ---------------------------------------------------------------- steps 6-11: generate
def generate(W: OracleWeights, pixels_bits: np.ndarray, prompt_ids: np.ndarray, gen_len: int,
             s: ModelShape, force_tokens=None, taps: dict | None = None):
    """Encode -> prefill -> greedy decode with KV cache.

    Returns dict(tokens[gen_len], logits[gen_len][V], e_vis, margins[gen_len]).
    `force_tokens` (teacher forcing) feeds the given token instead of the argmax
    from that step on; the reported token is still the argmax.
    """
    pix = bf16_bits_to_f32(pixels_bits).astype(W.dtype)
    e_vis, (gh, gw) = encode(W, pix, s, taps)
    emb = W["model.language_model.embed_tokens.weight"]
    x = np.concatenate([e_vis, emb[np.asarray(prompt_ids)]], axis=0)
    S = x.shape[0]
    pos3 = mrope_positions(gh, gw, len(prompt_ids), s.merge)
    cache = {"k": {}, "v": {}}
    x = llm_forward_rows(x, pos3, W, s, cache, 0, taps, "pre_")
    logits = [final_logits(x[-1], W, s)]
    last_pos = int(pos3[0, -1])
    for k in range(1, gen_len):
        prev = argmax_lowest(logits[-1])
        if force_tokens is not None and k - 1 < len(force_tokens):
            prev = int(force_tokens[k - 1])
        xk = emb[[prev]]
        p3 = np.full((3, 1), last_pos + k)
        xk = llm_forward_rows(xk, p3, W, s, cache, S + k - 1)
        logits.append(final_logits(xk[-1], W, s))
    L = np.stack(logits)
    toks = np.array([argmax_lowest(l) for l in L], dtype=np.int32)
    srt = np.sort(L, axis=1)
    return {"tokens": toks, "logits": L, "e_vis": e_vis, "margins": srt[:, -1] - srt[:, -2],
            "grid": (gh, gw), "S": S}


def full_recompute_logits(W: OracleWeights, pixels_bits, prompt_ids, tokens, s: ModelShape):
    """Logits for every generated step by re-running the whole sequence (no cache reuse).

    Invariant pin: equals the KV-cached `generate` logits."""
    pix = bf16_bits_to_f32(pixels_bits).astype(W.dtype)
    e_vis, (gh, gw) = encode(W, pix, s)
    emb = W["model.language_model.embed_tokens.weight"]
    n = len(prompt_ids)
    out = []
    for k in range(len(tokens)):
        ids = list(prompt_ids) + list(tokens[:k])
        x = np.concatenate([e_vis, emb[np.asarray(ids, dtype=np.int64)]], axis=0)
        pos3 = mrope_positions(gh, gw, n + k, s.merge)
        x = llm_forward_rows(x, pos3, W, s, {"k": {}, "v": {}}, 0)
        out.append(final_logits(x[-1], W, s))
    return np.stack(out)
