"""Library pin for the oracle: HF transformers Qwen2-VL modules run in float64.

HF forces four steps to float32 regardless of the model dtype (vision RoPE
application, the text rotary tables, RMSNorm, eager-attention softmax).  To compare at
1e-9 those *precision casts* are lifted to float64 (the arithmetic is HF's
own); SDPA attention is used, which computes in the input dtype.
"""
from __future__ import annotations

import numpy as np
import torch

import transformers.models.qwen2_vl.modeling_qwen2_vl as M
from transformers import Qwen2VLConfig, Qwen2VLForConditionalGeneration

from synth.models import ModelShape
from synth.weights import bf16_bits_to_f32

_patched = False


def _patch_fp64():
    global _patched
    if _patched:
        return

    def rope_vis(q, k, cos, sin):
        cos, sin = cos.unsqueeze(-2).to(q.dtype), sin.unsqueeze(-2).to(q.dtype)
        return q * cos + M.rotate_half(q) * sin, k * cos + M.rotate_half(k) * sin

    def rot_fwd(self, x, position_ids):
        n = self.inv_freq.numel()
        theta = self.config.rope_parameters["rope_theta"]
        inv = 1.0 / (theta ** (torch.arange(0, 2 * n, 2, dtype=torch.float64) / (2 * n)))
        freqs = (inv[None, None, :, None].expand(3, position_ids.shape[1], -1, 1)
                 @ position_ids[:, :, None, :].double()).transpose(2, 3)
        emb = torch.cat((freqs, freqs), -1)
        return emb.cos().to(x.dtype), emb.sin().to(x.dtype)

    def rms_fwd(self, h):
        var = h.pow(2).mean(-1, keepdim=True)
        return self.weight * (h * torch.rsqrt(var + self.variance_epsilon))

    M.apply_rotary_pos_emb_vision = rope_vis
    M.Qwen2VLRMSNorm.forward = rms_fwd
    M.Qwen2VLRotaryEmbedding.forward = rot_fwd
    _patched = True


def build(s: ModelShape, bits: dict):
    _patch_fp64()
    cfg = Qwen2VLConfig(
        vision_config=dict(depth=s.vit_depth, embed_dim=s.vit_dim, hidden_size=s.llm_dim,
                           num_heads=s.vit_heads, mlp_ratio=s.vit_mlp // s.vit_dim,
                           patch_size=s.patch, temporal_patch_size=s.temporal_patch,
                           spatial_merge_size=s.merge, in_channels=s.in_ch, hidden_act="quick_gelu"),
        text_config=dict(hidden_size=s.llm_dim, intermediate_size=s.llm_ffn,
                         num_hidden_layers=s.llm_layers, num_attention_heads=s.llm_heads,
                         num_key_value_heads=s.llm_kv_heads, vocab_size=s.vocab, rms_norm_eps=s.rms_eps,
                         rope_parameters={"rope_type": "default", "rope_theta": s.llm_theta,
                                          "mrope_section": list(s.mrope_section)},
                         max_position_embeddings=32768, tie_word_embeddings=s.tie_embed),
        tie_word_embeddings=s.tie_embed)
    for c in (cfg, cfg.vision_config, cfg.text_config):
        c._attn_implementation = "sdpa"
    m = Qwen2VLForConditionalGeneration(cfg).double().eval()
    dim = m.model.visual.rotary_pos_emb.dim
    m.model.visual.rotary_pos_emb.inv_freq = 1.0 / (s.vit_theta ** (torch.arange(0, dim, 2, dtype=torch.float64) / dim))
    sd = {k: torch.from_numpy(bf16_bits_to_f32(v).astype(np.float64)) for k, v in bits.items()}
    if s.tie_embed:
        sd["lm_head.weight"] = sd["model.language_model.embed_tokens.weight"]
    m.load_state_dict(sd, strict=True)
    return m


@torch.no_grad()
def hf_logits(m, X0: np.ndarray, grid_hw, prompt_ids, tokens, pos3: np.ndarray):
    """E_vis and logits for every generated step (full-sequence forward, no cache)."""
    gh, gw = grid_hw
    ev = m.model.visual(torch.from_numpy(X0), grid_thw=torch.tensor([[1, gh, gw]])).pooler_output
    emb = m.model.language_model.embed_tokens.weight
    ids = list(prompt_ids) + list(tokens[:-1])
    x = torch.cat([ev, emb[torch.tensor(ids, dtype=torch.long)]], 0)[None]
    pos = torch.from_numpy(pos3)[:, None, :]
    h = m.model.language_model(inputs_embeds=x, position_ids=pos).last_hidden_state
    lg = m.lm_head(h)[0, -len(tokens):]
    return ev.numpy(), lg.numpy()
