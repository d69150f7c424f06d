"""Model shapes and the weight schema (names, shapes, init kinds).

This module is part of the *seeded input generators* shared by the oracle
(`oracle/`) and the CUDA path (`paper_2509_21301_b200/`).  It holds no
arithmetic of the method: only shapes, tensor names and which random
distribution each tensor is drawn from.

Model family.  The paper evaluates CogAgent (§V-A) with trained
weights, which are out of scope; BASELINE.json fixes Qwen2-VL-shaped
random-init models instead.  Tensor names are the HF Qwen2-VL ``state_dict``
keys (reading R1) so a library model can be loaded with the same
file as an independent pin of the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict, replace


@dataclass(frozen=True)
class ModelShape:
    name: str
    # vision tower (ViT)
    vit_depth: int
    vit_dim: int
    vit_heads: int
    vit_mlp: int
    patch: int = 14
    temporal_patch: int = 2
    merge: int = 2
    in_ch: int = 3
    # language model
    llm_layers: int = 2
    llm_dim: int = 128
    llm_heads: int = 4
    llm_kv_heads: int = 2
    head_dim: int = 32
    llm_ffn: int = 384
    vocab: int = 512
    tie_embed: bool = False
    mrope_section: tuple = (4, 6, 6)
    vit_theta: float = 1.0e4
    llm_theta: float = 1.0e6
    ln_eps: float = 1.0e-6
    rms_eps: float = 1.0e-6

    @property
    def vit_head_dim(self) -> int:
        return self.vit_dim // self.vit_heads

    @property
    def patch_dim(self) -> int:
        return self.in_ch * self.temporal_patch * self.patch * self.patch

    @property
    def merge_dim(self) -> int:
        return self.vit_dim * self.merge * self.merge

    @property
    def unit(self) -> int:
        """Image side granularity in pixels (patch * merge = 28)."""
        return self.patch * self.merge

    def to_dict(self) -> dict:
        d = asdict(self)
        d["mrope_section"] = list(self.mrope_section)
        return d


# cfg 1 (BASELINE.json configs[0]); constants per SURVEY.md §8(c) c1.
TINY = ModelShape(name="tiny", vit_depth=2, vit_dim=64, vit_heads=4, vit_mlp=256,
                  llm_layers=2, llm_dim=128, llm_heads=4, llm_kv_heads=2, head_dim=32,
                  llm_ffn=384, vocab=512, tie_embed=False, mrope_section=(4, 6, 6))

# Qwen2-VL-2B-shaped (public config; SURVEY.md §8 shape legend).
Q2B = ModelShape(name="qwen2vl-2b", vit_depth=32, vit_dim=1280, vit_heads=16, vit_mlp=5120,
                 llm_layers=28, llm_dim=1536, llm_heads=12, llm_kv_heads=2, head_dim=128,
                 llm_ffn=8960, vocab=151936, tie_embed=True, mrope_section=(16, 24, 24))

# Qwen2-VL-7B-shaped.
Q7B = ModelShape(name="qwen2vl-7b", vit_depth=32, vit_dim=1280, vit_heads=16, vit_mlp=5120,
                 llm_layers=28, llm_dim=3584, llm_heads=28, llm_kv_heads=4, head_dim=128,
                 llm_ffn=18944, vocab=152064, tie_embed=False, mrope_section=(16, 24, 24))

PRESETS = {"tiny": TINY, "2b": Q2B, "7b": Q7B}


def reduced_depth(shape: ModelShape, vit_depth: int = 2, llm_layers: int = 2) -> ModelShape:
    """Full-width, reduced-depth variant used for full-size parity tests."""
    return replace(shape, name=f"{shape.name}-d{vit_depth}l{llm_layers}",
                   vit_depth=vit_depth, llm_layers=llm_layers)


# ---------------------------------------------------------------- weight schema
# init kinds:
#   ("normal", std)  N(0, std^2)         ("uniform", a)  U(-a, a)
#   ("gamma", a)     1 + U(-a, a)
def weight_specs(s: ModelShape) -> list[tuple[str, tuple, tuple]]:
    """List of (name, shape, init) in file order."""
    specs: list[tuple[str, tuple, tuple]] = []
    d, m = s.vit_dim, s.vit_mlp
    lin = lambda fan_in, gain=1.0: ("normal", gain / fan_in ** 0.5)
    bias = ("uniform", 0.05)
    gamma = ("gamma", 0.1)
    specs.append(("model.visual.patch_embed.proj.weight",
                  (d, s.in_ch, s.temporal_patch, s.patch, s.patch), lin(s.patch_dim)))
    for i in range(s.vit_depth):
        p = f"model.visual.blocks.{i}."
        specs += [
            (p + "norm1.weight", (d,), gamma), (p + "norm1.bias", (d,), bias),
            (p + "norm2.weight", (d,), gamma), (p + "norm2.bias", (d,), bias),
            (p + "attn.qkv.weight", (3 * d, d), lin(d)), (p + "attn.qkv.bias", (3 * d,), bias),
            (p + "attn.proj.weight", (d, d), lin(d, 0.5)), (p + "attn.proj.bias", (d,), bias),
            (p + "mlp.fc1.weight", (m, d), lin(d)), (p + "mlp.fc1.bias", (m,), bias),
            (p + "mlp.fc2.weight", (d, m), lin(m, 0.5)), (p + "mlp.fc2.bias", (d,), bias),
        ]
    md = s.merge_dim
    specs += [
        ("model.visual.merger.ln_q.weight", (d,), gamma),
        ("model.visual.merger.ln_q.bias", (d,), bias),
        ("model.visual.merger.mlp.0.weight", (md, md), lin(md)),
        ("model.visual.merger.mlp.0.bias", (md,), bias),
        ("model.visual.merger.mlp.2.weight", (s.llm_dim, md), lin(md)),
        ("model.visual.merger.mlp.2.bias", (s.llm_dim,), bias),
    ]
    D, H, KV, hd, F = s.llm_dim, s.llm_heads, s.llm_kv_heads, s.head_dim, s.llm_ffn
    specs.append(("model.language_model.embed_tokens.weight", (s.vocab, D), ("normal", 1.0)))
    for i in range(s.llm_layers):
        p = f"model.language_model.layers.{i}."
        specs += [
            (p + "self_attn.q_proj.weight", (H * hd, D), lin(D)), (p + "self_attn.q_proj.bias", (H * hd,), bias),
            (p + "self_attn.k_proj.weight", (KV * hd, D), lin(D)), (p + "self_attn.k_proj.bias", (KV * hd,), bias),
            (p + "self_attn.v_proj.weight", (KV * hd, D), lin(D)), (p + "self_attn.v_proj.bias", (KV * hd,), bias),
            (p + "self_attn.o_proj.weight", (D, H * hd), lin(H * hd, 0.5)),
            (p + "mlp.gate_proj.weight", (F, D), lin(D)),
            (p + "mlp.up_proj.weight", (F, D), lin(D)),
            (p + "mlp.down_proj.weight", (D, F), lin(F, 0.5)),
            (p + "input_layernorm.weight", (D,), gamma),
            (p + "post_attention_layernorm.weight", (D,), gamma),
        ]
    specs.append(("model.language_model.norm.weight", (D,), gamma))
    if not s.tie_embed:
        specs.append(("lm_head.weight", (s.vocab, D), ("normal", 2.0 / D ** 0.5)))
    return specs


def vit_layer_names(s: ModelShape, i: int) -> list[str]:
    return [n for n, _, _ in weight_specs(replace(s, vit_depth=max(s.vit_depth, i + 1)))
            if n.startswith(f"model.visual.blocks.{i}.")]


def param_count(s: ModelShape) -> int:
    tot = 0
    for _, shp, _ in weight_specs(s):
        n = 1
        for x in shp:
            n *= x
        tot += n
    return tot
