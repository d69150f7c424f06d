// L2 stage programs: the vision encode, LLM prefill and LLM decode forward passes
// (§II-A, Table stage_duration; SURVEY.md §8(a) rows
// a5, a6, a7) as launch sequences of the sm_100a kernels, plus the engine's
// weight / workspace layout in HBM and the layer-wise ViT weight offload ring
// (§III-E, Eq. 7).
#include <algorithm>
#include <cstring>

#include "engine.h"

namespace nova {

#define CUDA_TRY(x)                          \
  do {                                       \
    cudaError_t _e = (x);                    \
    if (_e != cudaSuccess) return _e;        \
  } while (0)

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

void Dims::init(const nova_model_config& mc) {
  m = mc;
  vit_hd = m.vit_dim / m.vit_heads;
  patch_dim = m.in_ch * m.temporal_patch * m.patch * m.patch;
  merge_dim = m.vit_dim * m.merge * m.merge;
  qkv_n = 3 * m.vit_dim;
  llm_qkv_n = (m.llm_heads + 2 * m.llm_kv_heads) * m.head_dim;
}

void VitLayerLayout::init(const Dims& d) {
  const size_t D = d.m.vit_dim, M = d.m.vit_mlp;
  size_t o = 0;
  auto take = [&](size_t n) {
    size_t r = o;
    o = align_up(o + n, 128);
    return r;
  };
  n1g = take(D);
  n1b = take(D);
  n2g = take(D);
  n2b = take(D);
  qkv_w = take(3 * D * D);
  qkv_b = take(3 * D);
  proj_w = take(D * D);
  proj_b = take(D);
  fc1_w = take(M * D);
  fc1_b = take(M);
  fc2_w = take(D * M);
  fc2_b = take(D);
  elems = o;
}

// Bump layout over the weights buffer (base == nullptr: size only).
size_t Engine::plan_weights(const Dims& d, const nova_engine_config& c, Weights* w, VitLayerLayout* vlo,
                            uint8_t* base) {
  VitLayerLayout vl;
  vl.init(d);
  if (vlo) *vlo = vl;
  size_t off = 0;
  auto take = [&](size_t elems) -> bf16* {
    bf16* p = base ? reinterpret_cast<bf16*>(base + off) : nullptr;
    off = align_up(off + elems * 2, 256);
    return p;
  };
  const auto& m = d.m;
  const size_t D = m.llm_dim, F = m.llm_ffn, V = m.vocab, md = d.merge_dim;
  Weights tmp;
  Weights& W = w ? *w : tmp;
  W.patch_w = take((size_t)m.vit_dim * d.patch_dim);
  const int nblk = c.vit_resident_layers > 0 ? std::min(c.vit_resident_layers, m.vit_depth) : m.vit_depth;
  W.vit_dev.assign(nblk, nullptr);
  for (int i = 0; i < nblk; ++i) W.vit_dev[i] = take(vl.elems);
  W.mlnq_g = take(m.vit_dim);
  W.mlnq_b = take(m.vit_dim);
  W.m1_w = take(md * md);
  W.m1_b = take(md);
  W.m2_w = take(D * md);
  W.m2_b = take(D);
  W.embed = take(V * D);
  W.llm.assign(m.llm_layers, LlmLayerW{});
  for (int i = 0; i < m.llm_layers; ++i) {
    LlmLayerW& L = W.llm[i];
    L.ln1 = take(D);
    L.qkv_w = take((size_t)d.llm_qkv_n * D);
    L.qkv_b = take(d.llm_qkv_n);
    L.o_w = take(D * m.llm_heads * m.head_dim);
    L.ln2 = take(D);
    L.gu_w = take(2 * F * D);
    L.down_w = take(D * F);
  }
  W.final_norm = take(D);
  W.lm_head = m.tie_embed ? W.embed : take(V * D);
  // Decode streams every LLM linear once per iteration from a slice of the SMs; it reads a
  // second copy in the streaming layout (contiguous, pre-swizzled 64 x 64 tiles: one bulk copy
  // per tile, full DRAM bursts -- scripts/probe_bw.cu measured row-major 128-byte tile rows at
  // ~56% of contiguous bandwidth on a 24-SM partition).  The prefill GEMM keeps [out][in].
  for (int i = 0; i < m.llm_layers; ++i) {
    LlmLayerW& L = W.llm[i];
    L.qkv_wb = take((size_t)d.llm_qkv_n * D);
    L.o_wb = take(D * m.llm_heads * m.head_dim);
    L.gu_wb = take(2 * F * D);
    L.down_wb = take(D * F);
  }
  W.lm_head_b = take(V * D);
  return off;
}

size_t Engine::plan_kv(const Dims& d, const nova_engine_config& c) {
  return (size_t)d.m.llm_layers * c.kv_pages * 2 * d.m.llm_kv_heads * 64 * d.m.head_dim * 2;
}

static int s_max_of(const Dims& d, const nova_engine_config& c) {
  return c.max_patches / (d.m.merge * d.m.merge) + c.max_prompt;
}

size_t Engine::plan_workspace(const Dims& d, const nova_engine_config& c, Engine* e, uint8_t* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> uint8_t* {
    uint8_t* p = base ? base + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  const auto& m = d.m;
  const size_t N = c.max_patches, S = s_max_of(d, c), D = m.llm_dim, F = m.llm_ffn, V = m.vocab;
  const size_t B = c.max_decode_batch, Hhd = (size_t)m.llm_heads * m.head_dim;
  const int n_slots = c.max_requests + 17;  // + 1 front and 16 decode profiling slots
  const int max_ctx = (int)S + c.max_gen;
  const int max_pages = (max_ctx + 63) / 64;
  FrontWS f{};
  DecWS w{};
  f.x0 = (bf16*)take(N * d.patch_dim * 2);
  f.vhid = (float*)take(N * m.vit_dim * 4);
  f.xb = (bf16*)take(std::max(N * m.vit_dim, S * D) * 2);
  f.qkv = (bf16*)take(std::max(N * d.qkv_n, S * d.llm_qkv_n) * 2);
  f.attn = (bf16*)take(std::max(N * m.vit_dim, S * Hhd) * 2);
  f.act = (bf16*)take(std::max(std::max(N * m.vit_mlp, (N / 4) * d.merge_dim), S * F) * 2);
  f.hid = (float*)take(S * D * 4);
  f.nss = (float*)take(S * ((D + 31) / 32) * 4);
  f.rscale = (float*)take(S * 4);
  f.rope_tab = (float2*)take((size_t)std::max<size_t>(N, 64) * 20 * 8);  // a grid side is at most N patches
  f.xf = (float*)take(D * 4);
  f.logits = (float*)take(V * 4);
  f.pos3 = (int*)take(3 * S * 4);
  f.tok = (int*)take(16 * 4);
  f.keys = (unsigned long long*)take(16 * 8);
  w.hid = (float*)take(B * D * 4);
  w.xf = (float*)take(B * D * 4);
  w.xb = (bf16*)take(B * std::max(std::max(D, F), Hhd) * 2);
  w.qkv = (bf16*)take(B * d.llm_qkv_n * 2);
  w.attn = (bf16*)take(B * Hhd * 2);
  w.act = (bf16*)take(B * F * 2);
  w.logits = (float*)take(B * V * 4);
  const size_t nch = (max_ctx + 255) / 256;
  const size_t nparts = std::max(nch, (size_t)(max_ctx + 127) / 128 * 4);  // >= 128-key chunks of the fused kernel  // decode attention partials per head
  // >= the fused decode's chunk partials: B x KV x ceil((max_ctx + 1) / 128) x (32 + (H / KV) hd)
  const size_t fused_parts = B * m.llm_kv_heads * ((max_ctx + 1 + 127) / 128) * (32 + (size_t)(m.llm_heads / m.llm_kv_heads) * m.head_dim);
  // >= the virtual-CTA decode attention's warp states: B x H x (8 virtual CTAs x 6 warps) x (hd + 2)
  const size_t vstates = B * m.llm_heads * 48 * (size_t)(m.head_dim + 2);
  w.attn_ws = (float*)take(std::max(std::max(B * m.llm_heads * nparts * (m.head_dim + 2), fused_parts), vstates) * 4);
  // split partials: mma.sync GEMVs 16 x B x N, gemv_umma P x B x N with N * P <= 2^20 (gemv_umma_plan)
  w.gemv_ws = (float*)take(std::max((size_t)16 * std::max(std::max(D, F), (size_t)d.llm_qkv_n), (size_t)1 << 20) * B * 4);
  w.tickets = (int*)take(8192 * 4);
  w.qkvf = (float*)take(B * d.llm_qkv_n * 4);
  w.ss = (float*)take(B * ((D / 64 + 3) / 4 * 4) * 4);
  w.xlo = (bf16*)take(B * D * 2);
  w.bar = (unsigned long long*)take(512 * 8);  // per-phase counters of the fused decode kernel
  w.rows = (DecodeRow*)take(B * sizeof(DecodeRow));
  w.tok = (int*)take(B * 4);
  w.keys = (unsigned long long*)take(B * 8);
  // CHUNK mode (hybrid iterations): up to NOVA_CHUNK_MAX prefill rows + 16 decode rows
  Engine::HybWS h{};
  {
    const size_t MH = NOVA_CHUNK_MAX + 16;
    h.pre = (float*)take(S * D * 4);
    h.hid = (float*)take(MH * D * 4);
    h.xf = (float*)take(17 * D * 4);
    h.logits = (float*)take(17 * V * 4);
    h.xb = (bf16*)take(MH * std::max(std::max(D, F), Hhd) * 2);
    h.qkv = (bf16*)take(MH * d.llm_qkv_n * 2);
    h.attn = (bf16*)take(MH * Hhd * 2);
    h.act = (bf16*)take(MH * F * 2);
    h.rows = (DecodeRow*)take(MH * sizeof(DecodeRow));
    h.lm_rows = (DecodeRow*)take(17 * sizeof(DecodeRow));
    h.pos3 = (int*)take(3 * NOVA_CHUNK_MAX * 4);
    h.tok = (int*)take(17 * 4);
    h.keys = (unsigned long long*)take(17 * 8);
  }
  const size_t pix = (size_t)m.in_ch * N * m.patch * m.patch;
  bf16* d_pix = (bf16*)take(n_slots * pix * 2);
  int* d_prompt = (int*)take((size_t)n_slots * c.max_prompt * 4);
  int* d_bt = (int*)take((size_t)n_slots * max_pages * 4);
  int* d_last = (int*)take((size_t)n_slots * 4);
  if (e) {
    e->fw = f;
    e->dw = w;
    e->hw.pre = h.pre, e->hw.hid = h.hid, e->hw.xf = h.xf, e->hw.logits = h.logits, e->hw.xb = h.xb;
    e->hw.qkv = h.qkv, e->hw.attn = h.attn, e->hw.act = h.act, e->hw.rows = h.rows, e->hw.lm_rows = h.lm_rows;
    e->hw.pos3 = h.pos3, e->hw.tok = h.tok, e->hw.keys = h.keys;
    e->d_pix = d_pix;
    e->d_prompt = d_prompt;
    e->d_bt = d_bt;
    e->d_last = d_last;
    e->pix_stride = pix;
    e->max_pages_per_req = max_pages;
    e->n_slots_total = n_slots;
  }
  return off;
}

// ---------------------------------------------------------------- weight loading
static bool parse_idx(const std::string& s, const std::string& pre, int* idx, std::string* rest) {
  if (s.compare(0, pre.size(), pre) != 0) return false;
  size_t p = pre.size(), q = s.find('.', p);
  if (q == std::string::npos) return false;
  *idx = std::atoi(s.substr(p, q - p).c_str());
  *rest = s.substr(q + 1);
  return true;
}

nova_status Engine::load_tensor(const char* cname, const void* src, uint64_t nbytes, int on_dev) {
  if (sim) return NOVA_OK;
  const std::string name(cname);
  const auto& m = dims.m;
  const size_t D = m.llm_dim, F = m.llm_ffn, hd = m.head_dim;
  auto copy = [&](void* dst, size_t expect) -> nova_status {
    if (nbytes != expect) return fail(NOVA_E_INVAL, "size mismatch for " + name);
    if (cudaMemcpy(dst, src, nbytes, cudaMemcpyDefault) != cudaSuccess)
      return fail(NOVA_E_CUDA, "copy failed for " + name);
    return NOVA_OK;
  };
  int i;
  std::string rest;
  if (name == "model.visual.patch_embed.proj.weight") return copy(W.patch_w, (size_t)m.vit_dim * dims.patch_dim * 2);
  if (parse_idx(name, "model.visual.blocks.", &i, &rest)) {
    if (i < 0 || i >= m.vit_depth) return fail(NOVA_E_NOTFOUND, name);
    const size_t Dv = m.vit_dim, Mv = m.vit_mlp;
    size_t off, n;
    if (rest == "norm1.weight") off = vl.n1g, n = Dv;
    else if (rest == "norm1.bias") off = vl.n1b, n = Dv;
    else if (rest == "norm2.weight") off = vl.n2g, n = Dv;
    else if (rest == "norm2.bias") off = vl.n2b, n = Dv;
    else if (rest == "attn.qkv.weight") off = vl.qkv_w, n = 3 * Dv * Dv;
    else if (rest == "attn.qkv.bias") off = vl.qkv_b, n = 3 * Dv;
    else if (rest == "attn.proj.weight") off = vl.proj_w, n = Dv * Dv;
    else if (rest == "attn.proj.bias") off = vl.proj_b, n = Dv;
    else if (rest == "mlp.fc1.weight") off = vl.fc1_w, n = Mv * Dv;
    else if (rest == "mlp.fc1.bias") off = vl.fc1_b, n = Mv;
    else if (rest == "mlp.fc2.weight") off = vl.fc2_w, n = Dv * Mv;
    else if (rest == "mlp.fc2.bias") off = vl.fc2_b, n = Dv;
    else return fail(NOVA_E_NOTFOUND, name);
    if (vit_K > 0) {  // offload: the layer lives in the pinned host arena
      return copy(host_vit + (size_t)i * vl.elems + off, n * 2);
    }
    return copy(W.vit_dev[i] + off, n * 2);
  }
  if (name == "model.visual.merger.ln_q.weight") return copy(W.mlnq_g, (size_t)m.vit_dim * 2);
  if (name == "model.visual.merger.ln_q.bias") return copy(W.mlnq_b, (size_t)m.vit_dim * 2);
  if (name == "model.visual.merger.mlp.0.weight") return copy(W.m1_w, (size_t)dims.merge_dim * dims.merge_dim * 2);
  if (name == "model.visual.merger.mlp.0.bias") return copy(W.m1_b, (size_t)dims.merge_dim * 2);
  if (name == "model.visual.merger.mlp.2.weight") return copy(W.m2_w, D * dims.merge_dim * 2);
  if (name == "model.visual.merger.mlp.2.bias") return copy(W.m2_b, D * 2);
  if (name == "model.language_model.embed_tokens.weight") return copy(W.embed, (size_t)m.vocab * D * 2);
  if (name == "model.language_model.norm.weight") return copy(W.final_norm, D * 2);
  if (name == "lm_head.weight") {
    if (m.tie_embed) return NOVA_OK;
    return copy(W.lm_head, (size_t)m.vocab * D * 2);
  }
  if (parse_idx(name, "model.language_model.layers.", &i, &rest)) {
    if (i < 0 || i >= m.llm_layers) return fail(NOVA_E_NOTFOUND, name);
    LlmLayerW& L = W.llm[i];
    const size_t H = m.llm_heads, KV = m.llm_kv_heads;
    if (rest == "input_layernorm.weight") return copy(L.ln1, D * 2);
    if (rest == "post_attention_layernorm.weight") return copy(L.ln2, D * 2);
    if (rest == "self_attn.q_proj.weight") return copy(L.qkv_w, H * hd * D * 2);
    if (rest == "self_attn.k_proj.weight") return copy(L.qkv_w + H * hd * D, KV * hd * D * 2);
    if (rest == "self_attn.v_proj.weight") return copy(L.qkv_w + (H + KV) * hd * D, KV * hd * D * 2);
    if (rest == "self_attn.q_proj.bias") return copy(L.qkv_b, H * hd * 2);
    if (rest == "self_attn.k_proj.bias") return copy(L.qkv_b + H * hd, KV * hd * 2);
    if (rest == "self_attn.v_proj.bias") return copy(L.qkv_b + (H + KV) * hd, KV * hd * 2);
    if (rest == "self_attn.o_proj.weight") return copy(L.o_w, D * H * hd * 2);
    if (rest == "mlp.down_proj.weight") return copy(L.down_w, D * F * 2);
    if (rest == "mlp.gate_proj.weight" || rest == "mlp.up_proj.weight") {
      // interleave in blocks of 16 rows: [16 gate | 16 up] (layout only)
      if (nbytes != F * D * 2) return fail(NOVA_E_INVAL, "size mismatch for " + name);
      bf16* dst = L.gu_w + (rest == "mlp.up_proj.weight" ? 16 * D : 0);
      if (cudaMemcpy2D(dst, 32 * D * 2, src, 16 * D * 2, 16 * D * 2, F / 16, cudaMemcpyDefault) != cudaSuccess)
        return fail(NOVA_E_CUDA, "copy failed for " + name);
      return NOVA_OK;
    }
    return fail(NOVA_E_NOTFOUND, name);
  }
  return fail(NOVA_E_NOTFOUND, name);
}

}  // namespace nova
