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
  f.xf = (float*)take(D * 4);
  f.logits = (float*)take(V * 4);
  f.pos3 = (int*)take(3 * S * 4);
  f.tok = (int*)take(16 * 4);
  w.hid = (float*)take(B * D * 4);
  w.xf = (float*)take(B * D * 4);
  w.xb = (bf16*)take(B * std::max(std::max(D, F), Hhd) * 2);
  w.qkv = (bf16*)take(B * d.llm_qkv_n * 2);
  w.attn = (bf16*)take(B * Hhd * 2);
  w.act = (bf16*)take(B * F * 2);
  w.logits = (float*)take(B * V * 4);
  const size_t nch = (max_ctx + 255) / 256;
  w.attn_ws = (float*)take(B * m.llm_heads * nch * (m.head_dim + 2) * 4);
  w.rows = (DecodeRow*)take(B * sizeof(DecodeRow));
  w.tok = (int*)take(B * 4);
  const size_t pix = (size_t)m.in_ch * N * m.patch * m.patch;
  bf16* d_pix = (bf16*)take(n_slots * pix * 2);
  int* d_prompt = (int*)take((size_t)n_slots * c.max_prompt * 4);
  int* d_bt = (int*)take((size_t)n_slots * max_pages * 4);
  int* d_last = (int*)take((size_t)n_slots * 4);
  if (e) {
    e->fw = f;
    e->dw = w;
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

// ---------------------------------------------------------------- stage programs
cudaError_t Engine::run_encode(Request* r, cudaStream_t s, int sms) {
  const auto& m = dims.m;
  const int gh = r->gh, gw = r->gw, N = gh * gw, Dv = m.vit_dim, hd = dims.vit_hd;
  const int H = gh * m.patch, Wd = gw * m.patch;
  CUDA_TRY(cudaStreamWaitEvent(s, ev_upload[r->slot], 0));
  CUDA_TRY(patchify(d_pix + (size_t)r->slot * pix_stride, m.in_ch, H, Wd, m.patch, m.temporal_patch, m.merge, fw.x0, s));
  CUDA_TRY(gemm_tc(fw.x0, dims.patch_dim, W.patch_w, dims.patch_dim, fw.vhid, Dv, nullptr, N, Dv, dims.patch_dim,
                   EPI_F32_STORE, sms, s));
  const int L = m.vit_depth;
  for (int l = 0; l < L; ++l) {
    bf16* blk;
    int k = 0;
    if (vit_K > 0) {  // Eq. 7 ring: slot l mod K holds logical layer l
      k = l % vit_K;
      CUDA_TRY(cudaStreamWaitEvent(s, ev_loaded[k], 0));
      blk = W.vit_dev[k];
    } else {
      blk = W.vit_dev[l];
    }
    CUDA_TRY(layernorm(fw.vhid, Dv, blk + vl.n1g, blk + vl.n1b, fw.xb, Dv, N, Dv, m.ln_eps, s));
    CUDA_TRY(gemm_tc(fw.xb, Dv, blk + vl.qkv_w, Dv, fw.qkv, 3 * Dv, blk + vl.qkv_b, N, 3 * Dv, Dv, EPI_BF16, sms, s));
    CUDA_TRY(vit_rope(fw.qkv, N, m.vit_heads, hd, gw, m.merge, m.vit_theta, s));
    CUDA_TRY(flash_attn(fw.qkv, 3 * Dv, fw.attn, Dv, N, m.vit_heads, m.vit_heads, hd, 0, s));
    CUDA_TRY(gemm_tc(fw.attn, Dv, blk + vl.proj_w, Dv, fw.vhid, Dv, blk + vl.proj_b, N, Dv, Dv, EPI_F32_RESID, sms, s));
    CUDA_TRY(layernorm(fw.vhid, Dv, blk + vl.n2g, blk + vl.n2b, fw.xb, Dv, N, Dv, m.ln_eps, s));
    CUDA_TRY(gemm_tc(fw.xb, Dv, blk + vl.fc1_w, Dv, fw.act, m.vit_mlp, blk + vl.fc1_b, N, m.vit_mlp, Dv,
                     EPI_BF16_QGELU, sms, s));
    CUDA_TRY(gemm_tc(fw.act, m.vit_mlp, blk + vl.fc2_w, m.vit_mlp, fw.vhid, Dv, blk + vl.fc2_b, N, Dv, m.vit_mlp,
                     EPI_F32_RESID, sms, s));
    if (vit_K > 0) {  // swap in logical layer (l + K) mod L once slot k is free
      CUDA_TRY(cudaEventRecord(ev_free[k], s));
      CUDA_TRY(cudaStreamWaitEvent(copy_stream, ev_free[k], 0));
      const int nxt = (l + vit_K) % L;
      CUDA_TRY(cudaMemcpyAsync(W.vit_dev[k], host_vit + (size_t)nxt * vl.elems, vl.elems * 2,
                               cudaMemcpyHostToDevice, copy_stream));
      CUDA_TRY(cudaEventRecord(ev_loaded[k], copy_stream));
    }
  }
  // merger: LN -> view [N/4][4 Dv] -> Linear + GELU -> Linear -> E_vis rows 0..n_v of the prefill hidden
  const int nv = N / (m.merge * m.merge), md = dims.merge_dim;
  CUDA_TRY(layernorm(fw.vhid, Dv, W.mlnq_g, W.mlnq_b, fw.xb, Dv, N, Dv, m.ln_eps, s));
  CUDA_TRY(gemm_tc(fw.xb, md, W.m1_w, md, fw.act, md, W.m1_b, nv, md, md, EPI_BF16_GELU, sms, s));
  CUDA_TRY(gemm_tc(fw.act, md, W.m2_w, md, fw.hid, m.llm_dim, W.m2_b, nv, m.llm_dim, md, EPI_F32_STORE, sms, s));
  return cudaSuccess;
}

cudaError_t Engine::run_prefill(Request* r, cudaStream_t s, int sms) {
  const auto& m = dims.m;
  const int D = m.llm_dim, H = m.llm_heads, KV = m.llm_kv_heads, hd = m.head_dim, F = m.llm_ffn;
  const int nv = r->n_v(), S = r->S(), ldq = dims.llm_qkv_n;
  // M-RoPE positions (HF get_rope_index, image first): vision (0, r, c), text st + i
  const int lw = r->gw / m.merge, st = std::max(r->gh / m.merge, lw);
  for (int j = 0; j < S; ++j) {
    if (j < nv) {
      fw.h_pos3[j] = 0;
      fw.h_pos3[S + j] = j / lw;
      fw.h_pos3[2 * S + j] = j % lw;
    } else {
      fw.h_pos3[j] = fw.h_pos3[S + j] = fw.h_pos3[2 * S + j] = st + (j - nv);
    }
  }
  CUDA_TRY(cudaMemcpyAsync(fw.pos3, fw.h_pos3, 3 * S * sizeof(int), cudaMemcpyHostToDevice, s));
  CUDA_TRY(embed(W.embed, D, d_prompt + (size_t)r->slot * cfg.max_prompt, nullptr, nullptr, fw.hid + (size_t)nv * D,
                 D, r->n_prompt, s));
  bf16* pool = reinterpret_cast<bf16*>(buf.kv_dev);
  for (int l = 0; l < m.llm_layers; ++l) {
    const LlmLayerW& L = W.llm[l];
    CUDA_TRY(rmsnorm(fw.hid, D, L.ln1, fw.xb, 0, D, S, D, m.rms_eps, s));
    CUDA_TRY(gemm_tc(fw.xb, D, L.qkv_w, D, fw.qkv, ldq, L.qkv_b, S, ldq, D, EPI_BF16, sms, s));
    CUDA_TRY(llm_rope_kv(fw.qkv, ldq, S, H, KV, hd, m.llm_theta, m.mrope_section[0], m.mrope_section[1], fw.pos3, S,
                         nullptr, r->slot, 0, pool, l, cfg.kv_pages, d_bt, max_pages_per_req, s));
    CUDA_TRY(flash_attn(fw.qkv, ldq, fw.attn, H * hd, S, H, KV, hd, 1, s));
    CUDA_TRY(gemm_tc(fw.attn, H * hd, L.o_w, H * hd, fw.hid, D, nullptr, S, D, H * hd, EPI_F32_RESID, sms, s));
    CUDA_TRY(rmsnorm(fw.hid, D, L.ln2, fw.xb, 0, D, S, D, m.rms_eps, s));
    CUDA_TRY(gemm_tc(fw.xb, D, L.gu_w, D, fw.act, F, nullptr, S, 2 * F, D, EPI_BF16_SILUMUL, sms, s));
    CUDA_TRY(gemm_tc(fw.act, F, L.down_w, F, fw.hid, D, nullptr, S, D, F, EPI_F32_RESID, sms, s));
  }
  // token 0: final RMSNorm (f32 out) of the last row -> lm_head GEMV (f32 logits) -> argmax
  CUDA_TRY(rmsnorm(fw.hid + (size_t)(S - 1) * D, D, W.final_norm, fw.xf, 1, D, 1, D, m.rms_eps, s));
  CUDA_TRY(gemv(fw.xf, 1, D, W.lm_head, m.vocab, D, fw.logits, m.vocab, nullptr, 1, EPI_F32_STORE, s));
  CUDA_TRY(argmax_rows(fw.logits, m.vocab, m.vocab, 1, fw.tok, nullptr, d_last, r->slot, s));
  CUDA_TRY(cudaMemcpyAsync(fw.h_tok, fw.tok, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (cfg.debug_keep_logits)
    CUDA_TRY(cudaMemcpyAsync(fw.h_logits, fw.logits, (size_t)m.vocab * 4, cudaMemcpyDeviceToHost, s));
  return cudaSuccess;
}

cudaError_t Engine::run_decode(const std::vector<Request*>& rq, const std::vector<int>& forced, cudaStream_t s) {
  const auto& m = dims.m;
  const int D = m.llm_dim, H = m.llm_heads, KV = m.llm_kv_heads, hd = m.head_dim, F = m.llm_ffn;
  const int B = (int)rq.size(), ldq = dims.llm_qkv_n;
  int max_ctx = 0;
  for (int b = 0; b < B; ++b) {
    Request* r = rq[b];
    const int e = r->emitted;  // tokens emitted so far; feed token e-1
    const int st = std::max(r->gh / m.merge, r->gw / m.merge);
    dw.h_rows[b] = DecodeRow{r->slot, r->S() + e - 1, st + r->n_prompt - 1 + e, 0};
    max_ctx = std::max(max_ctx, dw.h_rows[b].ctx);
  }
  CUDA_TRY(cudaMemcpyAsync(dw.rows, dw.h_rows, B * sizeof(DecodeRow), cudaMemcpyHostToDevice, s));
  for (int b = 0; b < B; ++b)
    if (forced[b] >= 0) {
      dw.h_forced[b] = forced[b];
      CUDA_TRY(cudaMemcpyAsync(d_last + rq[b]->slot, dw.h_forced + b, 4, cudaMemcpyHostToDevice, s));
    }
  CUDA_TRY(embed(W.embed, D, nullptr, dw.rows, d_last, dw.hid, D, B, s));
  bf16* pool = reinterpret_cast<bf16*>(buf.kv_dev);
  for (int l = 0; l < m.llm_layers; ++l) {
    const LlmLayerW& L = W.llm[l];
    CUDA_TRY(rmsnorm(dw.hid, D, L.ln1, dw.xb, 0, D, B, D, m.rms_eps, s));
    CUDA_TRY(gemv(dw.xb, 0, D, L.qkv_w, ldq, D, dw.qkv, ldq, L.qkv_b, B, EPI_BF16, s));
    CUDA_TRY(llm_rope_kv(dw.qkv, ldq, B, H, KV, hd, m.llm_theta, m.mrope_section[0], m.mrope_section[1], nullptr, 0,
                         dw.rows, 0, 0, pool, l, cfg.kv_pages, d_bt, max_pages_per_req, s));
    CUDA_TRY(decode_attn(dw.qkv, ldq, dw.attn, H * hd, pool, l, cfg.kv_pages, H, KV, hd, d_bt, max_pages_per_req,
                         dw.rows, B, max_ctx, dw.attn_ws, s));
    CUDA_TRY(gemv(dw.attn, 0, H * hd, L.o_w, D, H * hd, dw.hid, D, nullptr, B, EPI_F32_RESID, s));
    CUDA_TRY(rmsnorm(dw.hid, D, L.ln2, dw.xb, 0, D, B, D, m.rms_eps, s));
    CUDA_TRY(gemv(dw.xb, 0, D, L.gu_w, 2 * F, D, dw.act, F, nullptr, B, EPI_BF16_SILUMUL, s));
    CUDA_TRY(gemv(dw.act, 0, F, L.down_w, D, F, dw.hid, D, nullptr, B, EPI_F32_RESID, s));
  }
  CUDA_TRY(rmsnorm(dw.hid, D, W.final_norm, dw.xf, 1, D, B, D, m.rms_eps, s));
  CUDA_TRY(gemv(dw.xf, 1, D, W.lm_head, m.vocab, D, dw.logits, m.vocab, nullptr, B, EPI_F32_STORE, s));
  CUDA_TRY(argmax_rows(dw.logits, m.vocab, m.vocab, B, dw.tok, dw.rows, d_last, -1, s));
  CUDA_TRY(cudaMemcpyAsync(dw.h_tok, dw.tok, B * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (cfg.debug_keep_logits)
    CUDA_TRY(cudaMemcpyAsync(dw.h_logits, dw.logits, (size_t)B * m.vocab * 4, cudaMemcpyDeviceToHost, s));
  return cudaSuccess;
}

}  // namespace nova
