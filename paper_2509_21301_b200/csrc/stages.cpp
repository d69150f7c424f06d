// L2 stage programs: the vision encode, LLM prefill and LLM decode forward passes
// (§II-A, Table stage_duration; SURVEY.md §8(a) rows a5,
// a6, a7) as launch sequences of the sm_100a kernels, with the layer-wise ViT
// weight swap-in of PAPER.md §III-E (Eq. 7; row a9) inside encode.
// Every launch goes through t_gemm / t_gemv / t_attn, which add the kernel's
// ALGORITHMIC work to the pass total and, on sampled passes, bracket it with CUDA
// events on its own stream (live roofline numbers, nova_kernel_stats).
#include <algorithm>
#include <cstdlib>

#include "engine.h"

namespace nova {

// env NOVA_FOLD_NORM=0 keeps the standalone RMSNorm kernel before gate|up (A/B switch)
static const int g_fold_norm = getenv("NOVA_FOLD_NORM") ? atoi(getenv("NOVA_FOLD_NORM")) : 1;

#define CUDA_TRY(x)                   \
  do {                                \
    cudaError_t _e = (x);             \
    if (_e != cudaSuccess) return _e; \
  } while (0)

// ---------------------------------------------------------------- kernel timer
void KTimer::init(int pairs) {
  ev.assign(2 * pairs, nullptr);
  for (auto& e : ev) cudaEventCreate(&e);
}
void KTimer::destroy() {
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  ev.clear();
}
int KTimer::begin(cudaStream_t s) {
  if (!on || n + 2 > (int)ev.size()) return -1;
  cudaEventRecord(ev[n], s);
  return n;
}
void KTimer::end(int i0, int cls, double work, cudaStream_t s) {
  if (i0 < 0) return;
  cudaEventRecord(ev[i0 + 1], s);
  recs.push_back(Rec{cls, work, i0});
  n += 2;
}
void KTimer::harvest(KStat* out, std::mutex& mu) {
  std::lock_guard<std::mutex> g(mu);
  for (const Rec& r : recs) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ev[r.i0], ev[r.i0 + 1]) == cudaSuccess) {
      out[r.cls].ms += ms;
      out[r.cls].work += r.work;
      out[r.cls].launches += 1;
      out[r.cls].sm_ms += ms * share;
    }
  }
  recs.clear();
  n = 0;
}

static cudaError_t t_gemm(Engine* E, int role, int cls, const bf16* A, int lda, const bf16* W, int ldw, void* C,
                          int ldc, const bf16* bias, int M, int N, int K, int epi, int sms, cudaStream_t s,
                          const GemmFold* fold = nullptr, const GemmRope* rope = nullptr) {
  const double w = 2.0 * M * N * K;
  E->pass_work[role] += w;
  const int i = E->ktimer[role].begin(s);
  CUDA_TRY(gemm_tc(A, lda, W, ldw, C, ldc, bias, M, N, K, epi, sms, s, fold, rope));
  E->ktimer[role].end(i, cls, w, s);
  return cudaSuccess;
}

// Decode linear: x_mode 0 = bf16 x, 2 = f32 residual rows with the RMSNorm applied on load
// (gamma in aux), 3 = same in f32 (lm_head).  Algorithmic bytes = weights + x + y (+ KV append).
static cudaError_t t_gemv(Engine* E, int cls, const void* X, int xmode, int ldx, const bf16* W, int N, int K, void* Y,
                          int ldy, const bf16* bias, int B, int epi, const GemvAux& aux, cudaStream_t s) {
  const int nout = epi == EPI_BF16_SILUMUL ? N / 2 : N;
  const int ysz = epi == EPI_F32_RESID ? 8 : ((epi == EPI_F32_STORE || epi == EPI_F32_ARGMAX) ? 4 : 2);
  const double bytes = (double)N * K * 2 + (double)B * K * (xmode ? 4 : 2) + (double)B * nout * ysz;
  E->pass_work[1] += bytes;
  const int i = E->ktimer[1].begin(s);
  CUDA_TRY(gemv_ex(X, xmode, ldx, W, N, K, Y, ldy, bias, B, epi, aux, s));
  E->ktimer[1].end(i, cls, bytes, s);
  return cudaSuccess;
}

// Which decode linears run on gemv_umma: env NOVA_UMMA_MASK (bits as g_dec_tma_mask: 1 qkv, 2 o,
// 4 gate|up, 8 down, 16 lm_head); the choice depends on the op only, never on the partition (co-execution
// is bitwise == serial).  Default all five (31; qkv with its RoPE + KV-append epilogue and the ln1 RMSNorm
// folded, R25, since round 2 session 3): with the stream-K decomposition and one elect per ring
// stage (gemv_umma.cu) decode iterations on 24-SM slices and the full GPU are faster than with o /
// down on the mma.sync GEMVs at B = 2..16 (scripts/gpu_r2_mask.sh; 2B 24 SMs B = 16 6.18 -> 5.97 ms,
// full GPU 2.64 -> 2.29 ms; 7B 24 SMs B = 16 15.5 -> 12.6 ms), the 48-56-SM 2B range excepted.
static int umma_mask() {
  static const int m = getenv("NOVA_UMMA_MASK") ? atoi(getenv("NOVA_UMMA_MASK")) : 31;
  return g_dec_umma ? m : 0;
}

// TMA-streamed decode linear (bf16 x): gate|up, where it streams at ~99% of HBM (scripts/kbench.py)
static cudaError_t t_gemv_tma(Engine* E, const bf16* X, int ldx, const bf16* W, const bf16* Wb, int N, int K, void* Y,
                              int ldy, const bf16* bias, int B, int epi, int sms, const GemvAux* aux, cudaStream_t s,
                              const bf16* X_lo = nullptr, int cls = NOVA_K_DEC_GEMV, const float* norm_hid = nullptr,
                              float norm_eps = 0.f) {
  const int nout = epi == EPI_BF16_SILUMUL ? N / 2 : N;
  const int ysz = epi == EPI_F32_RESID ? 8 : ((epi == EPI_F32_STORE || epi == EPI_F32_ARGMAX) ? 4 : 2);
  const double bytes = (double)N * K * 2 + (double)B * K * (X_lo ? 4 : 2) + (double)B * nout * ysz;
  E->pass_work[1] += bytes;
  const int i = E->ktimer[1].begin(s);
  const int op_bit = epi == EPI_QKV_ROPE_KV ? 1 : epi == EPI_BF16_SILUMUL ? 4 : epi == EPI_F32_ARGMAX ? 16 : (K > N ? 8 : 2);
  if ((umma_mask() & op_bit) && Wb && gemv_umma_supported(N, K, epi) && (epi != EPI_F32_ARGMAX || X_lo)) {
    // tcgen05 consumer (gemv_umma.cu): the same contract, the ring stage released by the MMA commit
    CUDA_TRY(gemv_umma(X, ldx, Wb, N, K, Y, ldy, bias, B, epi, E->dw.gemv_ws, E->dw.tickets, s, sms,
                       aux ? aux->keys : nullptr, X_lo, norm_hid, norm_eps, aux ? aux->ngamma : nullptr,
                       aux ? aux->nxout : nullptr, aux ? aux->ldnx : 0, epi == EPI_QKV_ROPE_KV ? aux : nullptr));
  } else {
    if (norm_hid || (aux && aux->nxout)) return cudaErrorInvalidValue;  // the R25 fold needs the tcgen05 GEMV
    CUDA_TRY(gemv_tma(X, ldx, W, N, K, Y, ldy, bias, B, epi, E->dw.gemv_ws, E->dw.tickets, s, sms, aux, Wb, X_lo));
  }
  E->ktimer[1].end(i, cls, bytes, s);
  return cudaSuccess;
}

// ---------------------------------------------------------------- vision encode (a5)
// §8(f) f4: at a layer-group boundary, move the rest of the front pass to the partition the policy
// gives now (the paper fixes it per pass): the stream switch is an event edge, so kernel order
// and results are unchanged (every kernel is partition-invariant).
cudaError_t Engine::front_regroup(FrontRG* rg, cudaStream_t& s, int& sms) {
  const int want = front_hint.load(std::memory_order_relaxed);
  if (want < 0 || want == rg->s_dec) return cudaSuccess;
  CUDA_TRY(cudaEventRecord(regroup_ev, s));
  cudaStream_t ns = stream_for(0, NOVA_CTX_DV, want);
  CUDA_TRY(cudaStreamWaitEvent(ns, regroup_ev, 0));
  s = ns;
  sms = front_sms(want);
  rg->s_dec = want;
  front_switches.fetch_add(1, std::memory_order_relaxed);
  return cudaSuccess;
}

cudaError_t Engine::run_encode(Request* r, cudaStream_t& s, int sms, FrontRG* rg) {
  const auto& m = dims.m;
  const int gh = r->gh, gw = r->gw, N = gh * gw, Dv = m.vit_dim, hd = dims.vit_hd;
  const int H = gh * m.patch, Wd = gw * m.patch;
  pass_work[0] = 0;
  CUDA_TRY(cudaStreamWaitEvent(s, ev_upload[r->slot], 0));
  CUDA_TRY(patchify(d_pix + (size_t)r->slot * pix_stride, m.in_ch, H, Wd, m.patch, m.temporal_patch, m.merge, fw.x0, s));
  CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.x0, dims.patch_dim, W.patch_w, dims.patch_dim, fw.vhid, Dv, nullptr, N,
                  Dv, dims.patch_dim, EPI_F32_STORE, sms, s));
  const int L = m.vit_depth;
  // 2D RoPE fused into the qkv GEMM epilogue where a 160-column tile holds whole heads (hd 80, the
  // Qwen2-VL ViT; env NOVA_VIT_ROPE_FUSED=0 restores the separate vit_rope kernel)
  static const int g_vrf = getenv("NOVA_VIT_ROPE_FUSED") ? atoi(getenv("NOVA_VIT_ROPE_FUSED")) : 1;
  const bool rope_fused = g_vrf && hd == 80 && (3 * Dv) % 160 == 0 && (2 * Dv) % 160 == 0 && gw % m.merge == 0;
  GemmRope vrope;
  vrope.qk_cols = 2 * Dv, vrope.gw = gw, vrope.merge = m.merge, vrope.log2_theta = log2f(m.vit_theta);
  vrope.tab = fw.rope_tab;
  if (rope_fused) CUDA_TRY(rope2d_table(fw.rope_tab, std::max(gh, gw), vrope.log2_theta, s));
  for (int l = 0; l < L; ++l) {
    if (rg && l > 0 && l % rg->group == 0) CUDA_TRY(front_regroup(rg, s, sms));
    bf16* blk;
    int k = 0;
    if (vit_K > 0) {  // Eq. 7 ring: the slot that received logical layer l
      k = vit_slot_of[l];
      if (k < 0) return cudaErrorInvalidValue;  // ring bookkeeping broken (never expected)
      CUDA_TRY(cudaStreamWaitEvent(s, ev_loaded[k], 0));
      blk = W.vit_dev[k];
    } else {
      blk = W.vit_dev[l];
    }
    CUDA_TRY(layernorm(fw.vhid, Dv, blk + vl.n1g, blk + vl.n1b, fw.xb, Dv, N, Dv, m.ln_eps, s));
    if (rope_fused) {  // 2D RoPE in the qkv GEMM epilogue (hd 80: two heads per 256 x 160 tile)
      CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.xb, Dv, blk + vl.qkv_w, Dv, fw.qkv, 3 * Dv, blk + vl.qkv_b, N,
                      3 * Dv, Dv, EPI_BF16_ROPE2D, sms, s, nullptr, &vrope));
    } else {
      CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.xb, Dv, blk + vl.qkv_w, Dv, fw.qkv, 3 * Dv, blk + vl.qkv_b, N,
                      3 * Dv, Dv, EPI_BF16, sms, s));
      CUDA_TRY(vit_rope(fw.qkv, N, m.vit_heads, hd, gw, m.merge, m.vit_theta, s));
    }
    {
      const double w = 4.0 * N * N * hd * m.vit_heads;
      pass_work[0] += w;
      const int i = ktimer[0].begin(s);
      CUDA_TRY(flash_attn(fw.qkv, 3 * Dv, fw.attn, Dv, N, m.vit_heads, m.vit_heads, hd, 0, sms, s));
      ktimer[0].end(i, NOVA_K_VIT_ATTN, w, s);
    }
    CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.attn, Dv, blk + vl.proj_w, Dv, fw.vhid, Dv, blk + vl.proj_b, N, Dv,
                    Dv, EPI_F32_RESID, sms, s));
    CUDA_TRY(layernorm(fw.vhid, Dv, blk + vl.n2g, blk + vl.n2b, fw.xb, Dv, N, Dv, m.ln_eps, s));
    CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.xb, Dv, blk + vl.fc1_w, Dv, fw.act, m.vit_mlp, blk + vl.fc1_b, N,
                    m.vit_mlp, Dv, EPI_BF16_QGELU, sms, s));
    CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.act, m.vit_mlp, blk + vl.fc2_w, m.vit_mlp, fw.vhid, Dv,
                    blk + vl.fc2_b, N, Dv, m.vit_mlp, EPI_F32_RESID, sms, s));
    if (vit_K > 0) {  // swap in logical layer (l + K) mod L once slot k is free (Eq. 7)
      CUDA_TRY(cudaEventRecord(ev_free[k], s));
      CUDA_TRY(cudaStreamWaitEvent(copy_stream, ev_free[k], 0));
      const int nxt = (l + vit_K) % L;
      vit_slot_of[l] = -1;
      vit_slot_of[nxt] = k;
      CUDA_TRY(cudaMemcpyAsync(W.vit_dev[k], host_vit + (size_t)nxt * vl.elems, vl.elems * 2, cudaMemcpyHostToDevice,
                               copy_stream));
      CUDA_TRY(cudaEventRecord(ev_loaded[k], copy_stream));
    }
  }
  // merger: LN -> view [N/4][4 Dv] -> Linear + GELU -> Linear -> E_vis rows 0..n_v of the prefill hidden
  const int nv = N / (m.merge * m.merge), md = dims.merge_dim;
  CUDA_TRY(layernorm(fw.vhid, Dv, W.mlnq_g, W.mlnq_b, fw.xb, Dv, N, Dv, m.ln_eps, s));
  CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.xb, md, W.m1_w, md, fw.act, md, W.m1_b, nv, md, md, EPI_BF16_GELU, sms,
                  s));
  CUDA_TRY(t_gemm(this, 0, NOVA_K_VIT_GEMM, fw.act, md, W.m2_w, md, fw.hid, m.llm_dim, W.m2_b, nv, m.llm_dim, md,
                  EPI_F32_STORE, sms, s));
  return cudaSuccess;
}

// ---------------------------------------------------------------- LLM prefill (a6)
cudaError_t Engine::run_prefill(Request* r, cudaStream_t& s, int sms, FrontRG* rg) {
  const auto& m = dims.m;
  const int D = m.llm_dim, H = m.llm_heads, KV = m.llm_kv_heads, hd = m.head_dim, F = m.llm_ffn;
  const int nv = r->n_v(), S = r->S(), ldq = dims.llm_qkv_n;
  pass_work[0] = 0;
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
  // RMSNorm folded into the GEMMs (R25, the decode fold's GEMM form; experimental, env NOVA_PREFILL_FOLD=1):
  // the residual GEMMs write the next norm's x~ = bf16(h * gamma) and 32-column sums of h^2, fold_rows turns
  // them into row scales, qkv / gate|up scale their rows after the GEMM.  Measured 1-4% slower than the
  // rmsnorm kernel it replaces (2B 4.71 vs 4.64 ms, 7B 16.4-16.7 vs 15.8-16.6 ms), so off.
  static const int g_pfold = getenv("NOVA_PREFILL_FOLD") ? atoi(getenv("NOVA_PREFILL_FOLD")) : 0;
  const bool pfold = g_pfold && g_fold_norm && D % 128 == 0;
  GemmFold fin, fout;
  fin.rscale = fw.rscale;
  fout.nxout = fw.xb, fout.ldnx = D, fout.nss = fw.nss, fout.nss_ld = D / 32;
  if (pfold) {
    CUDA_TRY(rms_prep(fw.hid, D, W.llm[0].ln1, fw.xb, D, fw.nss, D / 32, S, D, s));
    CUDA_TRY(fold_rows(fw.nss, D / 32, D, m.rms_eps, fw.rscale, S, s));
  }
  for (int l = 0; l < m.llm_layers; ++l) {
    if (rg && l > 0 && l % rg->group == 0) CUDA_TRY(front_regroup(rg, s, sms));
    const LlmLayerW& L = W.llm[l];
    if (!pfold) CUDA_TRY(rmsnorm(fw.hid, D, L.ln1, fw.xb, 0, D, S, D, m.rms_eps, s));
    CUDA_TRY(t_gemm(this, 0, NOVA_K_LLM_GEMM, fw.xb, D, L.qkv_w, D, fw.qkv, ldq, L.qkv_b, S, ldq, D, EPI_BF16, sms, s,
                    pfold ? &fin : nullptr));
    CUDA_TRY(llm_rope_kv(fw.qkv, ldq, S, H, KV, hd, m.llm_theta, m.mrope_section[0], m.mrope_section[1], fw.pos3, S,
                         nullptr, r->slot, 0, pool, l, cfg.kv_pages, d_bt, max_pages_per_req, s));
    {
      const double w = 2.0 * S * S * hd * H;
      pass_work[0] += w;
      const int i = ktimer[0].begin(s);
      CUDA_TRY(flash_attn(fw.qkv, ldq, fw.attn, H * hd, S, H, KV, hd, 1, sms, s));
      ktimer[0].end(i, NOVA_K_PRE_ATTN, w, s);
    }
    fout.ngamma = L.ln2;
    CUDA_TRY(t_gemm(this, 0, NOVA_K_LLM_GEMM, fw.attn, H * hd, L.o_w, H * hd, fw.hid, D, nullptr, S, D, H * hd,
                    EPI_F32_RESID, sms, s, pfold ? &fout : nullptr));
    if (pfold)
      CUDA_TRY(fold_rows(fw.nss, D / 32, D, m.rms_eps, fw.rscale, S, s));
    else
      CUDA_TRY(rmsnorm(fw.hid, D, L.ln2, fw.xb, 0, D, S, D, m.rms_eps, s));
    CUDA_TRY(t_gemm(this, 0, NOVA_K_LLM_GEMM, fw.xb, D, L.gu_w, D, fw.act, F, nullptr, S, 2 * F, D, EPI_BF16_SILUMUL,
                    sms, s, pfold ? &fin : nullptr));
    fout.ngamma = l + 1 < m.llm_layers ? W.llm[l + 1].ln1 : nullptr;  // the last layer's feeds only the final norm
    CUDA_TRY(t_gemm(this, 0, NOVA_K_LLM_GEMM, fw.act, F, L.down_w, F, fw.hid, D, nullptr, S, D, F, EPI_F32_RESID, sms,
                    s, (pfold && fout.ngamma) ? &fout : nullptr));
    if (pfold && fout.ngamma) CUDA_TRY(fold_rows(fw.nss, D / 32, D, m.rms_eps, fw.rscale, S, s));
  }
  // token 0: final RMSNorm of the last row (applied on load, f32) -> lm_head -> fused greedy argmax
  pass_work[0] += 2.0 * D * m.vocab;
  {
    GemvAux ax;
    ax.gamma = W.final_norm;
    ax.eps = m.rms_eps;
    ax.keys = fw.keys;
    CUDA_TRY(gemv_ex(fw.hid + (size_t)(S - 1) * D, 3, D, W.lm_head, m.vocab, D, fw.logits, m.vocab, nullptr, 1,
                     EPI_F32_ARGMAX, ax, s));
  }
  CUDA_TRY(argmax_finalize(fw.keys, 1, fw.tok, nullptr, d_last, r->slot, s));
  CUDA_TRY(cudaMemcpyAsync(fw.h_tok, fw.tok, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (cfg.debug_keep_logits)
    CUDA_TRY(cudaMemcpyAsync(fw.h_logits, fw.logits, (size_t)m.vocab * 4, cudaMemcpyDeviceToHost, s));
  return cudaSuccess;
}

// ---------------------------------------------------------------- LLM decode iteration (a7)
cudaError_t Engine::run_decode(const std::vector<Request*>& rq, const std::vector<int>& forced, cudaStream_t s,
                               int sms) {
  const auto& m = dims.m;
  const int D = m.llm_dim, H = m.llm_heads, KV = m.llm_kv_heads, hd = m.head_dim, F = m.llm_ffn;
  const int B = (int)rq.size(), ldq = dims.llm_qkv_n;
  pass_work[1] = 0;
  int max_ctx = 0;
  double kv_bytes_layer = 0;
  for (int b = 0; b < B; ++b) {
    Request* r = rq[b];
    const int e = r->emitted;  // tokens emitted so far; feed token e-1
    const int st = std::max(r->gh / m.merge, r->gw / m.merge);
    dw.h_rows[b] = DecodeRow{r->slot, r->S() + e - 1, st + r->n_prompt - 1 + e, 0};
    max_ctx = std::max(max_ctx, dw.h_rows[b].ctx);
    kv_bytes_layer += (double)(dw.h_rows[b].ctx + 1) * 2 * KV * hd * 2;
  }
  CUDA_TRY(cudaMemcpyAsync(dw.rows, dw.h_rows, B * sizeof(DecodeRow), cudaMemcpyHostToDevice, s));
  for (int b = 0; b < B; ++b)
    if (forced[b] >= 0) {
      dw.h_forced[b] = forced[b];
      CUDA_TRY(cudaMemcpyAsync(d_last + rq[b]->slot, dw.h_forced + b, 4, cudaMemcpyHostToDevice, s));
    }
  bf16* pool = reinterpret_cast<bf16*>(buf.kv_dev);
  int l0 = 0, sub0 = 0;  // where the per-op path starts (layer, sub-step)
  if (dfs) {  // one persistent launch for the whole iteration (decode_fused.cu)
    const size_t wbytes = ((size_t)m.llm_layers * ((size_t)ldq * D + (size_t)D * H * hd + 3 * (size_t)F * D) +
                           (size_t)m.vocab * D) * 2;
    const double bytes = (double)wbytes + kv_bytes_layer * m.llm_layers;
    pass_work[1] = bytes;
    DecFusedRun fr{};
    fr.L = m.llm_layers, fr.D = D, fr.H = H, fr.KV = KV, fr.hd = hd, fr.F = F, fr.V = m.vocab, fr.B = B;
    fr.max_ctx = max_ctx, fr.eps = m.rms_eps, fr.theta = m.llm_theta;
    fr.embed = W.embed, fr.final_norm = W.final_norm, fr.lm_wb = W.lm_head_b;
    fr.hid = dw.hid, fr.xg = dw.xb, fr.xlo = dw.xlo, fr.qkvf = dw.qkvf, fr.attn = dw.attn, fr.act = dw.act;
    fr.ss = dw.ss, fr.logits = dw.logits, fr.keys = dw.keys, fr.ws = dw.gemv_ws, fr.tickets = dw.tickets;
    fr.aws = dw.attn_ws, fr.atk = dw.tickets + 4096, fr.bar = dw.bar, fr.bar_base = dec_bar_base;
    fr.pool = pool, fr.n_pages = cfg.kv_pages, fr.max_pages = max_pages_per_req, fr.bt = d_bt, fr.rows = dw.rows;
    fr.last_tok = d_last, fr.tok_out = dw.tok, fr.store_logits = cfg.debug_keep_logits;
    fr.mch = attn_mch();
    // debug bisection (env NOVA_DEC_FUSED_STOP = k): the fused kernel runs phases < k (0 embed,
    // 1 + 5 l + {0 qkv, 1 attention, 2 o, 3 gate|up, 4 down}, 5 L + 1 lm_head), the per-op path
    // finishes the iteration from there (k = 1 + 5 l + {0, 2, 3, 4} or 5 L + 1)
    static const int stop = getenv("NOVA_DEC_FUSED_STOP") ? atoi(getenv("NOVA_DEC_FUSED_STOP")) : 0;
    fr.ph_end = stop;
    const int i = ktimer[1].begin(s);
    CUDA_TRY(decode_fused(dfs, fr, sms, s));
    ktimer[1].end(i, NOVA_K_DEC_FUSED, bytes, s);
    dec_bar_base += (unsigned long long)decode_fused_grid(sms);  // every phase counter gains one arrival per CTA
    static const int halt = getenv("NOVA_DEC_FUSED_HALT") ? atoi(getenv("NOVA_DEC_FUSED_HALT")) : 0;
    if (halt) {  // debug: stop the engine right after the (partial) fused kernel, buffers intact
      CUDA_TRY(cudaStreamSynchronize(s));
      return cudaErrorNotReady;
    }
    if (stop <= 0) {
      CUDA_TRY(cudaMemcpyAsync(dw.h_tok, dw.tok, B * sizeof(int), cudaMemcpyDeviceToHost, s));
      if (cfg.debug_keep_logits)
        CUDA_TRY(cudaMemcpyAsync(dw.h_logits, dw.logits, (size_t)B * m.vocab * 4, cudaMemcpyDeviceToHost, s));
      return cudaSuccess;
    }
    l0 = stop > 5 * m.llm_layers ? m.llm_layers : (stop - 1) / 5;
    sub0 = stop > 5 * m.llm_layers ? 0 : (stop - 1) % 5;
    if (sub0 == 1) return cudaErrorInvalidValue;  // the per-op path cannot resume at attention
  } else {
    CUDA_TRY(embed(W.embed, D, nullptr, dw.rows, d_last, dw.hid, D, B, s));
  }
  GemvAux qa;  // RMSNorm(ln1) on load; bias + RoPE + KV append epilogue
  qa.eps = m.rms_eps;
  qa.H = H;
  qa.KV = KV;
  qa.hd = hd;
  qa.log2_theta = log2f(m.llm_theta);
  qa.rows = dw.rows;
  qa.pool = pool;
  qa.n_pages = cfg.kv_pages;
  qa.bt = d_bt;
  qa.max_pages = max_pages_per_req;
  // Per linear: the persistent TMA GEMV over the streaming layout, sized to the decode partition
  // (sms SMs, 4 CTAs each), or the register-streaming GEMV (fixed grid; RMSNorm on load for qkv).
  // g_dec_tma_mask bit 0 qkv, 1 o, 2 gate|up, 3 down, 4 lm_head (env NOVA_DEC_TMA overrides).
  // Default, from the model shape only (scripts/gpu_s3p.sh, decode iterations on 8..148 SMs):
  // gate|up, down and lm_head on the TMA GEMV; o as well once it is >= 8 M weights (7B: 4-15%
  // faster on slices, level on the full GPU; 2B's 2.4 M o-proj is faster on the register GEMV).
  // Round 2 session 3: with the stream-K gemv_umma (+ qkv on it, umma_mask) the o-proj goes there for
  // every shape -- 2B decode B = 2 / 16 on a 24-SM slice 2.56 -> 2.38 / 5.65 -> 5.21 ms, full GPU level
  // (scripts/gpu_r2_qkv.sh).
  const int tm = g_dec_tma_mask >= 0 ? g_dec_tma_mask : 30;
  const bool rope_tma = (tm & 1) && hd == 128;
  // qkv on gemv_umma (RoPE + KV append in its epilogue) with RMSNorm(ln1) folded (R25): x~ = bf16(h * ln1)
  // comes from the previous layer's down-proj epilogue (or a scale kernel for the first layer run here)
  const bool qkv_umma = (umma_mask() & 1) && hd == 128 && g_fold_norm && gemv_umma_supported(ldq, D, EPI_QKV_ROPE_KV);
  bool xt_ln1 = false;  // dw.xb holds x~ for this layer's ln1
  for (int l = l0; l < m.llm_layers; ++l) {
    const LlmLayerW& L = W.llm[l];
    qa.gamma = L.ln1;
    qa.layer = l;
    const int sub = l == l0 ? sub0 : 0;
    if (sub > 0) goto resume;
    if (qkv_umma) {
      if (!xt_ln1) CUDA_TRY(scale_rows_bf16(dw.hid, D, L.ln1, dw.xb, D, B, D, s));
      CUDA_TRY(t_gemv_tma(this, dw.xb, D, L.qkv_w, L.qkv_wb, ldq, D, dw.qkv, ldq, L.qkv_b, B, EPI_QKV_ROPE_KV, sms,
                          &qa, s, nullptr, NOVA_K_DEC_GEMV, dw.hid, m.rms_eps));
    } else if (rope_tma) {
      CUDA_TRY(rmsnorm(dw.hid, D, L.ln1, dw.xb, 0, D, B, D, m.rms_eps, s));
      CUDA_TRY(t_gemv_tma(this, dw.xb, D, L.qkv_w, L.qkv_wb, ldq, D, dw.qkv, ldq, L.qkv_b, B, EPI_QKV_ROPE_KV, sms,
                          &qa, s));
    } else {
      CUDA_TRY(t_gemv(this, NOVA_K_DEC_GEMV, dw.hid, 2, D, L.qkv_w, ldq, D, dw.qkv, ldq, L.qkv_b, B, EPI_QKV_ROPE_KV,
                      qa, s));
    }
    {
      pass_work[1] += kv_bytes_layer;
      const int i = ktimer[1].begin(s);
      if (g_dec_attn_p)  // persistent, sized to the partition (decode_attn_p.cu)
        CUDA_TRY(decode_attn_p(dw.qkv, ldq, dw.attn, H * hd, pool, l, cfg.kv_pages, H, KV, hd, d_bt,
                               max_pages_per_req, dw.rows, B, max_ctx, dw.attn_ws, dw.tickets + 4096, attn_mch(), sms,
                               s));
      else
        CUDA_TRY(decode_attn(dw.qkv, ldq, dw.attn, H * hd, pool, l, cfg.kv_pages, H, KV, hd, d_bt, max_pages_per_req,
                             dw.rows, B, max_ctx, dw.attn_ws, dw.tickets + 4096, s, sms));
      ktimer[1].end(i, NOVA_K_DEC_ATTN, kv_bytes_layer, s);
    }
  resume:
    // RMSNorm(ln2) folded (R25) when gate|up runs on gemv_umma and o on a GEMV with the next-norm
    // epilogue (the mma.sync register GEMV or gemv_umma): the o-proj residual epilogue writes
    // x~ = bf16(h * ln2) into dw.xb, gate|up scales rows by rsqrt(mean h^2 + eps).  Shape-only choice.
    const bool o_umma = (tm & 2) && (umma_mask() & 2) && gemv_umma_supported(D, H * hd, EPI_F32_RESID);
    const bool fold = (tm & 4) && (umma_mask() & 4) && (!(tm & 2) || o_umma) && sub == 0 &&
                      gemv_umma_supported(2 * F, D, EPI_BF16_SILUMUL) && g_fold_norm;
    if (sub <= 2) {
    GemvAux oa;
    if (fold) oa.ngamma = L.ln2, oa.nxout = dw.xb, oa.ldnx = D;
    if (tm & 2)
      CUDA_TRY(t_gemv_tma(this, dw.attn, H * hd, L.o_w, L.o_wb, D, H * hd, dw.hid, D, nullptr, B, EPI_F32_RESID, sms,
                          &oa, s));
    else
      CUDA_TRY(t_gemv(this, NOVA_K_DEC_GEMV, dw.attn, 0, H * hd, L.o_w, D, H * hd, dw.hid, D, nullptr, B,
                      EPI_F32_RESID, oa, s));
    }
    if (sub <= 3) {
    if (tm & 4) {
      if (!fold) CUDA_TRY(rmsnorm(dw.hid, D, L.ln2, dw.xb, 0, D, B, D, m.rms_eps, s));
      CUDA_TRY(t_gemv_tma(this, dw.xb, D, L.gu_w, L.gu_wb, 2 * F, D, dw.act, F, nullptr, B, EPI_BF16_SILUMUL, sms,
                          nullptr, s, nullptr, NOVA_K_DEC_GEMV, fold ? dw.hid : nullptr, m.rms_eps));
    } else {
      GemvAux na;
      na.gamma = L.ln2;
      na.eps = m.rms_eps;
      CUDA_TRY(t_gemv(this, NOVA_K_DEC_GEMV, dw.hid, 2, D, L.gu_w, 2 * F, D, dw.act, F, nullptr, B, EPI_BF16_SILUMUL,
                      na, s));
    }
    }
    {
    // the next layer's folded ln1 input from this residual epilogue (gemv_umma or the register GEMV)
    GemvAux da;
    const bool down_umma = (tm & 8) && (umma_mask() & 8) && gemv_umma_supported(D, F, EPI_F32_RESID);
    xt_ln1 = qkv_umma && l + 1 < m.llm_layers && (down_umma || !(tm & 8));
    if (xt_ln1) da.ngamma = W.llm[l + 1].ln1, da.nxout = dw.xb, da.ldnx = D;
    if (tm & 8)
      CUDA_TRY(t_gemv_tma(this, dw.act, F, L.down_w, L.down_wb, D, F, dw.hid, D, nullptr, B, EPI_F32_RESID, sms,
                          &da, s));
    else
      CUDA_TRY(t_gemv(this, NOVA_K_DEC_GEMV, dw.act, 0, F, L.down_w, D, F, dw.hid, D, nullptr, B, EPI_F32_RESID,
                      da, s));
    }
  }
  // final RMSNorm -> lm_head -> fused greedy argmax (f32 lm_head input, R7)
  GemvAux la;
  la.keys = dw.keys;
  if (tm & 16) {  // bf16 hi + lo rows into the streaming GEMV (two products)
    CUDA_TRY(rmsnorm(dw.hid, D, W.final_norm, dw.xb, 2, D, B, D, m.rms_eps, s));
    CUDA_TRY(t_gemv_tma(this, dw.xb, D, W.lm_head, W.lm_head_b, m.vocab, D, dw.logits, m.vocab, nullptr, B,
                        EPI_F32_ARGMAX, sms, &la, s, dw.xb + (size_t)B * D, NOVA_K_LM_HEAD));
  } else {
    CUDA_TRY(rmsnorm(dw.hid, D, W.final_norm, dw.xf, 1, D, B, D, m.rms_eps, s));
    CUDA_TRY(t_gemv(this, NOVA_K_LM_HEAD, dw.xf, 1, D, W.lm_head, m.vocab, D, dw.logits, m.vocab, nullptr, B,
                    EPI_F32_ARGMAX, la, s));
  }
  CUDA_TRY(argmax_finalize(dw.keys, B, dw.tok, dw.rows, d_last, -1, s));
  CUDA_TRY(cudaMemcpyAsync(dw.h_tok, dw.tok, B * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (cfg.debug_keep_logits)
    CUDA_TRY(cudaMemcpyAsync(dw.h_logits, dw.logits, (size_t)B * m.vocab * 4, cudaMemcpyDeviceToHost, s));
  return cudaSuccess;
}

// ---------------------------------------------------------------- CHUNK: hybrid iteration (f1)
// The paper's chunked-prefill baseline (R26): one batch of M = C + B rows --
// rows [0, C) are prefill rows [c0, c0 + C) of reqs[0] (its E_vis | prompt embeds, staged at the
// first chunk), rows [C, M) the decode rows of reqs[1..].  Every linear is one tcgen05 GEMM over
// the M rows; RoPE / KV append per row (M-RoPE positions for the chunk, 1D for generated tokens);
// attention is the paged decode kernel with one query row per token: a chunk row at cache index j
// attends to keys [0, j] (the prefix of earlier chunks + the causal part of its own chunk, both
// already in the pages) -- chunk_attn for the chunk rows (one pass over the prefix per 64-row query
// tile), the paged decode kernel for the decode rows.  lm_head on the last chunk row (token 0, once the prefill completes) and
// on the decode rows.
cudaError_t Engine::run_hybrid(const std::vector<Request*>& rq, const std::vector<int>& forced, cudaStream_t s,
                               int sms) {
  const auto& m = dims.m;
  const int D = m.llm_dim, H = m.llm_heads, KV = m.llm_kv_heads, hd = m.head_dim, F = m.llm_ffn, V = m.vocab;
  const int ldq = dims.llm_qkv_n;
  Request* P = rq[0];
  const int c0 = P->chunk_c0, C = P->chunk_n, B = (int)rq.size() - 1, M = C + B;
  const int nv = P->n_v(), S = P->S();
  const bool last = c0 + C >= S;
  if (C < 1 || C > NOVA_CHUNK_MAX || B > 16) return cudaErrorInvalidValue;
  pass_work[1] = 0;
  bf16* pool = reinterpret_cast<bf16*>(buf.kv_dev);
  if (c0 == 0) {  // stage the request's input rows: E_vis (vision merger output) | prompt embeddings
    CUDA_TRY(cudaMemcpyAsync(hw.pre, fw.hid, (size_t)nv * D * 4, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(embed(W.embed, D, d_prompt + (size_t)P->slot * cfg.max_prompt, nullptr, nullptr, hw.pre + (size_t)nv * D,
                   D, P->n_prompt, s));
  }
  CUDA_TRY(cudaMemcpyAsync(hw.hid, hw.pre + (size_t)c0 * D, (size_t)C * D * 4, cudaMemcpyDeviceToDevice, s));
  // chunk rows: M-RoPE positions (HF get_rope_index, image first) and cache index c0 + r
  const int lw = P->gw / m.merge, st = std::max(P->gh / m.merge, lw);
  int max_ctx = 0;
  for (int r = 0; r < C; ++r) {
    const int j = c0 + r;
    if (j < nv) {
      hw.h_pos3[r] = 0;
      hw.h_pos3[C + r] = j / lw;
      hw.h_pos3[2 * C + r] = j % lw;
    } else {
      hw.h_pos3[r] = hw.h_pos3[C + r] = hw.h_pos3[2 * C + r] = st + (j - nv);
    }
    hw.h_rows[r] = DecodeRow{P->slot, j, hw.h_pos3[2 * C + r], 0};
    max_ctx = std::max(max_ctx, j);
  }
  for (int b = 0; b < B; ++b) {  // decode rows (as run_decode): feed token emitted - 1
    Request* r = rq[1 + b];
    const int e = r->emitted;
    const int stb = std::max(r->gh / m.merge, r->gw / m.merge);
    hw.h_rows[C + b] = DecodeRow{r->slot, r->S() + e - 1, stb + r->n_prompt - 1 + e, 0};
    max_ctx = std::max(max_ctx, hw.h_rows[C + b].ctx);
  }
  int n_lm = 0;  // lm_head rows: [0] the chunk's last row (if it completes the prefill), [1..B] decode rows
  hw.h_lm_rows[0] = DecodeRow{P->slot, S - 1, 0, 0};
  for (int b = 0; b < B; ++b) hw.h_lm_rows[1 + b] = hw.h_rows[C + b];
  CUDA_TRY(cudaMemcpyAsync(hw.rows, hw.h_rows, M * sizeof(DecodeRow), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(hw.lm_rows, hw.h_lm_rows, (B + 1) * sizeof(DecodeRow), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(hw.pos3, hw.h_pos3, 3 * C * sizeof(int), cudaMemcpyHostToDevice, s));
  for (int b = 0; b < B; ++b)
    if (forced[1 + b] >= 0) {
      hw.h_forced[b] = forced[1 + b];
      CUDA_TRY(cudaMemcpyAsync(d_last + rq[1 + b]->slot, hw.h_forced + b, 4, cudaMemcpyHostToDevice, s));
    }
  if (B > 0) CUDA_TRY(embed(W.embed, D, nullptr, hw.rows + C, d_last, hw.hid + (size_t)C * D, D, B, s));
  for (int l = 0; l < m.llm_layers; ++l) {
    const LlmLayerW& L = W.llm[l];
    CUDA_TRY(rmsnorm(hw.hid, D, L.ln1, hw.xb, 0, D, M, D, m.rms_eps, s));
    CUDA_TRY(t_gemm(this, 1, NOVA_K_LLM_GEMM, hw.xb, D, L.qkv_w, D, hw.qkv, ldq, L.qkv_b, M, ldq, D, EPI_BF16, sms, s));
    CUDA_TRY(llm_rope_kv(hw.qkv, ldq, C, H, KV, hd, m.llm_theta, m.mrope_section[0], m.mrope_section[1], hw.pos3, C,
                         nullptr, P->slot, c0, pool, l, cfg.kv_pages, d_bt, max_pages_per_req, s));
    if (B > 0)
      CUDA_TRY(llm_rope_kv(hw.qkv + (size_t)C * ldq, ldq, B, H, KV, hd, m.llm_theta, m.mrope_section[0],
                           m.mrope_section[1], nullptr, 0, hw.rows + C, -1, 0, pool, l, cfg.kv_pages, d_bt,
                           max_pages_per_req, s));
    CUDA_TRY(chunk_attn(hw.qkv, ldq, hw.attn, H * hd, C, c0, H, KV, hd, pool, l, cfg.kv_pages,
                        d_bt + (size_t)P->slot * max_pages_per_req, s));
    if (B > 0)
      CUDA_TRY(decode_attn_p(hw.qkv + (size_t)C * ldq, ldq, hw.attn + (size_t)C * H * hd, H * hd, pool, l,
                             cfg.kv_pages, H, KV, hd, d_bt, max_pages_per_req, hw.rows + C, B, max_ctx, dw.attn_ws,
                             dw.tickets + 4096, attn_mch(), sms, s));
    CUDA_TRY(t_gemm(this, 1, NOVA_K_LLM_GEMM, hw.attn, H * hd, L.o_w, H * hd, hw.hid, D, nullptr, M, D, H * hd,
                    EPI_F32_RESID, sms, s));
    CUDA_TRY(rmsnorm(hw.hid, D, L.ln2, hw.xb, 0, D, M, D, m.rms_eps, s));
    CUDA_TRY(t_gemm(this, 1, NOVA_K_LLM_GEMM, hw.xb, D, L.gu_w, D, hw.act, F, nullptr, M, 2 * F, D, EPI_BF16_SILUMUL,
                    sms, s));
    CUDA_TRY(t_gemm(this, 1, NOVA_K_LLM_GEMM, hw.act, F, L.down_w, F, hw.hid, D, nullptr, M, D, F, EPI_F32_RESID, sms,
                    s));
  }
  // final RMSNorm (f32) -> lm_head -> greedy argmax; the prefill row and the decode rows are two
  // GEMV launches (each <= 16 rows)
  GemvAux la;
  if (last) {
    CUDA_TRY(rmsnorm(hw.hid + (size_t)(C - 1) * D, D, W.final_norm, hw.xf, 1, D, 1, D, m.rms_eps, s));
    la.keys = hw.keys;
    CUDA_TRY(gemv_ex(hw.xf, 1, D, W.lm_head, V, D, hw.logits, V, nullptr, 1, EPI_F32_ARGMAX, la, s));
  }
  if (B > 0) {
    CUDA_TRY(rmsnorm(hw.hid + (size_t)C * D, D, W.final_norm, hw.xf + D, 1, D, B, D, m.rms_eps, s));
    la.keys = hw.keys + 1;
    CUDA_TRY(gemv_ex(hw.xf + D, 1, D, W.lm_head, V, D, hw.logits + V, V, nullptr, B, EPI_F32_ARGMAX, la, s));
  }
  n_lm = B + 1;
  const int lm0 = last ? 0 : 1;
  if (n_lm - lm0 > 0)
    CUDA_TRY(argmax_finalize(hw.keys + lm0, n_lm - lm0, hw.tok + lm0, hw.lm_rows + lm0, d_last, -1, s));
  CUDA_TRY(cudaMemcpyAsync(hw.h_tok, hw.tok, (size_t)n_lm * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (cfg.debug_keep_logits)
    CUDA_TRY(cudaMemcpyAsync(hw.h_logits, hw.logits, (size_t)n_lm * V * 4, cudaMemcpyDeviceToHost, s));
  return cudaSuccess;
}

}  // namespace nova
