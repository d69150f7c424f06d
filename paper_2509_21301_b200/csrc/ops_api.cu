// C ABI of the individual kernels (include/nova_ops.h): argument marshalling only.
#include "../../include/nova_ops.h"
#include "kernels.h"

using namespace nova;

static int st(cudaError_t e) { return e == cudaSuccess ? 0 : -(int)e; }
static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static_assert(sizeof(nova_decode_row) == sizeof(DecodeRow), "row layout");

extern "C" {

int nova_op_gemm(const void* A, int lda, const void* W, int ldw, void* C, int ldc, const void* bias, int M, int N,
                 int K, int epi, int max_ctas, void* stream) {
  return st(gemm_tc((const bf16*)A, lda, (const bf16*)W, ldw, C, ldc, (const bf16*)bias, M, N, K, epi, max_ctas,
                    S(stream)));
}
int nova_op_gemm_fold(const void* A, int lda, const void* W, int ldw, void* C, int ldc, const void* bias, int M, int N,
                      int K, int epi, int max_ctas, const void* ngamma, void* nxout, int ldnx, float* nss, int nss_ld,
                      const float* rscale, void* stream) {
  GemmFold f;
  f.ngamma = (const bf16*)ngamma;
  f.nxout = (bf16*)nxout;
  f.ldnx = ldnx;
  f.nss = nss;
  f.nss_ld = nss_ld;
  f.rscale = rscale;
  return st(gemm_tc((const bf16*)A, lda, (const bf16*)W, ldw, C, ldc, (const bf16*)bias, M, N, K, epi, max_ctas,
                    S(stream), &f));
}
int nova_op_rms_prep(const float* x, int ldx, const void* gamma, void* y, int ldy, float* ss, int ss_ld, int M, int d,
                     void* stream) {
  return st(rms_prep(x, ldx, (const bf16*)gamma, (bf16*)y, ldy, ss, ss_ld, M, d, S(stream)));
}
int nova_op_gemm_rope2d(const void* A, int lda, const void* W, int ldw, void* C, int ldc, const void* bias, int M,
                        int N, int K, int qk_cols, int gw, int merge, float theta, int max_ctas, void* stream) {
  GemmRope r;
  r.qk_cols = qk_cols;
  r.gw = gw;
  r.merge = merge;
  r.log2_theta = log2f(theta);
  // the per-pass angle table (the engine keeps one in its front workspace; this test-facing op keeps a
  // process-wide one, grown on demand -- not for concurrent use)
  static float2* tab = nullptr;
  static int cap = 0;
  if (gw <= 0 || M % gw) return st(cudaErrorInvalidValue);
  const int npos = std::max(gw, M / gw);
  if (npos > cap) {
    if (tab) cudaFree(tab);
    tab = nullptr;
    if (cudaMalloc(&tab, (size_t)npos * 20 * sizeof(float2)) != cudaSuccess) return st(cudaErrorMemoryAllocation);
    cap = npos;
  }
  cudaError_t e = rope2d_table(tab, npos, r.log2_theta, S(stream));
  if (e != cudaSuccess) return st(e);
  r.tab = tab;
  return st(gemm_tc((const bf16*)A, lda, (const bf16*)W, ldw, C, ldc, (const bf16*)bias, M, N, K, EPI_BF16_ROPE2D,
                    max_ctas, S(stream), nullptr, &r));
}
int nova_op_fold_rows(const float* ss, int ss_ld, int d, float eps, float* rscale, int M, void* stream) {
  return st(fold_rows(ss, ss_ld, d, eps, rscale, M, S(stream)));
}
int nova_op_gemm_mode(int mode) { return gemm_tc_set_mode(mode); }
int nova_op_gemm_config(int M, int N, int K) { return gemm_tc_config(M, N, K); }
int nova_op_gemv(const void* X, int x_f32, int ldx, const void* W, int N, int K, void* Y, int ldy, const void* bias,
                 int B, int epi, void* stream) {
  return st(gemv(X, x_f32, ldx, (const bf16*)W, N, K, Y, ldy, (const bf16*)bias, B, epi, S(stream)));
}
int nova_op_gemv_tma(const void* X, int ldx, const void* W, int N, int K, void* Y, int ldy, const void* bias, int B,
                     int epi, float* ws, int32_t* tickets, int max_ctas, void* stream) {
  return st(gemv_tma((const bf16*)X, ldx, (const bf16*)W, N, K, Y, ldy, (const bf16*)bias, B, epi, ws, tickets,
                     S(stream), max_ctas));
}
int nova_op_flash_attn(const void* qkv, int ld, void* out, int ldo, int Sq, int H, int KV, int hd, int causal,
                       int max_ctas, void* stream) {
  return st(flash_attn((const bf16*)qkv, ld, (bf16*)out, ldo, Sq, H, KV, hd, causal, max_ctas, S(stream)));
}
int nova_op_flash_attn_mma(const void* qkv, int ld, void* out, int ldo, int Sq, int H, int KV, int hd, int causal,
                           void* stream) {
  return st(flash_attn_mma((const bf16*)qkv, ld, (bf16*)out, ldo, Sq, H, KV, hd, causal, S(stream)));
}
int nova_op_decode_attn(const void* qkv, int ld, void* out, int ldo, const void* kv_pool, int layer, int n_pages,
                        int H, int KV, int hd, const int32_t* bt, int max_pages, const nova_decode_row* rows, int B,
                        int max_ctx, float* ws, int32_t* tickets, int max_ctas, void* stream) {
  return st(decode_attn((const bf16*)qkv, ld, (bf16*)out, ldo, (const bf16*)kv_pool, layer, n_pages, H, KV, hd, bt,
                        max_pages, (const DecodeRow*)rows, B, max_ctx, ws, tickets, S(stream), max_ctas));
}
int nova_op_gemv_fused(const void* X, int x_mode, int ldx, const void* W, int N, int K, void* Y, int ldy,
                       const void* bias, int B, int epi, const void* gamma, float eps, int H, int KV, int hd,
                       float theta, const nova_decode_row* rows, void* kv_pool, int layer, int n_pages,
                       const int32_t* bt, int max_pages, uint64_t* keys, void* stream) {
  GemvAux a;
  a.gamma = (const bf16*)gamma;
  a.eps = eps;
  a.H = H;
  a.KV = KV;
  a.hd = hd;
  a.log2_theta = theta > 0.f ? log2f(theta) : 0.f;
  a.rows = (const DecodeRow*)rows;
  a.pool = (bf16*)kv_pool;
  a.layer = layer;
  a.n_pages = n_pages;
  a.bt = bt;
  a.max_pages = max_pages;
  a.keys = (unsigned long long*)keys;
  if (x_mode == 0 && epi == EPI_QKV_ROPE_KV) {  // bf16 x: the persistent TMA-streamed kernel
    static float* ws = nullptr;  // split-K partials / tickets of this op-level entry point
    static int* tk = nullptr;
    if (!ws && (cudaMalloc(&ws, (size_t)16 << 20) != cudaSuccess || cudaMalloc(&tk, 8192 * 4) != cudaSuccess ||
                cudaMemset(tk, 0, 8192 * 4) != cudaSuccess))
      return st(cudaErrorMemoryAllocation);
    return st(gemv_tma((const bf16*)X, ldx, (const bf16*)W, N, K, Y, ldy, (const bf16*)bias, B, epi, ws, tk,
                       S(stream), 0, &a));
  }
  return st(gemv_ex(X, x_mode, ldx, (const bf16*)W, N, K, Y, ldy, (const bf16*)bias, B, epi, a, S(stream)));
}
int nova_op_block_weights(const void* W, void* W_blocked, int N, int K, void* stream) {
  return st(block_weights((const bf16*)W, (bf16*)W_blocked, N, K, S(stream)));
}
int nova_op_gemv_stream(const void* X, const void* X_lo, int ldx, const void* W_blocked, int N, int K, void* Y, int ldy,
                        const void* bias, int B, int epi, float* ws, int32_t* tickets, uint64_t* keys, int max_ctas,
                        void* stream) {
  GemvAux a;
  a.keys = (unsigned long long*)keys;
  return st(gemv_tma((const bf16*)X, ldx, nullptr, N, K, Y, ldy, (const bf16*)bias, B, epi, ws, tickets, S(stream),
                     max_ctas, &a, (const bf16*)W_blocked, (const bf16*)X_lo));
}
int nova_op_gemv_umma(const void* X, const void* X_lo, int ldx, const void* W_blocked, int N, int K, void* Y, int ldy,
                      const void* bias, int B, int epi, float* ws, int32_t* tickets, uint64_t* keys, int max_ctas,
                      const float* norm_hid, float norm_eps, const void* ngamma, void* nxout, int ldnx,
                      void* stream) {
  return st(gemv_umma((const bf16*)X, ldx, (const bf16*)W_blocked, N, K, Y, ldy, (const bf16*)bias, B, epi, ws,
                      tickets, S(stream), max_ctas, (unsigned long long*)keys, (const bf16*)X_lo, norm_hid, norm_eps,
                      (const bf16*)ngamma, (bf16*)nxout, ldnx));
}
int nova_op_gemv_umma_qkv(const void* X, int ldx, const void* W_blocked, int N, int K, void* Q, int ldq,
                          const void* bias, int B, const float* norm_hid, float norm_eps, int H, int KV, int hd,
                          float theta, const nova_decode_row* rows, void* kv_pool, int layer, int n_pages,
                          const int32_t* bt, int max_pages, float* ws, int32_t* tickets, int max_ctas, void* stream) {
  GemvAux a;
  a.H = H;
  a.KV = KV;
  a.hd = hd;
  a.log2_theta = theta > 0.f ? log2f(theta) : 0.f;
  a.rows = (const DecodeRow*)rows;
  a.pool = (bf16*)kv_pool;
  a.layer = layer;
  a.n_pages = n_pages;
  a.bt = bt;
  a.max_pages = max_pages;
  return st(gemv_umma((const bf16*)X, ldx, (const bf16*)W_blocked, N, K, Q, ldq, (const bf16*)bias, B,
                      EPI_QKV_ROPE_KV, ws, tickets, S(stream), max_ctas, nullptr, nullptr, norm_hid, norm_eps, nullptr,
                      nullptr, 0, &a));
}
int nova_op_scale_rows_bf16(const float* x, int ldx, const void* gamma, void* y, int ldy, int M, int d, void* stream) {
  return st(scale_rows_bf16(x, ldx, (const bf16*)gamma, (bf16*)y, ldy, M, d, S(stream)));
}
int nova_op_gemv_umma_splits(int N, int K, int epi) { return gemv_umma_plan(N, K, epi).P; }
int nova_op_decode_attn_p(const void* qkv, int ld, void* out, int ldo, const void* kv_pool, int layer, int n_pages,
                          int H, int KV, int hd, const int32_t* bt, int max_pages, const nova_decode_row* rows, int B,
                          int max_ctx, float* ws, int32_t* tickets, int mch, int max_ctas, void* stream) {
  return st(decode_attn_p((const bf16*)qkv, ld, (bf16*)out, ldo, (const bf16*)kv_pool, layer, n_pages, H, KV, hd, bt,
                          max_pages, (const DecodeRow*)rows, B, max_ctx, ws, tickets, mch, max_ctas, S(stream)));
}
int nova_op_chunk_attn(const void* qkv, int ld, void* out, int ldo, int C, int c0, int H, int KV, int hd,
                       const void* kv_pool, int layer, int n_pages, const int32_t* block_table_row, void* stream) {
  return st(chunk_attn((const bf16*)qkv, ld, (bf16*)out, ldo, C, c0, H, KV, hd, (const bf16*)kv_pool, layer, n_pages,
                       block_table_row, S(stream)));
}
int nova_op_argmax_finalize(uint64_t* keys, int n, int32_t* out_tok, const nova_decode_row* rows, int32_t* last_tok,
                            int single_slot, void* stream) {
  return st(argmax_finalize((unsigned long long*)keys, n, out_tok, (const DecodeRow*)rows, last_tok, single_slot,
                            S(stream)));
}
int nova_op_layernorm(const float* x, int ldx, const void* g, const void* b, void* y, int ldy, int M, int d, float eps,
                      void* stream) {
  return st(layernorm(x, ldx, (const bf16*)g, (const bf16*)b, (bf16*)y, ldy, M, d, eps, S(stream)));
}
int nova_op_rmsnorm(const float* x, int ldx, const void* g, void* y, int y_f32, int ldy, int M, int d, float eps,
                    void* stream) {
  return st(rmsnorm(x, ldx, (const bf16*)g, y, y_f32, ldy, M, d, eps, S(stream)));
}
int nova_op_patchify(const void* pix, int C, int H, int W, int P, int T, int merge, void* X0, void* stream) {
  return st(patchify((const bf16*)pix, C, H, W, P, T, merge, (bf16*)X0, S(stream)));
}
int nova_op_vit_rope(void* qkv, int N, int heads, int hd, int gw, int merge, float theta, void* stream) {
  return st(vit_rope((bf16*)qkv, N, heads, hd, gw, merge, theta, S(stream)));
}
int nova_op_llm_rope_kv(void* qkv, int ld, int nrows, int H, int KV, int hd, float theta, int sec0, int sec1,
                        const int32_t* pos3, int ld_pos, const nova_decode_row* rows, int slot, int ctx0,
                        void* kv_pool, int layer, int n_pages, const int32_t* bt, int max_pages, void* stream) {
  return st(llm_rope_kv((bf16*)qkv, ld, nrows, H, KV, hd, theta, sec0, sec1, pos3, ld_pos, (const DecodeRow*)rows,
                        slot, ctx0, (bf16*)kv_pool, layer, n_pages, bt, max_pages, S(stream)));
}
int nova_op_embed(const void* table, int d, const int32_t* ids, const nova_decode_row* rows, const int32_t* last_tok,
                  float* out, int ldo, int n, void* stream) {
  return st(embed((const bf16*)table, d, ids, (const DecodeRow*)rows, last_tok, out, ldo, n, S(stream)));
}
int nova_op_argmax(const float* logits, int ldl, int V, int n, int32_t* out_tok, const nova_decode_row* rows,
                   int32_t* last_tok, int single_slot, void* stream) {
  return st(argmax_rows(logits, ldl, V, n, out_tok, (const DecodeRow*)rows, last_tok, single_slot, S(stream)));
}

}  // extern "C"
