// Internal host-side launchers for the sm_100a stage kernels (L1).  Plain
// pointers and sizes; every call enqueues on `stream` and returns the launch
// status.  Layouts: activations row-major, weights [out][in] (HF convention),
// residual stream f32, GEMM operands bf16, accumulation f32.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <atomic>
#include <vector>

namespace nova {

typedef __nv_bfloat16 bf16;

// Number of libnova kernels launched in this process (incremented by every launcher).
extern std::atomic<unsigned long long> g_kernel_launches;
inline void count_launch(int n = 1) { g_kernel_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

// Programmatic dependent launch (PDL) for the decode chain: the next kernel's CTAs are
// scheduled while the previous one drains and run their weight-streaming prologue early.
extern bool g_use_pdl;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && g_use_pdl) ? 1 : 0;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// GEMM / GEMV epilogues (C = A . W^T + bias, then):
enum Epi {
  EPI_BF16 = 0,         // out bf16
  EPI_BF16_QGELU = 1,   // out bf16, QuickGELU (ViT MLP)
  EPI_BF16_GELU = 2,    // out bf16, GELU(erf) (merger)
  EPI_BF16_SILUMUL = 3, // W rows interleaved gate/up in blocks of 16; out[:, N/2] = silu(g) * u
  EPI_F32_RESID = 4,    // out f32 += result (residual add)
  EPI_F32_STORE = 5,    // out f32 = result
  EPI_QKV_ROPE_KV = 6,  // decode qkv: bias + M-RoPE on q/k; q -> out bf16, k/v -> paged KV cache (GemvAux)
  EPI_F32_ARGMAX = 7,   // logits f32 = result, and greedy argmax into GemvAux::keys (64-bit atomicMax)
  EPI_BF16_ROPE2D = 8,  // ViT qkv: out bf16 = result + bias, 2D RoPE on the q / k columns (GemmRope; hd 80)
};

// tcgen05/TMEM/TMA persistent GEMM. A [M][K] (lda), W [N][K] (ldw), C [M][N] (ldc elems).
// grid = min(tiles, max_ctas): max_ctas is the SM budget of the partition.
// RMSNorm folded into the prefill GEMMs (DESIGN R25, the decode fold's GEMM form):
//  * EPI_F32_RESID with nxout: besides C[m][n] += acc, write x~[m][n] = bf16(C_new[m][n] * ngamma[n]) and, per
//    32-column chunk t = n / 32, nss[m * nss_ld + t] = sum of C_new[m][n]^2 over the chunk (fixed order);
//  * EPI_BF16 / EPI_BF16_SILUMUL with rscale: A is x~ and every accumulator of row m is multiplied by
//    rscale[m] (fold_rows: rsqrt(sum of the row's chunk sums / d + eps)) before the bias.
struct GemmFold {
  const bf16* ngamma = nullptr;
  bf16* nxout = nullptr;
  int ldnx = 0;
  float* nss = nullptr;
  int nss_ld = 0;
  const float* rscale = nullptr;
};
// EPI_BF16_ROPE2D (ViT qkv, hd 80): columns [0, qk_cols) are q | k heads of 80, rotated by the 2D RoPE of
// their row's patch (merge-group-major rows of a grid gw patches wide: as vit_rope) in the epilogue, on
// the f32 accumulators + bias; the tile is forced to the 256 x 160 CTA pair (two heads per tile).
struct GemmRope {
  int qk_cols = 0, gw = 0, merge = 2;
  float log2_theta = 0.f;
  const float2* tab = nullptr;  // rope2d_table: (cos, sin)[pos][j] for j < 20, pos < npos (required)
};
// (cos, sin) of pos * theta^(-4 j / 80) for pos < npos, j < 20 (the ViT 2D RoPE angles at hd 80)
cudaError_t rope2d_table(float2* tab, int npos, float log2_theta, cudaStream_t s);
cudaError_t gemm_tc(const bf16* A, int lda, const bf16* W, int ldw, void* C, int ldc, const bf16* bias, int M,
                    int N, int K, int epi, int max_ctas, cudaStream_t s, const GemmFold* fold = nullptr,
                    const GemmRope* rope = nullptr);
// x~ = bf16(x * g) and the 32-column partial sums of squares ss[r][t] (the first folded RMSNorm's inputs)
cudaError_t rms_prep(const float* x, int ldx, const bf16* g, bf16* y, int ldy, float* ss, int ss_ld, int M, int d,
                     cudaStream_t s);
// rscale[m] = rsqrt((ss[m][0] + ... + ss[m][d / 32 - 1], in chunk order) / d + eps)
cudaError_t fold_rows(const float* ss, int ss_ld, int d, float eps, float* rscale, int M, cudaStream_t s);

// Tile-configuration override (0 auto, 1 single-CTA tiles only, 2 CTA-pair tiles only); returns
// the previous mode.  Test / benchmark hook: a forced mode still picks its tile by shape only.
int gemm_tc_set_mode(int mode);
// Tile chosen for a shape: pair * 1000 + BN (e.g. 1256 = CTA pair, 256 x 256 tile).
int gemm_tc_config(int M, int N, int K);

// Decode GEMV (B <= 16 rows): Y[b][n] = sum_k X[b][k] W[n][k] (+bias), epilogue as above.
// X bf16 (x_f32 = 0) or f32 (x_f32 = 1, split hi/lo on the tensor core).
cudaError_t gemv(const void* X, int x_f32, int ldx, const bf16* W, int N, int K, void* Y, int ldy,
                 const bf16* bias, int B, int epi, cudaStream_t s);

// Persistent TMA-streamed decode GEMV (bf16 X): grid = the partition's SM budget (max_ctas,
// 0 = 148), one continuous weight ring per CTA over its static list of (row block x K split)
// units.  Decomposition from (N, K, epi) only (gemv_tma_plan); split-K partials in ws
// (P * B * N floats) reduced in split order by the last CTA of a row block (tickets: N / RB
// ints, zero on entry, left zero).  EPI_QKV_ROPE_KV needs aux (hd 128).
struct GemvTmaPlan {
  int RB = 64, P = 1, ks = 0, units = 0;
};
GemvTmaPlan gemv_tma_plan(int N, int K, int epi);
int gemv_tma_splits(int N, int K);
struct GemvAux;
// W_blocked: the same weight in the streaming layout (block_weights) -> 8 KB bulk copies
// instead of tensor-map boxes.  X_lo: f32 x given as bf16 hi (X) + lo rows (rmsnorm mode 2);
// required by EPI_F32_ARGMAX (lm_head).
cudaError_t gemv_tma(const bf16* X, int ldx, const bf16* W, int N, int K, void* Y, int ldy, const bf16* bias, int B,
                     int epi, float* ws, int* tickets, cudaStream_t s, int max_ctas = 0,
                     const GemvAux* aux = nullptr, const bf16* W_blocked = nullptr, const bf16* X_lo = nullptr);
extern bool g_use_tma_gemv;
// Decode GEMV on tcgen05 (gemv_umma.cu): weights (streaming layout) as the M = 128 operand, x as
// N = 16; one thread issues the MMAs and tcgen05.commit releases each ring stage.  Same contract as
// gemv_tma (shape-only split plan, bitwise grid / batch invariant); epilogues BF16, SILUMUL,
// F32_RESID, F32_STORE, F32_ARGMAX (X_lo required: f32 x as hi + lo).  sms = partition budget.
extern int g_dec_umma;  // env NOVA_DEC_UMMA (default 1): decode linears on gemv_umma where supported
GemvTmaPlan gemv_umma_plan(int N, int K, int epi);
bool gemv_umma_supported(int N, int K, int epi);
// norm_hid != null (EPI_BF16_SILUMUL, EPI_QKV_ROPE_KV): X is x~ = bf16(h * gamma) and every output row b is
// scaled by rsqrt(mean_k h[b][k]^2 + eps) after the GEMV, before the bias (h = norm_hid rows, ld D) --
// RMSNorm folded (R25).  EPI_QKV_ROPE_KV needs qa (hd 128: one 128-row block per head; rows, pool, bt, ...).
cudaError_t gemv_umma(const bf16* X, int ldx, const bf16* W_blocked, int N, int K, void* Y, int ldy, const bf16* bias,
                      int B, int epi, float* ws, int* tickets, cudaStream_t s, int sms, unsigned long long* keys,
                      const bf16* X_lo, const float* norm_hid = nullptr, float norm_eps = 0.f,
                      const bf16* ngamma = nullptr, bf16* nxout = nullptr, int ldnx = 0,
                      const GemvAux* qa = nullptr);
extern int g_dec_tma_mask;  // decode linears on the persistent TMA GEMV: bit 0 qkv, 1 o, 2 gate|up, 3 down, 4 lm_head

// Flash attention over a fused qkv buffer [S][(H + 2KV) * hd] (q heads, k heads, v heads).
// out [S][H * hd] (ldo).  causal: key j <= query i.  Query head h reads KV head h / (H / KV).
// max_ctas: SM budget of the partition (0 = whole GPU); results do not depend on it.
cudaError_t flash_attn(const bf16* qkv, int ldqkv, bf16* out, int ldo, int S, int H, int KV, int hd, int causal,
                       int max_ctas, cudaStream_t s);
// tcgen05/TMEM/TMA version (hd 80 / 128); flash_attn() dispatches to it for those head dims.
cudaError_t flash_attn_tc(const bf16* qkv, int ldqkv, bf16* out, int ldo, int S, int H, int KV, int hd, int causal,
                          int max_ctas, cudaStream_t s);
extern int g_fmha_version;  // 4 (default, env NOVA_FMHA): v3 + 64-key tiles, double-buffered S; 3: persistent 2-Q-tile ping-pong; 2: 2 CTAs/SM; 1: P in smem
// legacy warp-MMA (mma.sync) version, kept for head dims 16/32/64 and as the measured baseline
cudaError_t flash_attn_mma(const bf16* qkv, int ldqkv, bf16* out, int ldo, int S, int H, int KV, int hd, int causal,
                           cudaStream_t s);

// Paged KV cache: pool [L][P][2][KV][64][hd] bf16; block table per request slot [max_pages].
struct DecodeRow {
  int slot;   // request slot (block table row, last-token cell)
  int ctx;    // tokens already in the cache = cache index of this step's token
  int pos;    // M-RoPE position (t = h = w for generated text)
  int pad;
};
// Extra operands of the fused decode GEMV modes (gemv_ex).
struct GemvAux {
  const bf16* gamma = nullptr;  // x modes 2/3: RMSNorm gain, x = f32 residual rows
  float eps = 0.f;
  int H = 0, KV = 0, hd = 0;    // EPI_QKV_ROPE_KV
  float log2_theta = 0.f;
  const DecodeRow* rows = nullptr;
  bf16* pool = nullptr;
  int layer = 0, n_pages = 0;
  const int* bt = nullptr;
  int max_pages = 0;
  unsigned long long* keys = nullptr;  // EPI_F32_ARGMAX: [B] packed (ordered logit, ~index), zero on entry
  // EPI_F32_RESID, next-norm prep (DESIGN R25): also write nxout[b][n] = bf16(Y_new[b][n] * ngamma[n])
  // -- the next linear contracts W . x~ and applies the RMSNorm row scale after the GEMV
  const bf16* ngamma = nullptr;
  bf16* nxout = nullptr;
  int ldnx = 0;
};
// x modes: 0 bf16, 1 f32 (hi/lo split), 2 f32 residual + RMSNorm on load -> bf16, 3 same -> hi/lo
cudaError_t gemv_ex(const void* X, int xmode, int ldx, const bf16* W, int N, int K, void* Y, int ldy,
                    const bf16* bias, int B, int epi, const GemvAux& aux, cudaStream_t s);
// Fused persistent decode iteration (decode_fused.cu): ONE launch runs embed -> L x (qkv,
// attention, o, gate|up, down) -> lm_head + argmax for B <= 16 rows on a grid of 4 CTAs per SM of
// the decode partition, phases separated by in-kernel grid barriers (decode_fused_barriers(L) <= 512
// monotone per-phase counters, each gaining `grid` per launch; the caller keeps the running base).  Bitwise
// independent of the grid size.  Supported shapes: decode_fused_supported().
extern int g_dec_fused;  // env NOVA_DEC_FUSED=1: use the fused kernel where supported (default 0: the per-op path is faster)
struct DecFusedState;
struct DecFusedSetup {
  int L, D, H, KV, hd, F, V, bmax, n_pages;
  const bf16 *xg, *xlo, *attn, *act, *pool;  // activation tile buffers [bmax][cols]; paged pool
  std::vector<const bf16*> ln1, ln2, qkv_b, qkv_wb, o_wb, gu_wb, down_wb;
};
struct DecFusedRun {
  int L, D, H, KV, hd, F, V, B, max_ctx;
  float eps, theta;
  const bf16 *embed, *final_norm, *lm_wb;
  float* hid;
  bf16 *xg, *xlo;
  float* qkvf;
  bf16 *attn, *act;
  float* ss;
  float* logits;
  unsigned long long* keys;
  float* ws;
  int* tickets;
  float* aws;
  int* atk;
  unsigned long long* bar;
  unsigned long long bar_base;
  bf16* pool;
  int n_pages, max_pages;
  const int* bt;
  const DecodeRow* rows;
  int* last_tok;
  int* tok_out;
  int store_logits;
  int mch;     // aws chunk capacity per (request, KV head): >= ceil((max_ctx + 1) / 128)
  int ph_end;  // 0 = whole iteration; k > 0: stop before phase k (debug bisection)
};
int decode_fused_phase_chunk();  // keys per attention chunk (aws sizing)
bool decode_fused_supported(int D, int H, int KV, int hd, int F, int V);
DecFusedState* decode_fused_create(const DecFusedSetup& su);
void decode_fused_destroy(DecFusedState* st);
int decode_fused_barriers(int L);
int decode_fused_smem();
int decode_fused_grid(int sms);  // CTAs of a launch on an sms-SM partition (0 = whole GPU)
cudaError_t decode_fused(DecFusedState* st, const DecFusedRun& r, int sms, cudaStream_t s);

// keys[r] -> out_tok[r], last_tok[rows[r].slot] (or last_tok[single_slot]); keys reset to 0
cudaError_t argmax_finalize(unsigned long long* keys, int n, int* out_tok, const DecodeRow* rows, int* last_tok,
                            int single_slot, cudaStream_t s);

extern bool g_decode_attn_tc;  // tensor-core decode attention (default) vs the CUDA-core version
// ws: B * H * (ceil((max_ctx+1)/128)*4) * (hd+2) floats; tickets: B * KV ints, zero on entry
// (restored to zero by the kernel).  Tensor-core path: one launch (chunk partials + last-CTA
// fixed-order merge); CUDA-core path: partial + combine kernels.
cudaError_t decode_attn(const bf16* qkv, int ldqkv, bf16* out, int ldo, const bf16* kv_pool, int layer, int n_pages,
                        int H, int KV, int hd, const int* block_tables, int max_pages, const DecodeRow* rows, int B,
                        int max_ctx, float* ws, int* tickets, cudaStream_t s, int sms = 0);

// Persistent paged decode attention (decode_attn_p.cu): units (request, KV head, 128-key chunk)
// on a grid of 3 CTAs per SM of the partition (sms; 0 = whole GPU), chunk partials in ws
// (B * KV * mch * (32 + (H / KV) hd) floats, mch >= ceil((max_ctx + 1) / 128), <= 64) merged in
// chunk order by the CTA that completes a (request, KV head) (tickets: B * KV ints, zero, left
// zero).  Bitwise independent of sms.  B <= 16, H / KV <= 16.
extern int g_dec_attn_p;  // env NOVA_DEC_ATTN_P=1: the decode path uses decode_attn_p (default 0, measured no faster)
int decode_attn_p_chunk();
cudaError_t decode_attn_p(const bf16* qkv, int ld, bf16* out, int ldo, const bf16* pool, int layer, int n_pages, int H,
                          int KV, int hd, const int* bt, int max_pages, const DecodeRow* rows, int B, int max_ctx,
                          float* ws, int* tickets, int mch, int sms, cudaStream_t s);

// Chunked-prefill attention (CHUNK mode): C query rows (cache indices c0 .. c0 + C - 1 of one
// request, K/V already appended) attend causally to the request's paged cache; block_table_row =
// that request's block table (device).  out rows [0, C) (ldo).
cudaError_t chunk_attn(const bf16* qkv, int ld, bf16* out, int ldo, int C, int c0, int H, int KV, int hd,
                       const bf16* kv_pool, int layer, int n_pages, const int* block_table_row, cudaStream_t s);

cudaError_t layernorm(const float* x, int ldx, const bf16* g, const bf16* b, bf16* y, int ldy, int M, int d,
                      float eps, cudaStream_t s);
// y_f32: 0 bf16 rows, 1 f32 rows, 2 bf16 hi rows at y and bf16 lo rows at y + M * ldy
cudaError_t rmsnorm(const float* x, int ldx, const bf16* g, void* y, int y_f32, int ldy, int M, int d, float eps,
                    cudaStream_t s);
// x~ = bf16(x * g) rows (the R25 fold's GEMV input when no preceding epilogue wrote it)
cudaError_t scale_rows_bf16(const float* x, int ldx, const bf16* g, bf16* y, int ldy, int M, int d, cudaStream_t s);
// streaming layout of a decode weight: [N/64][K/64] pre-swizzled 64 x 64 tiles (8 KB each)
cudaError_t block_weights(const bf16* src, bf16* dst, int N, int K, cudaStream_t s);

// pixels bf16 [C][H][W] -> X0 [N][C*T*P*P] merge-group-major rows
cudaError_t patchify(const bf16* pix, int C, int H, int W, int P, int T, int merge, bf16* X0, cudaStream_t s);
// ViT 2D RoPE in place on the q and k parts of qkv [N][3][heads][hd]; grid gw patches wide
cudaError_t vit_rope(bf16* qkv, int N, int heads, int hd, int gw, int merge, float theta, cudaStream_t s);
// LLM M-RoPE in place on q/k of qkv rows + write k, v to the paged cache.
// Row r: positions pos3[0][r], pos3[1][r], pos3[2][r]  (pos3 may be null -> rows[] give pos),
// cache index (ctx0 + r) for prefill (rows == null), or rows[r].ctx for decode.
cudaError_t llm_rope_kv(bf16* qkv, int ldqkv, int nrows, int H, int KV, int hd, float theta, int sec0, int sec1,
                        const int* pos3, int ld_pos, const DecodeRow* rows, int slot, int ctx0, bf16* kv_pool,
                        int layer, int n_pages, const int* block_tables, int max_pages, cudaStream_t s);
// hidden f32 rows <- bf16 table rows; ids from `ids` or from last_tok[rows[b].slot]
cudaError_t embed(const bf16* table, int d, const int* ids, const DecodeRow* rows, const int* last_tok, float* out,
                  int ldo, int n, cudaStream_t s);
// argmax over each row (lowest index on ties); writes out_tok[r] and last_tok[rows[r].slot] (if rows)
cudaError_t argmax_rows(const float* logits, int ldl, int V, int n, int* out_tok, const DecodeRow* rows,
                        int* last_tok, int single_slot, cudaStream_t s);

}  // namespace nova
