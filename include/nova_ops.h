/* nova_ops.h -- C ABI of the individual sm_100a stage kernels (libnova.so).
 *
 * These are the building blocks of the Nova stage programs (vision encode,
 * LLM prefill, LLM decode; §II-A, Table resource_stage
 * P:130-145), exposed one by one for per-kernel parity tests against the CPU
 * oracle and for roofline micro-benchmarks.  The engine ABI is nova.h.
 *
 * Conventions (all calls):
 *   - Every pointer is a DEVICE pointer owned by the caller (allocated e.g. by
 *     torch); the call only enqueues work on `stream` (a cudaStream_t passed as
 *     void*, NULL = legacy default stream) and never synchronises.
 *   - Matrices are row-major with leading dimensions in ELEMENTS; "bf16" is
 *     IEEE bfloat16 bits (uint16), "f32" IEEE float.  Weights are [out][in].
 *   - Return 0 on success, or the negative CUDA error code of the failed
 *     launch (-1 = cudaErrorInvalidValue for unsupported shapes).  Errors of
 *     the asynchronous execution surface on the caller's next synchronisation.
 */
#ifndef NOVA_OPS_H
#define NOVA_OPS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Epilogues shared by GEMM and GEMV:  R = A . W^T + bias  (f32 accumulate)          */
enum {
  NOVA_EPI_BF16 = 0,          /* C bf16 = R                                          */
  NOVA_EPI_BF16_QGELU = 1,    /* C bf16 = R * sigmoid(1.702 R)     (ViT MLP, QuickGELU) */
  NOVA_EPI_BF16_GELU = 2,     /* C bf16 = GELU_erf(R)              (patch merger)      */
  NOVA_EPI_BF16_SILUMUL = 3,  /* W rows interleaved [16 gate | 16 up]*; C[:, N/2] bf16 = silu(gate) * up */
  NOVA_EPI_F32_RESID = 4,     /* C f32 += R                        (residual add)     */
  NOVA_EPI_F32_STORE = 5,     /* C f32 = R                                            */
  NOVA_EPI_QKV_ROPE_KV = 6,   /* decode qkv (nova_op_gemv_fused only): R + bias, M-RoPE on q/k
                                 heads at rows[b].pos; q -> C bf16, k/v -> paged KV cache   */
  NOVA_EPI_F32_ARGMAX = 7     /* C f32 = R, and greedy argmax into keys[b] (nova_op_gemv_fused) */
};

/* Dense linear of the vision encoder / prefill: tcgen05 +
 * TMEM + TMA persistent GEMM.  A [M][K] bf16 (lda), W [N][K] bf16 (ldw), bias
 * bf16 [N] or NULL, C per epilogue (ldc).  Requires N % 64 == 0, lda/ldw/ldc % 8
 * == 0; M, K arbitrary (TMA zero-fills tails).  max_ctas = SM budget (grid cap).
 * Bitwise independent of max_ctas. */
int nova_op_gemm(const void* A, int lda, const void* W, int ldw, void* C, int ldc, const void* bias, int M, int N,
                 int K, int epi, int max_ctas, void* stream);
/* The same GEMM with the prefill RMSNorm fold (DESIGN R25; "kernel fusion ... RMSNorm";
 * RMSNorm(h) W^T = rsqrt(mean h^2 + eps) * ((h * gamma) W^T) row by row):
 *  - epi NOVA_EPI_F32_RESID with nxout != NULL (ngamma bf16 [N], nss f32 required; N % 32 == 0): after
 *    C[m][n] += acc also nxout[m * ldnx + n] = bf16(C[m][n] * ngamma[n]) and, for each 32-column chunk t,
 *    nss[m * nss_ld + t] = sum over the chunk of C[m][n]^2 (one fixed order);
 *  - epi NOVA_EPI_BF16 / NOVA_EPI_BF16_SILUMUL with rscale != NULL: A holds x~ and row m's accumulators are
 *    multiplied by rscale[m] (nova_op_fold_rows) before the bias.
 * NULL pointers = that half off.  Bitwise independent of max_ctas. */
int nova_op_gemm_fold(const void* A, int lda, const void* W, int ldw, void* C, int ldc, const void* bias, int M, int N,
                      int K, int epi, int max_ctas, const void* ngamma, void* nxout, int ldnx, float* nss, int nss_ld,
                      const float* rscale, void* stream);
/* ViT qkv projection with the 2D RoPE in the GEMM epilogue (SURVEY §8(a) a5 "QKV GEMM (+bias) -> 2D-RoPE(q,k)";
 * PAPER.md P:468 "kernel fusion ... RoPE"): C = A W^T + bias in bf16, the columns [0, qk_cols) being q | k
 * heads of hd = 80 rotated by the 2D RoPE of row m's patch -- rows merge-group-major over a grid gw patches
 * wide (merge x merge groups), as nova_op_vit_rope -- on the f32 accumulators before the one bf16 rounding.
 * N and qk_cols multiples of 160 (the kernel takes 256 x 160 CTA-pair tiles: two heads per tile); M = gh * gw.
 * Bitwise independent of max_ctas. */
int nova_op_gemm_rope2d(const void* A, int lda, const void* W, int ldw, void* C, int ldc, const void* bias, int M,
                        int N, int K, int qk_cols, int gw, int merge, float theta, int max_ctas, void* stream);
/* rscale[m] = rsqrt((ss[m * ss_ld + 0] + ... + ss[m * ss_ld + d / 32 - 1], in that order) / d + eps) for
 * M rows (d % 128 == 0, ss_ld % 4 == 0): the folded RMSNorm's row scales from the chunk sums. */
int nova_op_fold_rows(const float* ss, int ss_ld, int d, float eps, float* rscale, int M, void* stream);
/* The first folded RMSNorm's inputs from f32 rows x [M][d] (d % 32 == 0): y = bf16(x * gamma) (ldy) and
 * ss[m * ss_ld + t] = sum of x[m][32 t .. 32 t + 31]^2 in column order. */
int nova_op_rms_prep(const float* x, int ldx, const void* gamma, void* y, int ldy, float* ss, int ss_ld, int M, int d,
                     void* stream);

/* GEMM tile selection.  nova_op_gemm chooses, from the shape alone (never from max_ctas,
 * so results stay bitwise independent of the partition), between single-CTA 128 x BN
 * tiles and CTA-pair (tcgen05 cta_group::2, 2-CTA cluster) 256 x BN tiles.
 * nova_op_gemm_mode(mode): 0 = automatic (default, or env NOVA_GEMM), 1 = single-CTA
 * tiles only, 2 = CTA-pair tiles only, >= 1000 = exactly the tile pair * 1000 + BN
 * (benchmarks); returns the previous mode.  Process-wide, not
 * thread-safe against concurrent nova_op_gemm calls (a test / benchmark hook).
 * nova_op_gemm_config(M, N, K): the tile the current mode picks, pair * 1000 + BN. */
int nova_op_gemm_mode(int mode);
int nova_op_gemm_config(int M, int N, int K);

/* Decode linear (a7): Y[b][n] = sum_k X[b][k] W[n][k] (+bias) for B <= 16 rows.
 * X bf16 (x_f32 = 0) or f32 (x_f32 = 1).  N % 32 == 0, K % 32 == 0, ldx % 8 == 0.
 * Epilogues NOVA_EPI_BF16 / _SILUMUL / _F32_RESID / _F32_STORE.  Row b of Y is
 * bitwise independent of B and of the other rows. */
int nova_op_gemv(const void* X, int x_f32, int ldx, const void* W, int N, int K, void* Y, int ldy, const void* bias,
                 int B, int epi, void* stream);

/* Persistent TMA-streamed decode linear (bf16 X only; PAPER.md P:141, P:283 -- decode is
 * memory-bound and runs on an SM slice): same contract as nova_op_gemv for the
 * bf16 / SiLU / f32-residual / f32-store epilogues (N % 64 == 0, K % 64 == 0).  max_ctas =
 * the SM budget (0 = 148): one CTA per SM streams its units' weight tiles through one smem
 * ring.  ws: f32 workspace of 16*B*N floats for split-K partials; tickets: int32 [N/64]
 * zero-initialised once (the kernel leaves them zero).  Bitwise independent of max_ctas and B. */
int nova_op_gemv_tma(const void* X, int ldx, const void* W, int N, int K, void* Y, int ldy, const void* bias, int B,
                     int epi, float* ws, int32_t* tickets, int max_ctas, void* stream);

/* Flash attention (a5 ViT: causal = 0, KV = H; a6 prefill: causal = 1, GQA; PAPER.md
 * Table resource_stage P:139-140 "Attention").  qkv [S][(H + 2 KV) hd] bf16 (ld): q heads,
 * then k heads, then v heads; out [S][H hd] bf16 (ldo); scale hd^-1/2; hd in {16, 32, 64,
 * 80, 128}.  max_ctas = SM budget of the caller's partition (0 = whole GPU); the output is
 * bitwise independent of it. */
int nova_op_flash_attn(const void* qkv, int ld, void* out, int ldo, int S, int H, int KV, int hd, int causal,
                       int max_ctas, void* stream);

/* Same contract, forced onto the legacy warp-level mma.sync kernel (the measured
 * baseline the tcgen05 path is compared against); hd in {16, 32, 64, 80, 128}.
 * nova_op_flash_attn uses the tcgen05/TMEM kernel for hd 80 and 128. */
int nova_op_flash_attn_mma(const void* qkv, int ld, void* out, int ldo, int S, int H, int KV, int hd, int causal,
                           void* stream);

/* Row descriptor of one decode request (device memory, 16 bytes). */
typedef struct {
  int32_t slot; /* request slot: row of block_tables and of last_tok       */
  int32_t ctx;  /* tokens already cached = cache index of this step's token */
  int32_t pos;  /* M-RoPE position of this step's token (t = h = w)         */
  int32_t pad;
} nova_decode_row;

/* Paged decode attention (a7; PAPER.md P:141, P:283 -- memory-bound, PagedAttention
 * KV layout P:48).  Keys 0..ctx (inclusive) of each row.  kv_pool bf16
 * [layers][n_pages][2][KV][64][hd]; block_tables int32 [slots][max_pages];
 * ws f32 workspace of max(B*H*ceil((max_ctx+1)/64), B*H*48)*(hd+2) floats; tickets int32 [B*KV],
 * zero on entry and left zero (one launch: chunk partials + last-CTA fixed-order merge).
 * ceil((max_ctx+1)/128) <= 64, H/KV <= 16.  Deterministic, batch- and grid-invariant. */
int nova_op_decode_attn(const void* qkv, int ld, void* out, int ldo, const void* kv_pool, int layer, int n_pages,
                        int H, int KV, int hd, const int32_t* block_tables, int max_pages, const nova_decode_row* rows,
                        int B, int max_ctx, float* ws, int32_t* tickets, int max_ctas, void* stream);
/* max_ctas: SM budget of the partition (0 = whole GPU); it picks the K/V ring depth (2 stages, one CTA per
 * SM, or 1 stage, two CTAs per SM) and, when even that takes more than one wave, fewer physical CTAs per
 * (request, KV head) that run the cluster's virtual CTAs in turn and merge through ws -- never the result. */

/* Persistent paged decode attention (decode_attn_p.cu): same contract as nova_op_decode_attn
 * (rows[b] = {slot, ctx, pos, pad}: query b attends keys 0..ctx of its slot's pages; GQA), work
 * units (request, KV head, 128-key chunk) on a grid of 3 CTAs per SM of the partition (max_ctas =
 * SM budget, 0 = whole GPU); ws >= B * KV * mch * (32 + (H / KV) hd) floats with mch >=
 * ceil((max_ctx + 1) / 128) (<= 64), tickets >= B * KV ints (zero on entry, left zero).  Results
 * are bitwise independent of max_ctas and of the other rows of the batch. */
int nova_op_decode_attn_p(const void* qkv, int ld, void* out, int ldo, const void* kv_pool, int layer, int n_pages,
                          int H, int KV, int hd, const int32_t* block_tables, int max_pages,
                          const nova_decode_row* rows, int B, int max_ctx, float* ws, int32_t* tickets, int mch,
                          int max_ctas, void* stream);

/* Chunked-prefill attention (the paper's Chunk baseline; CHUNK mode): C query rows of one
 * request -- q at qkv rows [0, C) (heads 0..H-1, fused q|k|v layout, row stride ld) with cache
 * indices c0 .. c0 + C - 1 -- attend to that request's paged cache (block_table_row: its block
 * table, device; K/V of all C rows already appended), key j visible to row r iff j <= c0 + r;
 * GQA (query head h reads KV head h / (H / KV)), scale hd^-1/2.  out [C][H hd] bf16 (ldo). */
int nova_op_chunk_attn(const void* qkv, int ld, void* out, int ldo, int C, int c0, int H, int KV, int hd,
                       const void* kv_pool, int layer, int n_pages, const int32_t* block_table_row, void* stream);

/* Fused decode linear (a7; "kernel fusion ... RoPE and RMSNorm"):
 * Y = epilogue(Xin . W^T + bias) for B <= 16 rows, where Xin is, by x_mode:
 *   0: X bf16;  1: X f32 (hi/lo bf16 split, exact to ~2^-16);
 *   2: RMSNorm(X f32 residual rows; gamma bf16 [K], eps) rounded to bf16;
 *   3: RMSNorm(X) in f32, hi/lo split (the lm_head input).
 * Epilogues: the NOVA_EPI_* above, plus
 *   NOVA_EPI_QKV_ROPE_KV: W = fused [(H + 2 KV) hd][K] q|k|v rows; bias added, q and k
 *     rotated by RoPE at rows[b].pos (t = h = w for generated text; log2(theta) given as
 *     theta), q -> Y[b] (bf16, ldy), k and v -> kv_pool at cache index rows[b].ctx of
 *     request rows[b].slot (block_tables, max_pages);
 *   NOVA_EPI_F32_ARGMAX: logits -> Y f32, and keys[b] (uint64, zero on entry) receives the
 *     packed (order-preserving logit bits << 32 | ~index) maximum: argmax, ties -> lowest
 *     index.  nova_op_argmax_finalize turns keys into tokens.
 * x_mode 0 with NOVA_EPI_QKV_ROPE_KV runs the persistent TMA-streamed kernel (hd 128).
 * Unused pointer arguments may be NULL.  N % 32 == 0, K % 32 == 0. */
int nova_op_gemv_fused(const void* X, int x_mode, int ldx, const void* W, int N, int K, void* Y, int ldy,
                       const void* bias, int B, int epi, const void* gamma, float eps, int H, int KV, int hd,
                       float theta, const nova_decode_row* rows, void* kv_pool, int layer, int n_pages,
                       const int32_t* block_tables, int max_pages, uint64_t* keys, void* stream);

/* Streaming layout of a decode weight W [N][K] bf16 (N % 64 == 0, K % 64 == 0): W_blocked
 * [N/64][K/64] tiles of 64 rows x 64 k, each tile's 128-byte rows with their 16-byte chunks
 * XOR-swizzled by (row & 7) -- the shared-memory image of a TMA SWIZZLE_128B box, so decode
 * streams one contiguous 8 KB bulk copy per tile (full DRAM bursts on a small SM slice). */
int nova_op_block_weights(const void* W, void* W_blocked, int N, int K, void* stream);

/* Persistent decode linear over a weight in the streaming layout (same contract as
 * nova_op_gemv_tma; max_ctas = SM budget).  X_lo != NULL: the input is f32 given as bf16 hi
 * rows (X) + lo rows (X_lo) (two products on the tensor core); epi may then be
 * NOVA_EPI_F32_STORE or NOVA_EPI_F32_ARGMAX (keys as in nova_op_gemv_fused). */
int nova_op_gemv_stream(const void* X, const void* X_lo, int ldx, const void* W_blocked, int N, int K, void* Y, int ldy,
                        const void* bias, int B, int epi, float* ws, int32_t* tickets, uint64_t* keys, int max_ctas,
                        void* stream);

/* The same decode linear on the 5th-generation tensor cores (gemv_umma.cu): weights in the
 * streaming layout as the M = 128 tcgen05 operand, x as N = 16, one thread issuing the MMAs whose
 * commit frees each ring stage; 128-row blocks whose K range is cut into P shape-only chunks, the
 * result being the left fold of the chunk partials, the blocks x P chunks dealt out to the CTAs as
 * equal contiguous ranges (stream-K) -- results bitwise independent of max_ctas and of the batch
 * composition, not bitwise equal to nova_op_gemv_stream (another accumulation order).  N % 128 == 0, K % 64 == 0, B <= 16; epi NOVA_EPI_BF16,
 * NOVA_EPI_BF16_SILUMUL, NOVA_EPI_F32_RESID, NOVA_EPI_F32_STORE, or NOVA_EPI_F32_ARGMAX with X_lo.
 * ws: P * B * N floats (P * N <= 2^20) and tickets: N / 128 ints (zeroed, left zero) when the plan
 * cuts K into P > 1 chunks (nova_op_gemv_umma_splits).  max_ctas = SM budget of the partition (0 = whole GPU). */
int nova_op_gemv_umma(const void* X, const void* X_lo, int ldx, const void* W_blocked, int N, int K, void* Y, int ldy,
                      const void* bias, int B, int epi, float* ws, int32_t* tickets, uint64_t* keys, int max_ctas,
                      const float* norm_hid, float norm_eps, const void* ngamma, void* nxout, int ldnx,
                      void* stream);
/* norm_hid != NULL (epi NOVA_EPI_BF16_SILUMUL only): RMSNorm folded after the GEMV (DESIGN R25) -- X
 * holds x~ = bf16(h * gamma) and every output row b is scaled by rsqrt(mean_k h[b][k]^2 + norm_eps),
 * h = norm_hid [B][K] f32, before SiLU(gate) * up.
 * nxout != NULL (epi NOVA_EPI_F32_RESID only, ngamma [N] bf16 required): the other half of that fold --
 * after Y[b][n] += result, also nxout[b * ldnx + n] = bf16(Y[b][n] * ngamma[n]) (the next RMSNorm's
 * x~, read by the following NOVA_EPI_BF16_SILUMUL call).  NULL = off. */
int nova_op_gemv_umma_splits(int N, int K, int epi);
/* Decode qkv projection on the same tcgen05 GEMV (DESIGN R25 fold + the EPI_QKV_ROPE_KV epilogue of
 * nova_op_gemv_fused, SURVEY §8(a) a7 "QKV GEMV (+bias) + M-RoPE + KV append"): X = x~ = bf16(h * ln1)
 * [B][K] (ldx), h = norm_hid [B][K] f32; q/k/v = rsqrt(mean_k h^2 + norm_eps) * (x~ W^T) + bias, RoPE at
 * rows[b].pos on q and k; q heads -> Q [B][ldq] bf16 (first H * hd columns), k / v -> kv_pool at layer,
 * page bt[rows[b].slot][rows[b].ctx / 64], cell rows[b].ctx % 64.  hd must be 128 (one 128-row block
 * per head), N = (H + 2 KV) * hd, B <= 16; ws / tickets as nova_op_gemv_umma.  Bitwise independent of
 * max_ctas and of the batch composition. */
int nova_op_gemv_umma_qkv(const void* X, int ldx, const void* W_blocked, int N, int K, void* Q, int ldq,
                          const void* bias, int B, const float* norm_hid, float norm_eps, int H, int KV, int hd,
                          float theta, const nova_decode_row* rows, void* kv_pool, int layer, int n_pages,
                          const int32_t* bt, int max_pages, float* ws, int32_t* tickets, int max_ctas, void* stream);
/* y[r][c] = bf16(x[r][c] * gamma[c]) for M rows of d (the R25 fold's GEMV input). */
int nova_op_scale_rows_bf16(const float* x, int ldx, const void* gamma, void* y, int ldy, int M, int d, void* stream);

/* keys[r] (from NOVA_EPI_F32_ARGMAX) -> out_tok[r]; also last_tok[rows[r].slot] (rows != NULL)
 * or last_tok[single_slot] (>= 0); resets keys[r] to 0.  n <= 1024. */
int nova_op_argmax_finalize(uint64_t* keys, int n, int32_t* out_tok, const nova_decode_row* rows, int32_t* last_tok,
                            int single_slot, void* stream);

/* LayerNorm (ViT, mean/biased variance) and RMSNorm (LLM) of f32 rows [M][d].  RMSNorm y_f32:
 * 0 bf16 rows, 1 f32 rows, 2 bf16 hi rows at y then bf16 lo rows at y + M*ldy. */
int nova_op_layernorm(const float* x, int ldx, const void* gamma, const void* beta, void* y, int ldy, int M, int d,
                      float eps, void* stream);
int nova_op_rmsnorm(const float* x, int ldx, const void* gamma, void* y, int y_f32, int ldy, int M, int d, float eps,
                    void* stream);

/* Patchify (a1): pixels bf16 [C][H][W] -> X0 bf16 [N][C*T*P*P], merge-group-major rows. */
int nova_op_patchify(const void* pix, int C, int H, int W, int P, int T, int merge, void* X0, void* stream);

/* ViT 2D RoPE in place on q, k of qkv [N][3][heads][hd]; image grid gw patches wide. */
int nova_op_vit_rope(void* qkv, int N, int heads, int hd, int gw, int merge, float theta, void* stream);

/* LLM M-RoPE in place on q, k of nrows qkv rows, then K and V into the paged
 * cache.  Prefill: rows == NULL, positions pos3 int32 [3][ld_pos], cache index
 * ctx0 + r of request `slot`.  Decode: positions / cache index from rows[r]. */
int nova_op_llm_rope_kv(void* qkv, int ld, int nrows, int H, int KV, int hd, float theta, int sec0, int sec1,
                        const int32_t* pos3, int ld_pos, const nova_decode_row* rows, int slot, int ctx0,
                        void* kv_pool, int layer, int n_pages, const int32_t* block_tables, int max_pages,
                        void* stream);

/* Embedding gather into f32 rows: ids[r] (or last_tok[rows[r].slot] when ids == NULL). */
int nova_op_embed(const void* table, int d, const int32_t* ids, const nova_decode_row* rows, const int32_t* last_tok,
                  float* out, int ldo, int n, void* stream);

/* Greedy pick: argmax of each f32 row (ties -> lowest index) -> out_tok[r]; also
 * last_tok[rows[r].slot] (rows != NULL) or last_tok[single_slot] (>= 0). */
int nova_op_argmax(const float* logits, int ldl, int V, int n, int32_t* out_tok, const nova_decode_row* rows,
                   int32_t* last_tok, int single_slot, void* stream);

#ifdef __cplusplus
}
#endif
#endif
