/* nova.h -- C ABI of the Nova co-execution engine (libnova.so).
 *
 * What it does: serves agentic-VLM requests (a screenshot + an instruction,
 * PAPER.md §II-C) through three stages -- vision encode, LLM prefill,
 * LLM greedy decode (§II-A) -- that co-execute on disjoint SM
 * partitions of one B200 (§III-B).  A request scheduler implements
 * Algorithm 1; the decode share of the SMs follows Eq. 5
 * with SM_op from the Eq. 1-3 planner; ViT weights may
 * be offloaded layer-wise with the Eq. 7 swap-in ring (§III-E).
 * The paper's libsmctrl stream masks are replaced by CUDA green
 * contexts: one family of partitions built at nova_finalize, selected per
 * forward pass, never rebuilt.
 *
 * Conventions
 *   - Every call returns nova_status (0 = NOVA_OK, negative = error); no C++
 *     exception crosses the ABI.  nova_last_error(e) returns an engine-owned,
 *     NUL-terminated message for the last failure on that engine (NULL engine:
 *     the last creation error).
 *   - Ownership: the caller owns every pointer it passes.  Inputs are copied
 *     (or H2D-enqueued from the caller's memory) before the call returns.
 *     Device buffers in nova_buffers are allocated by the caller (e.g. torch)
 *     and BORROWED until nova_destroy; they must stay alive and untouched.
 *   - Threading: nova_submit may be called from any thread.  All other calls
 *     on one engine must come from a single driver thread.
 *   - After a CUDA error the engine latches FAILED: later calls return
 *     NOVA_E_STATE.  Sizes/shapes outside the configured maxima -> NOVA_E_INVAL.
 *   - Times are int64 nanoseconds of CLOCK_MONOTONIC (GPU backend) or of the
 *     virtual clock (Sim backend).
 */
#ifndef NOVA_H
#define NOVA_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct nova_engine nova_engine;
typedef int32_t nova_status;
enum {
  NOVA_OK = 0,
  NOVA_E_INVAL = -1,     /* bad argument / shape outside configured maxima        */
  NOVA_E_NOMEM = -2,     /* buffers too small / host allocation failed            */
  NOVA_E_CUDA = -3,      /* CUDA runtime or driver error (engine latches FAILED)   */
  NOVA_E_AGAIN = -4,     /* no free request slot: retry after requests finish     */
  NOVA_E_NOTFOUND = -5,  /* unknown request id / tensor name                       */
  NOVA_E_PARTITION = -6, /* SM budget not realisable at the partition granularity  */
  NOVA_E_STATE = -7      /* engine FAILED, or call out of order                    */
};

/* Model shape (Qwen2-VL family; SURVEY.md §8 shape legend). */
typedef struct {
  int32_t vit_depth, vit_dim, vit_heads, vit_mlp, patch, temporal_patch, merge, in_ch;
  int32_t llm_layers, llm_dim, llm_heads, llm_kv_heads, head_dim, llm_ffn, vocab, tie_embed;
  int32_t mrope_section[3];
  float vit_theta, llm_theta, ln_eps, rms_eps;
} nova_model_config;

enum { NOVA_BACKEND_GPU = 0, NOVA_BACKEND_SIM = 1 };

typedef struct {
  int32_t backend;              /* NOVA_BACKEND_GPU or NOVA_BACKEND_SIM (virtual time, no GPU)  */
  int32_t device;               /* CUDA device ordinal                                         */
  int32_t max_requests;         /* concurrent requests (slots)                                 */
  int32_t max_decode_batch;     /* B_max <= 16                                                 */
  int32_t kv_pages;             /* KV pool size in 64-token pages                              */
  int32_t max_patches;          /* max ViT patches per image (N)                               */
  int32_t max_prompt;           /* max prompt tokens                                           */
  int32_t max_gen;              /* max generated tokens per request (gen_len)                  */
  int32_t vit_resident_layers;  /* K physical ViT layer slots (Eq. 7); 0 = all layers resident */
  int32_t use_green_ctx;        /* 1: SM partitions via green contexts (nova_finalize fails with
                                   NOVA_E_CUDA if the driver cannot split the SMs); 0: primary
                                   context only (every split runs on all SMs)                    */
  int32_t debug_keep_logits;    /* keep every step's f32 logits for nova_debug_logits          */
  int32_t finished_retention;   /* finished requests kept for nova_request_stats / debug_logits;
                                   older ones are released oldest-first (0 = 4096, < 0 = all)   */
} nova_engine_config;

/* Device buffer sizes the caller must provide (GPU backend); pinned_host_bytes is
 * allocated by the engine itself (offload arena). */
nova_status nova_query_memory(const nova_model_config* m, const nova_engine_config* c, uint64_t* weights_bytes,
                              uint64_t* kv_bytes, uint64_t* workspace_bytes, uint64_t* pinned_host_bytes);

typedef struct {
  void* weights_dev;   uint64_t weights_bytes;    /* engine weight layout (filled by nova_load_tensor) */
  void* kv_dev;        uint64_t kv_bytes;         /* paged KV pool                                      */
  void* workspace_dev; uint64_t workspace_bytes;  /* activations of the three roles                      */
} nova_buffers;

/* Create an engine.  GPU backend: buffers required; Sim backend: buffers may be NULL. */
nova_status nova_create(const nova_model_config* m, const nova_engine_config* c, const nova_buffers* b,
                        nova_engine** out);
/* Place one weight tensor, given by its HF Qwen2-VL state_dict name, as bf16 bits
 * (row-major [out][in]); src is host (src_on_device = 0) or device memory.  q/k/v
 * are fused and gate/up interleaved by the engine (layout only, no arithmetic). */
nova_status nova_load_tensor(nova_engine* e, const char* name, const void* src, uint64_t nbytes,
                             int32_t src_on_device);
/* After all tensors: preload the K offload slots, build the partition family,
 * start the role workers.  The engine is then ready for nova_submit. */
nova_status nova_finalize(nova_engine* e);
nova_status nova_destroy(nova_engine* e);
const char* nova_last_error(nova_engine* e);

/* SMs of the device, partition granularity (8 on sm_100 green contexts), and the
 * number of decode splits s in {g, 2g, ..., (n_groups-1) g}. */
nova_status nova_query_sms(nova_engine* e, int32_t* total_sms, int32_t* granularity, int32_t* n_splits);

/* ------------------------------------------------------------------ requests */
typedef struct {
  const uint16_t* pixels_bf16; /* [3][height][width] bf16 bits, host or device memory (UVA)    */
  int32_t height, width;       /* multiples of patch * merge (28)                               */
  const int32_t* prompt_ids;   /* host [n_prompt], each < vocab                                 */
  int32_t n_prompt;
  int32_t gen_len;             /* >= 1 tokens to emit, counting the prefill token (no EOS)      */
  int64_t arrival_ns;          /* 0 = now (GPU); virtual arrival time (Sim)                     */
  uint64_t user_tag;
  /* Sim backend only: duration scale factors for this request's front passes */
  float sim_vision_scale, sim_prefill_scale;
} nova_request;
/* Thread-safe.  Copies the prompt, enqueues the pixel H2D copy; returns the id. */
nova_status nova_submit(nova_engine* e, const nova_request* r, uint64_t* req_id);

/* ------------------------------------------------------------------ partition policy */
/* SERIAL: Serial-RR, one pass at a time on all SMs, alternating decode / front (BASELINE).
 * STATIC: co-run, fixed decode SMs per context.  ADAPTIVE: co-run, Eq. 5 (Nova).
 * PF_LIMIT: the paper's prefill-first baseline: one pass at a time on all SMs, the
 *   front stage first; a decode iteration runs when more than pf_threshold requests wait for
 *   decode, or when no front work is ready.
 * MULTI_STREAM: the paper's multi-stream baseline: front and decode co-run on two
 *   streams that both see every SM (no partition; the hardware arbitrates).
 * FRONTIER: SURVEY.md §8(f) f3, the frontier-lookup controller: instead of Eq. 5's linear
 *   rule, each co-run pass takes the Pareto point (nova_set_frontier) with the lowest Eq. 1
 *   E2E among those whose Eq. 4 throughput covers the estimated arrival rate (the last
 *   `window` arrivals); if none does, the highest-throughput point (P:356 -- the frontier is
 *   the paper's justification for Eq. 5).
 * CHUNK: the paper's chunked-prefill baseline "Chunk" (Sarathi-style hybrid batching,
 *   token budget chunk_budget, the paper's best 128): one pass at a time on all SMs; an LLM step
 *   is a HYBRID iteration = the next min(remaining, chunk_budget - B) prefill tokens of the
 *   request in chunked prefill + the current decode batch (B requests) in one batch; vision
 *   encode cannot join the batch (separate weights) and runs as its own pass, alternating
 *   with LLM steps (R26).  The prefill token (index 0) is emitted by the last chunk. */
enum { NOVA_MODE_SERIAL = 0, NOVA_MODE_STATIC = 1, NOVA_MODE_ADAPTIVE = 2, NOVA_MODE_PF_LIMIT = 3,
       NOVA_MODE_MULTI_STREAM = 4, NOVA_MODE_FRONTIER = 5, NOVA_MODE_CHUNK = 6 };
#define NOVA_CHUNK_MAX 256  /* largest chunk_budget (hybrid workspace rows = NOVA_CHUNK_MAX + 16) */
enum { NOVA_CTX_DV = 0, NOVA_CTX_DP = 1, NOVA_CTX_SOLO = 2 };
typedef struct {
  int32_t mode;                        /* NOVA_MODE_*                                           */
  int32_t sm_decode_dv, sm_decode_dp;  /* STATIC: decode SMs while co-running with vision/prefill */
  int32_t sm_op_dv, sm_op_dp, sm_min;  /* ADAPTIVE (Eq. 5)                                       */
  float alpha_dv, alpha_dp;
  int32_t b_max;                       /* decode batch cap (<= max_decode_batch)                 */
  int32_t pf_threshold;                /* PF_LIMIT: decode when > pf_threshold wait (<= 0: 5)     */
  int32_t sm_dv_floor;                 /* ADAPTIVE / FRONTIER: decode SMs never below this while
                                          co-running with vision (offload-aware, see
                                          nova_offload_floor); 0 = none                       */
  int32_t chunk_budget;                /* CHUNK: tokens per hybrid iteration (<= 0: 128;
                                          <= NOVA_CHUNK_MAX)                                  */
  int32_t front_regroup;               /* STATIC / ADAPTIVE / FRONTIER: every
                                          front_regroup layers a running vision / prefill pass
                                          re-reads the split Eq. 5 (or the static / frontier rule)
                                          gives now and moves to that split's front partition
                                          (all SMs once no decode work is left); 0 = the paper's
                                          per-pass granularity                        */
} nova_partition_policy;
/* Takes effect at each role's next forward pass.  `applied` (may be NULL)
 * receives the values rounded down to the granularity.  NOVA_E_PARTITION if a
 * budget rounds to 0 or leaves the front stage no SM group. */
nova_status nova_set_partition(nova_engine* e, const nova_partition_policy* p, nova_partition_policy* applied);

/* ------------------------------------------------------------------ scheduler tick */
typedef struct {
  int32_t events;        /* completions + arrivals processed in this tick   */
  int32_t dispatched;    /* passes launched in this tick                    */
  int32_t n_pending;     /* N_pend (vision/prefill queued or running)       */
  int32_t sm_decode;     /* decode SMs of the last decode dispatch          */
  int32_t context;       /* NOVA_CTX_* of the last decode dispatch          */
  int32_t decode_batch;  /* size of the last decode batch                   */
  int32_t active;        /* requests admitted and not finished              */
  int32_t finished;      /* requests finished so far                        */
  int64_t now_ns;        /* tick time                                        */
} nova_step_info;
/* One Algorithm 1 iteration: process completed passes and arrivals, recount
 * N_pend, apply Eq. 5, dispatch.  Blocks up to max_wait_us for an event when
 * there is none (GPU); the Sim backend advances virtual time to the next event. */
nova_status nova_step(nova_engine* e, int64_t max_wait_us, nova_step_info* out);

enum { NOVA_TOK_FIRST = 1, NOVA_TOK_LAST = 2 };
typedef struct {
  uint64_t req_id;
  int32_t index;     /* 0 = the prefill token */
  int32_t token;
  int64_t t_emit_ns; /* time the host observed the token */
  int32_t flags;     /* NOVA_TOK_FIRST | NOVA_TOK_LAST   */
  int32_t pad;
} nova_token;
/* Drain up to cap emitted tokens (FIFO). */
nova_status nova_poll_tokens(nova_engine* e, nova_token* buf, int32_t cap, int32_t* n_out);

typedef struct {
  int64_t arrival, vis_start, vis_end, pre_start, pre_end, first_tok, last_tok;
  int32_t split_at_vis, split_at_pre; /* decode SMs at the front dispatch (0 = front alone) */
  int32_t n_tokens, finished;
} nova_req_stats;
nova_status nova_request_stats(nova_engine* e, uint64_t req_id, nova_req_stats* out);
/* Release a FINISHED request's record (stats, tokens, debug logits) now instead of at the
 * finished_retention bound.  NOVA_E_NOTFOUND if unknown, NOVA_E_STATE if not finished. */
nova_status nova_release_request(nova_engine* e, uint64_t req_id);

/* Decision log of Algorithm 1 (for replay against the oracle). */
/* NOVA_DEC_HYBRID (CHUNK mode): ids[0] = the request in chunked prefill, ids[1..] = the decode
 * batch; s_dec = the chunk's prefill token count (the pass itself runs on all SMs). */
enum { NOVA_DEC_VISION = 0, NOVA_DEC_PREFILL = 1, NOVA_DEC_DECODE = 2, NOVA_DEC_FINISH = 3, NOVA_DEC_HYBRID = 4 };
enum { NOVA_EV_VISION_DONE = 0, NOVA_EV_PREFILL_DONE = 1, NOVA_EV_DECODE_DONE = 2, NOVA_EV_ARRIVAL = 3,
       NOVA_EV_HYBRID_DONE = 4 };
typedef struct {
  int64_t t_ns;
  int32_t tick;      /* tick sequence number                                     */
  int32_t is_event;  /* 1: an input event of the tick, 0: a decision              */
  int32_t kind;      /* NOVA_EV_* or NOVA_DEC_*                                  */
  int32_t ctx;       /* decisions: NOVA_CTX_*                                     */
  int32_t s_dec;     /* decisions: decode SMs (0 = front alone)                   */
  int32_t n_ids;
  uint64_t ids[16];  /* request ids (batch for decode)                            */
} nova_log_record;
/* The log is a bounded ring of NOVA_LOG_CAPACITY records: record indices are absolute (0 = the
 * first record ever written); records below nova_decision_log_base() have been dropped.
 * Copy log records [start, start + cap) ; n_out = records copied; total = all records ever
 * written.  NOVA_E_NOTFOUND if start < nova_decision_log_base(). */
#define NOVA_LOG_CAPACITY (1 << 18)
nova_status nova_decision_log(nova_engine* e, int64_t start, nova_log_record* buf, int32_t cap, int32_t* n_out,
                              int64_t* total);
/* Index of the oldest retained log record (0 until the ring first wraps); -1 for a NULL engine. */
int64_t nova_decision_log_base(nova_engine* e);

/* ------------------------------------------------------------------ debug / parity */
/* f32 logits of token `index` of a request (needs debug_keep_logits). */
nova_status nova_debug_logits(nova_engine* e, uint64_t req_id, int32_t index, float* out, int32_t vocab);
/* Teacher forcing: decode step k (k >= 1) consumes tokens[k-1] instead of the argmax
 * of step k-1.  Must be called right after nova_submit. */
nova_status nova_debug_force_tokens(nova_engine* e, uint64_t req_id, const int32_t* tokens, int32_t n);

/* Front passes moved to another partition at a layer-group boundary so far (front_regroup, f4);
 * -1 for a NULL engine. */
int64_t nova_front_switches(nova_engine* e);

/* Copy an internal decode workspace buffer to host memory (parity debugging; synchronizes the
 * device).  name: "dec_hid" (f32 [max_decode_batch][llm_dim]), "dec_xg" / "dec_xlo" (bf16
 * [max_decode_batch][llm_dim]), "dec_qkvf" (f32 [max_decode_batch][(H + 2 KV) hd]), "dec_attn"
 * (bf16 [max_decode_batch][H hd]), "dec_act" (bf16 [max_decode_batch][ffn]), "dec_ss" (f32
 * [max_decode_batch][ceil4(llm_dim / 64)]); layer-0 weights "w_o0" (o_proj, [out][in]), "w_ob0" /
 * "w_qkvb0" (o / qkv in the decode streaming layout); "dec_dbg" (fused-decode phase timeline, u64).  bytes <= the buffer size, else NOVA_E_INVAL;
 * unknown name -> NOVA_E_NOTFOUND.  Works on a FAILED engine (post-mortem). */
nova_status nova_debug_read_buffer(nova_engine* e, const char* name, void* out, uint64_t bytes);

/* ------------------------------------------------------------------ live kernel timing */
/* Kernel classes with their ALGORITHMIC work unit (what the method must move or
 * compute, no padding):                                        */
enum {
  NOVA_K_DEC_GEMV = 0,   /* decode linears: bytes = N*K*2 (weights) + B*K*sx + B*N*sy       */
  NOVA_K_VIT_GEMM = 1,   /* ViT + merger linears: flops = 2*M*N*K                           */
  NOVA_K_LLM_GEMM = 2,   /* prefill linears: flops = 2*M*N*K                                */
  NOVA_K_VIT_ATTN = 3,   /* ViT attention: flops = 4*N^2*hd*heads                           */
  NOVA_K_PRE_ATTN = 4,   /* prefill causal attention: flops = 2*S^2*hd*heads (causal half)  */
  NOVA_K_DEC_ATTN = 5,   /* decode attention: bytes = sum_b (ctx_b+1)*2*KV*hd*2             */
  NOVA_K_LM_HEAD = 6,    /* lm_head GEMV: bytes = V*D*2                                     */
  NOVA_K_VIT_PASS = 7,   /* whole vision pass: flops (SURVEY §8(d) d2 a5 formula)           */
  NOVA_K_PRE_PASS = 8,   /* whole prefill pass: flops (a6 formula)                          */
  NOVA_K_DEC_PASS = 9,   /* whole decode iteration: bytes = weights + KV read (a7 formula)  */
  NOVA_K_DEC_FUSED = 10, /* fused decode-iteration kernel (one launch): bytes = a7 formula    */
  NOVA_K_COUNT = 11
};
/* every_n = 0 disables; n >= 1 brackets the kernels of every n-th pass of each role
 * with CUDA events on the stream they are launched on (whole passes: every pass). */
nova_status nova_kernel_timing(nova_engine* e, int32_t every_n);
/* out[0] = summed device ms, out[1] = summed algorithmic work, out[2] = launches. */
nova_status nova_kernel_stats(nova_engine* e, int32_t cls, double* out3);
/* *sm_ms = sum over the same launches of ms x (SM budget of the launching pass / total SMs): the time a
 * stage running on a partition would take on the whole GPU at the same per-SM rate, so work / sm_ms is the
 * partition-normalized rate (SURVEY.md §8(d) d2 "Partition-normalized: the same / (s / 148)"). */
nova_status nova_kernel_stats_sm(nova_engine* e, int32_t cls, double* sm_ms);
nova_status nova_kernel_stats_reset(nova_engine* e);
/* Total libnova kernel launches in this process so far (all engines and nova_op_*). */
uint64_t nova_launch_count(void);

/* ------------------------------------------------------------------ curves + planner */
/* Time one forward pass with the SM split s (decode SMs; front gets the rest,
 * s = 0: solo on all SMs).  stage 0 = vision (grid gh x gw), 1 = prefill
 * (S = n_v + n_prompt), 2 = decode iteration (batch B at context ctx).  With
 * corun = 1 the front stage runs while decode iterations (batch B) loop on the
 * complementary partition; out_ms[0] = front pass, out_ms[1] = mean decode
 * iteration.  Uses internal profiling slots; do not call while serving. */
nova_status nova_time_pass(nova_engine* e, int32_t stage, int32_t s, int32_t gh, int32_t gw, int32_t n_prompt,
                           int32_t B, int32_t ctx, int32_t corun, int32_t iters, double* out_ms);

typedef struct {
  int32_t n;             /* number of splits                                   */
  const int32_t* s;      /* decode SMs per split (ascending)                   */
  const double* t_v;     /* ms, vision pass on the front partition (total - s) */
  const double* t_p;     /* ms, prefill pass on the front partition            */
  const double* t_d_dv;  /* ms, decode iteration on s SMs co-running vision    */
  const double* t_d_dp;  /* ms, decode iteration on s SMs co-running prefill   */
  double t_d_full;       /* ms, decode iteration alone on all SMs              */
} nova_curves;
typedef struct {
  int32_t s_v, s_p;      /* P_v, P_p: decode SMs in the two co-run contexts     */
  double e2e_ms;         /* Eq. 1                                               */
  double thr_rps;        /* Eq. 4                                               */
  int32_t on_frontier;   /* Pareto frontier membership                          */
  int32_t pad;
} nova_plan_point;
/* Eqs. 1-4 over all split pairs, Pareto frontier, Eq. 3 argmin (ties -> more decode
 * SMs), SM_min (smallest s with co-run decode <= tau * t_d_full) and
 * alpha = (SM_op - SM_min) / 3 (R9-R12).  Pure host function. */
nova_status nova_plan(const nova_curves* c, double gen_len, double tau, nova_plan_point* pts, int32_t cap,
                      int32_t* n_out, nova_plan_point* best, int32_t* sm_min_out, double* alpha_dv_out,
                      double* alpha_dp_out);
/* Frontier points for NOVA_MODE_FRONTIER (copied; points with on_frontier == 0 are ignored;
 * s_v / s_p must be realisable splits).  window >= 2: arrivals in the rate estimate
 * lambda = (window - 1) / (t_last - t_first).  Set before selecting the mode. */
nova_status nova_set_frontier(nova_engine* e, const nova_plan_point* pts, int32_t n, int32_t window);
/* Offload-aware split (Eq. 8): with layer-wise ViT
 * offload a vision pass cannot finish before its weights stream in (t_h2d_ms), so front SMs
 * beyond those that meet t_h2d are idle.  Returns the largest decode split s[i] whose co-run
 * vision time t_v[i] is within 2% of max(t_h2d_ms, min_i t_v[i]) -- those SMs cost the vision
 * pass nothing -- or 0 if n == 0.  s ascending, t_v[i] the vision pass with decode on s[i] SMs
 * (measured with the offload ring active, so t_v already includes any PCIe stall). */
int32_t nova_offload_floor(const int32_t* s, const double* t_v, int32_t n, double t_h2d_ms);
/* Eq. 5: max(SM_min, floor_g(SM_op - alpha (max(N_pend, 1) - 1))). */
int32_t nova_adaptive_sm(int32_t sm_op, int32_t sm_min, double alpha, int32_t n_pending, int32_t granularity);
/* Eq. 7 and Eq. 8 (offload ring). */
int32_t nova_next_logical_layer(int32_t cur, int32_t K, int32_t L);
double nova_required_bandwidth(double bytes, double forward_s, int32_t L, int32_t K);

/* Sim backend: per-split durations (ns) the virtual executor uses; same layout as
 * nova_curves (t_v/t_p indexed by decode split, *_solo on all SMs). beta: decode
 * time grows by (1 + beta (B - 1)). */
typedef struct {
  int32_t n;
  const int32_t* s;
  const int64_t *t_v, *t_p, *t_d_dv, *t_d_dp;
  int64_t t_v_solo, t_p_solo, t_d_solo;
  double beta;
  int32_t total_sms, granularity;
} nova_sim_curves;
nova_status nova_sim_set_curves(nova_engine* e, const nova_sim_curves* c);

#ifdef __cplusplus
}
#endif
#endif
