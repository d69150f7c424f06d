// Nova engine internals: model/weight layout (L2 stage programs), partition
// executor (L3, green contexts + role workers), Algorithm 1 controller (L4) and the
// virtual-time Sim backend.  The public ABI is include/nova.h.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/nova.h"
#include "kernels.h"

namespace nova {

int64_t mono_ns();

// ------------------------------------------------------------------ model shape
struct Dims {
  nova_model_config m;
  int vit_hd, patch_dim, merge_dim, qkv_n, vit_layer_elems;
  int llm_qkv_n;  // (H + 2 KV) * hd
  void init(const nova_model_config& mc);
};

// Offsets (in bf16 elements) of the tensors of one ViT layer inside its block.
struct VitLayerLayout {
  size_t n1g, n1b, n2g, n2b, qkv_w, qkv_b, proj_w, proj_b, fc1_w, fc1_b, fc2_w, fc2_b, elems;
  void init(const Dims& d);
};

struct LlmLayerW {
  bf16 *ln1, *qkv_w, *qkv_b, *o_w, *ln2, *gu_w, *down_w;
  // decode copies in the streaming layout (blocked 64 x 64, SW128 pre-swizzled; block_weights)
  bf16 *qkv_wb, *o_wb, *gu_wb, *down_wb;
};

struct Weights {
  bf16* patch_w = nullptr;
  std::vector<bf16*> vit_dev;  // resident: L layer blocks; offload: K slot blocks
  bf16 *mlnq_g, *mlnq_b, *m1_w, *m1_b, *m2_w, *m2_b;
  bf16 *embed, *final_norm, *lm_head;
  bf16* lm_head_b = nullptr;  // lm_head in the streaming layout
  std::vector<LlmLayerW> llm;
};

// ------------------------------------------------------------------ requests
struct Request {
  uint64_t id = 0;
  int slot = -1;
  int gh = 0, gw = 0, n_prompt = 0, gen_len = 0;
  int64_t arrival = 0;
  int emitted = 0;
  int64_t join_seq = -1;
  float sim_vs = 1.f, sim_ps = 1.f;
  int pre_done = 0;                 // CHUNK: prefill tokens processed by finished hybrid passes
  int chunk_c0 = 0, chunk_n = 0;    // CHUNK: the chunk of the hybrid pass in flight
  std::vector<int> pages;
  std::vector<int> forced;          // teacher forcing
  std::vector<int> tokens;          // emitted tokens
  std::vector<std::vector<float>> logits;  // debug
  nova_req_stats st{};
  int n_v() const { return (gh / 2) * (gw / 2); }
  int S() const { return n_v() + n_prompt; }
};

// ------------------------------------------------------------------ Algorithm 1
struct Decision {
  int kind, ctx, s_dec;
  std::vector<Request*> reqs;
};
struct Event {
  int kind;      // NOVA_EV_*
  uint64_t key;  // request id (min id of a decode batch)
  std::vector<Request*> reqs;
  int64_t t;
  std::vector<int> tokens;  // tokens produced (prefill: 1, decode: one per request)
};

struct Alg1 {
  nova_partition_policy pol{};
  int total_sms = 148, granularity = 8, max_split = 112;
  std::deque<Request*> q_v, prefill_wait;
  Request* vision_running = nullptr;
  Request* prefill_running = nullptr;
  Request* chunk_req = nullptr;  // CHUNK: the request in chunked prefill (its chunks ride on LLM steps)
  std::vector<Request*> decode_running;
  bool decode_busy = false;
  std::vector<Request*> q_d;
  int64_t join_counter = 0;
  int last_pass = -1;  // 0 front, 1 decode
  // NOVA_MODE_FRONTIER: Pareto points and the recent arrival times (rate estimate)
  std::vector<nova_plan_point> frontier;
  int lam_window = 16;
  std::deque<int64_t> arr_t;
  double arrival_rate() const;  // req/s over the last lam_window arrivals (0 if < 2)
  int split(int ctx, int n_pend) const;
  int n_pend() const;
  bool front_running() const { return vision_running || prefill_running; }
  // Process one tick's events (already including finished detection); returns decisions.
  std::vector<Decision> tick(std::vector<Event>& evs);

 private:
  void emit(Request* r, std::vector<Decision>& out);
  void decode_ready(Request* r);
  void dispatch_front(std::vector<Decision>& out, bool corun, int npend, bool has_decode);
  void dispatch_decode(std::vector<Decision>& out, int ctx, int s);
  void dispatch_chunk(std::vector<Decision>& out);
};

// ------------------------------------------------------------------ partition family
struct Partition {
  int n_groups = 0, granularity = 8, total = 148;
  std::vector<cudaStream_t> dec_stream, front_stream;  // index k = decode groups (s = 8k)
  std::vector<CUgreenCtx> gctx;
  cudaStream_t solo_front = nullptr, solo_decode = nullptr;
  bool green = false;
  std::string init(int device, bool use_green);
  void destroy();
  int max_split() const { return (n_groups - 1) * granularity; }
};

// ------------------------------------------------------------------ live kernel timing
// Sampled CUDA-event brackets around the stage kernels (for the roofline report):
// per class the summed device time, the summed ALGORITHMIC work (bytes or FLOPs) and
// the launch count.  Classes are NOVA_K_* in nova.h.
struct KStat {
  double ms = 0, work = 0;
  int64_t launches = 0;
  double sm_ms = 0;  // sum of ms x (the pass's SM budget / total SMs): the partition-normalized time
};
struct KTimer {
  std::vector<cudaEvent_t> ev;
  struct Rec {
    int cls;
    double work;
    int i0;
  };
  std::vector<Rec> recs;
  int n = 0;
  bool on = false;
  double share = 1.0;  // SM budget of the current pass / total SMs
  void init(int pairs);
  void destroy();
  int begin(cudaStream_t s);
  void end(int i0, int cls, double work, cudaStream_t s);
  void harvest(KStat* out, std::mutex& mu);  // after the pass completed
};

// ------------------------------------------------------------------ GPU role worker
struct PassCmd {
  int kind;  // NOVA_DEC_VISION / PREFILL / DECODE
  int ctx, s_dec;
  std::vector<Request*> reqs;
  std::vector<int> forced_tok;  // per row, -1 = none
};

class Engine;

struct Worker {
  Engine* eng = nullptr;
  int role = 0;  // 0 front, 1 decode
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<PassCmd> q;
  bool stop = false;
  void start(Engine* e, int r);
  void push(PassCmd&& c);
  void run();
};

// ------------------------------------------------------------------ engine
class Engine {
 public:
  Dims dims;
  nova_engine_config cfg{};
  std::string err;             // guarded by err_mu (written by the role workers, submit, step)
  mutable std::mutex err_mu;
  std::atomic<bool> failed{false};
  bool finalized = false;
  bool sim = false;

  // memory
  nova_buffers buf{};
  Weights W;
  VitLayerLayout vl;
  int vit_K = 0;  // physical slots (0 = resident)
  // offload ring: physical slot holding each logical ViT layer (-1 = not resident).  Updated at
  // every swap-in, so the mapping stays right across passes when K does not divide L (Eq. 7
  // refills slot (l mod K) only in the first pass; afterwards the slots rotate).
  std::vector<int> vit_slot_of;
  uint16_t* host_vit = nullptr;  // pinned arena of all ViT layers (offload)
  cudaStream_t copy_stream = nullptr, upload_stream = nullptr;
  std::vector<cudaEvent_t> ev_loaded, ev_free;
  int n_slots_total = 0, max_pages_per_req = 0;
  // device per-slot state
  bf16* d_pix = nullptr;
  int* d_prompt = nullptr;
  int* d_bt = nullptr;
  int* d_last = nullptr;
  size_t pix_stride = 0;
  std::vector<cudaEvent_t> ev_upload;
  // workspaces
  struct FrontWS {
    bf16 *x0, *xb, *qkv, *attn, *act;
    float *hid, *vhid, *xf, *logits;
    float* nss;     // prefill RMSNorm fold (R25): [S][D / 32] partial sums of squares
    float* rscale;  // ... and the row scales [S]
    float2* rope_tab;  // ViT 2D RoPE (cos, sin) table [max grid side][20] for the fused qkv epilogue
    int *pos3, *tok;
    unsigned long long* keys;  // greedy argmax (EPI_F32_ARGMAX), zero between passes
    int* h_pos3;  // pinned
    int* h_tok;   // pinned
    float* h_logits;
  } fw{};
  struct DecWS {
    float *hid, *xf, *logits, *attn_ws, *gemv_ws;
    float *qkvf, *ss;           // fused decode: f32 raw qkv rows, per-64-column sums of squares
    bf16* xlo;                  // fused decode: lo tile of the f32 lm_head input
    unsigned long long* bar;    // fused decode: grid-barrier counter (monotone; see dec_bar_base)
    int* tickets;               // [0, 4096): gemv_tma row blocks; [4096, 8192): decode attention
    unsigned long long* keys;  // greedy argmax, zero between passes
    bf16 *xb, *qkv, *attn, *act;
    DecodeRow* rows;
    int* tok;
    DecodeRow* h_rows;
    int* h_tok;
    int* h_forced;
    float* h_logits;
  } dw{};
  struct HybWS {  // CHUNK mode: hybrid iterations (prefill chunk rows, then decode rows)
    float *pre, *hid, *xf, *logits;   // pre: the chunked request's input rows [S_max][D] (E_vis | prompt embeds)
    bf16 *xb, *qkv, *attn, *act;
    DecodeRow *rows, *lm_rows;        // per hybrid row (attention / RoPE) and per lm_head row
    int *pos3, *tok;
    unsigned long long* keys;
    DecodeRow *h_rows, *h_lm_rows;    // pinned
    int *h_pos3, *h_tok, *h_forced;   // pinned
    float* h_logits;                  // pinned [17][V]
  } hw{};
  Partition part;
  DecFusedState* dfs = nullptr;     // fused decode kernel state (null: per-op decode path)
  unsigned long long dec_bar_base = 0;  // grid-barrier counter value at the next fused launch
  Worker front_w, dec_w;
  KTimer ktimer[2];                  // per role (0 front, 1 decode)
  KStat kstats[NOVA_K_COUNT];
  std::mutex kmu;
  int64_t pass_count[2] = {0, 0};
  // §8(f) f4: front passes repartitioned every regroup_layers layers (0 = per pass) toward
  // front_hint = the decode split the policy gives now for the front's context (0 = no decode work:
  // all SMs to the front; -1 = none), published by step()
  std::atomic<int> regroup_layers{0};
  std::atomic<int> front_hint{-1};
  std::atomic<long long> front_switches{0};
  cudaEvent_t regroup_ev = nullptr;
  int sample_every = 0;              // 0 = kernel timing off; n = time every n-th pass of a role
  double pass_work[2] = {0, 0};      // algorithmic work of the last pass issued by each role

  // controller
  std::mutex ctl_mu;
  Alg1 alg;
  std::deque<Request*> inbox;
  std::mutex inbox_mu;
  std::condition_variable wake;
  std::mutex wake_mu;
  std::deque<Event> completions;  // from workers
  std::map<uint64_t, std::unique_ptr<Request>> reqs;
  uint64_t next_id = 1;
  std::vector<int> free_slots, free_pages;
  std::deque<nova_token> tok_q;
  std::mutex tok_mu;
  std::deque<nova_log_record> log;  // bounded ring (NOVA_LOG_CAPACITY); log[i] is record log_base + i
  int64_t log_base = 0;
  std::deque<uint64_t> finished_ids;  // release order for cfg.finished_retention
  int tick_no = 0;
  int finished = 0;
  nova_step_info last_info{};

  // sim backend
  nova_sim_curves sc{};
  std::vector<int32_t> sc_s;
  std::vector<int64_t> sc_tv, sc_tp, sc_tdv, sc_tdp;
  int64_t sim_now = 0;
  struct SimPending {
    int64_t t;
    Event ev;
  };
  std::vector<SimPending> sim_pending;

  // lifecycle
  nova_status create(const nova_model_config* m, const nova_engine_config* c, const nova_buffers* b);
  nova_status load_tensor(const char* name, const void* src, uint64_t nbytes, int on_dev);
  nova_status finalize();
  void shutdown();
  ~Engine() { shutdown(); }
  nova_status fail(nova_status s, const std::string& m) {
    {
      std::lock_guard<std::mutex> g(err_mu);
      err = m;
    }
    if (s == NOVA_E_CUDA) failed.store(true);
    return s;
  }
  std::string last_error() const {
    std::lock_guard<std::mutex> g(err_mu);
    return err;
  }

  // memory plans
  static size_t plan_weights(const Dims& d, const nova_engine_config& c, Weights* w, VitLayerLayout* vl, uint8_t* base);
  static size_t plan_workspace(const Dims& d, const nova_engine_config& c, Engine* e, uint8_t* base);
  static size_t plan_kv(const Dims& d, const nova_engine_config& c);

  // requests / ticks
  nova_status submit(const nova_request* r, uint64_t* id);
  nova_status step(int64_t max_wait_us, nova_step_info* out);
  void dispatch(const Decision& d);
  void post_completion(Event&& e);
  void finish_request(Request* r);
  void log_event(const Event& e);
  void log_push(const nova_log_record& r);
  void log_decision(const Decision& d, int64_t t);

  // stage programs (model.cpp); return cudaError
  int front_sms(int s_dec) const { return s_dec <= 0 ? part.total : part.total - s_dec; }
  struct FrontRG {  // live repartition of one front pass (f4)
    int s_dec;       // decode split the pass's partition leaves out (0 = all SMs)
    int group;       // layers per group
  };
  // every stage program may move `s` / `sms` to another front partition when rg != null
  cudaError_t run_encode(Request* r, cudaStream_t& s, int sms, FrontRG* rg = nullptr);
  cudaError_t run_prefill(Request* r, cudaStream_t& s, int sms, FrontRG* rg = nullptr);
  cudaError_t front_regroup(FrontRG* rg, cudaStream_t& s, int& sms);
  // decode SMs of a pass: the whole GPU when SOLO, else the partition's s_dec
  int dec_sms(int ctx, int s_dec) const { return (ctx == NOVA_CTX_SOLO || s_dec <= 0 || s_dec >= part.total) ? part.total : s_dec; }
  cudaError_t run_decode(const std::vector<Request*>& rows, const std::vector<int>& forced, cudaStream_t s, int sms);
  // CHUNK mode: one hybrid iteration -- reqs[0]'s chunk [chunk_c0, chunk_c0 + chunk_n) of prefill rows
  // and reqs[1..] as decode rows in one batch; writes hw.h_tok (prefill token first if last chunk)
  cudaError_t run_hybrid(const std::vector<Request*>& reqs, const std::vector<int>& forced, cudaStream_t s, int sms);
  cudaStream_t stream_for(int role, int ctx, int s_dec);
  int s_max_of_public() const;
  // 128-key chunk capacity of dw.attn_ws per (request, KV head) (decode_attn_p, fused decode)
  int attn_mch() const { return (s_max_of_public() + cfg.max_gen + 1 + 127) / 128; }
  nova_status time_pass(int stage, int s, int gh, int gw, int n_prompt, int B, int ctx, int corun, int iters,
                        double* out);
};

}  // namespace nova
