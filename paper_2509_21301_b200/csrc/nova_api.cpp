// L5: the C ABI of include/nova.h -- argument checking and marshalling only; no
// exception or C++ type crosses the boundary.
#include <algorithm>
#include <cstring>
#include <new>

#include "engine.h"

using namespace nova;

struct nova_engine {
  Engine e;
};

static thread_local std::string g_create_err;

#define GUARD(body)                                     \
  try {                                                 \
    body                                                \
  } catch (const std::bad_alloc&) {                     \
    return NOVA_E_NOMEM;                                \
  } catch (...) {                                       \
    return NOVA_E_STATE;                                \
  }

extern "C" {

nova_status nova_query_memory(const nova_model_config* m, const nova_engine_config* c, uint64_t* wb, uint64_t* kb,
                              uint64_t* ws, uint64_t* ph) {
  if (!m || !c) return NOVA_E_INVAL;
  GUARD({
    Dims d;
    d.init(*m);
    if (wb) *wb = Engine::plan_weights(d, *c, nullptr, nullptr, nullptr);
    if (kb) *kb = Engine::plan_kv(d, *c);
    if (ws) *ws = Engine::plan_workspace(d, *c, nullptr, nullptr);
    if (ph) {
      VitLayerLayout vl;
      vl.init(d);
      const bool off = c->vit_resident_layers > 0 && c->vit_resident_layers < m->vit_depth;
      *ph = off ? (uint64_t)m->vit_depth * vl.elems * 2 : 0;
    }
    return NOVA_OK;
  })
}

nova_status nova_create(const nova_model_config* m, const nova_engine_config* c, const nova_buffers* b,
                        nova_engine** out) {
  if (!m || !c || !out) return NOVA_E_INVAL;
  GUARD({
    nova_engine* e = new nova_engine();
    nova_status s = e->e.create(m, c, b);
    if (s != NOVA_OK) {
      g_create_err = e->e.last_error();
      delete e;
      *out = nullptr;
      return s;
    }
    *out = e;
    return NOVA_OK;
  })
}

nova_status nova_load_tensor(nova_engine* e, const char* name, const void* src, uint64_t nbytes, int32_t on_dev) {
  if (!e || !name || !src) return NOVA_E_INVAL;
  if (e->e.finalized) return e->e.fail(NOVA_E_STATE, "load_tensor after finalize");
  GUARD({ return e->e.load_tensor(name, src, nbytes, on_dev); })
}

nova_status nova_finalize(nova_engine* e) {
  if (!e) return NOVA_E_INVAL;
  GUARD({ return e->e.finalize(); })
}

nova_status nova_destroy(nova_engine* e) {
  if (!e) return NOVA_E_INVAL;
  GUARD({
    delete e;
    return NOVA_OK;
  })
}

// A thread-local copy: the engine's message may be rewritten by its worker threads at any time.
const char* nova_last_error(nova_engine* e) {
  static thread_local std::string msg;
  msg = e ? e->e.last_error() : g_create_err;
  return msg.c_str();
}

nova_status nova_query_sms(nova_engine* e, int32_t* total, int32_t* gran, int32_t* n_splits) {
  if (!e) return NOVA_E_INVAL;
  Engine& E = e->e;
  const bool live = !E.sim && E.finalized;
  if (total) *total = live ? E.part.total : E.alg.total_sms;
  if (gran) *gran = live ? E.part.granularity : E.alg.granularity;
  if (n_splits) *n_splits = live ? E.part.n_groups - 1 : E.alg.max_split / std::max(1, E.alg.granularity);
  return NOVA_OK;
}

nova_status nova_submit(nova_engine* e, const nova_request* r, uint64_t* id) {
  if (!e || !r || !id) return NOVA_E_INVAL;
  GUARD({ return e->e.submit(r, id); })
}

nova_status nova_set_frontier(nova_engine* e, const nova_plan_point* pts, int32_t n, int32_t window) {
  if (!e || (!pts && n > 0) || n < 0 || window < 2) return NOVA_E_INVAL;
  Engine& E = e->e;
  const int g = E.alg.granularity, mx = E.alg.max_split;
  std::vector<nova_plan_point> f;
  for (int i = 0; i < n; ++i) {
    if (!pts[i].on_frontier) continue;
    if (pts[i].s_v < g || pts[i].s_p < g || pts[i].s_v > mx || pts[i].s_p > mx || pts[i].s_v % g || pts[i].s_p % g)
      return E.fail(NOVA_E_PARTITION, "frontier split not realisable");
    f.push_back(pts[i]);
  }
  if (f.empty()) return E.fail(NOVA_E_INVAL, "no frontier point");
  E.alg.frontier = f;
  E.alg.lam_window = window;
  return NOVA_OK;
}

nova_status nova_set_partition(nova_engine* e, const nova_partition_policy* p, nova_partition_policy* applied) {
  if (!e || !p) return NOVA_E_INVAL;
  Engine& E = e->e;
  if (p->mode < NOVA_MODE_SERIAL || p->mode > NOVA_MODE_CHUNK) return E.fail(NOVA_E_INVAL, "mode");
  if (p->mode != NOVA_MODE_CHUNK && E.alg.chunk_req)
    return E.fail(NOVA_E_STATE, "a chunked prefill is in progress: leave CHUNK mode once it is done");
  if (p->chunk_budget > NOVA_CHUNK_MAX) return E.fail(NOVA_E_INVAL, "chunk_budget > NOVA_CHUNK_MAX");
  if (p->mode == NOVA_MODE_FRONTIER && E.alg.frontier.empty())
    return E.fail(NOVA_E_STATE, "FRONTIER mode needs nova_set_frontier first");
  const int g = E.alg.granularity, mx = E.alg.max_split;
  nova_partition_policy q = *p;
  auto rnd = [&](int v) { return v / g * g; };
  q.sm_decode_dv = rnd(q.sm_decode_dv);
  q.sm_decode_dp = rnd(q.sm_decode_dp);
  q.sm_op_dv = rnd(q.sm_op_dv);
  q.sm_op_dp = rnd(q.sm_op_dp);
  q.sm_min = rnd(q.sm_min);
  if (q.b_max <= 0 || q.b_max > E.cfg.max_decode_batch) q.b_max = E.cfg.max_decode_batch;
  if (q.pf_threshold <= 0) q.pf_threshold = 5;
  if (q.chunk_budget <= 0) q.chunk_budget = 128;
  if (q.front_regroup < 0) q.front_regroup = 0;
  if (q.mode != NOVA_MODE_STATIC && q.mode != NOVA_MODE_ADAPTIVE && q.mode != NOVA_MODE_FRONTIER) q.front_regroup = 0;
  q.sm_dv_floor = q.sm_dv_floor <= 0 ? 0 : std::min(rnd(q.sm_dv_floor), mx);
  if (q.mode == NOVA_MODE_STATIC && (q.sm_decode_dv < g || q.sm_decode_dp < g || q.sm_decode_dv > mx ||
                                     q.sm_decode_dp > mx))
    return E.fail(NOVA_E_PARTITION, "static decode budget outside [granularity, max split]");
  if (q.mode == NOVA_MODE_ADAPTIVE && (q.sm_min < g || q.sm_op_dv < q.sm_min || q.sm_op_dp < q.sm_min ||
                                       q.sm_op_dv > mx || q.sm_op_dp > mx || q.alpha_dv < 0 || q.alpha_dp < 0))
    return E.fail(NOVA_E_PARTITION, "adaptive budgets outside [granularity, max split]");
  E.alg.pol = q;
  E.regroup_layers.store(q.front_regroup);
  if (applied) *applied = q;
  return NOVA_OK;
}

nova_status nova_step(nova_engine* e, int64_t max_wait_us, nova_step_info* out) {
  if (!e) return NOVA_E_INVAL;
  GUARD({ return e->e.step(max_wait_us, out); })
}

nova_status nova_poll_tokens(nova_engine* e, nova_token* buf, int32_t cap, int32_t* n_out) {
  if (!e || (!buf && cap > 0) || !n_out) return NOVA_E_INVAL;
  Engine& E = e->e;
  std::lock_guard<std::mutex> g(E.tok_mu);
  int n = 0;
  while (n < cap && !E.tok_q.empty()) {
    buf[n++] = E.tok_q.front();
    E.tok_q.pop_front();
  }
  *n_out = n;
  return NOVA_OK;
}

nova_status nova_request_stats(nova_engine* e, uint64_t id, nova_req_stats* out) {
  if (!e || !out) return NOVA_E_INVAL;
  Engine& E = e->e;
  std::lock_guard<std::mutex> g(E.ctl_mu);
  auto it = E.reqs.find(id);
  if (it == E.reqs.end()) return NOVA_E_NOTFOUND;
  *out = it->second->st;
  return NOVA_OK;
}

nova_status nova_decision_log(nova_engine* e, int64_t start, nova_log_record* buf, int32_t cap, int32_t* n_out,
                              int64_t* total) {
  if (!e || start < 0) return NOVA_E_INVAL;
  Engine& E = e->e;
  const int64_t tot = E.log_base + (int64_t)E.log.size();
  if (start < E.log_base) return E.fail(NOVA_E_NOTFOUND, "decision log records before the ring base were dropped");
  if (cap > 0 && !buf) return NOVA_E_INVAL;
  int n = 0;
  for (int64_t i = start; i < tot && n < cap; ++i) buf[n++] = E.log[(size_t)(i - E.log_base)];
  if (n_out) *n_out = n;
  if (total) *total = tot;
  return NOVA_OK;
}

int64_t nova_decision_log_base(nova_engine* e) { return e ? e->e.log_base : -1; }

nova_status nova_release_request(nova_engine* e, uint64_t id) {
  if (!e) return NOVA_E_INVAL;
  Engine& E = e->e;
  std::lock_guard<std::mutex> g(E.ctl_mu);
  auto it = E.reqs.find(id);
  if (it == E.reqs.end()) return NOVA_E_NOTFOUND;
  if (!it->second->st.finished) return E.fail(NOVA_E_STATE, "request not finished");
  E.reqs.erase(it);
  return NOVA_OK;
}

nova_status nova_debug_logits(nova_engine* e, uint64_t id, int32_t index, float* out, int32_t vocab) {
  if (!e || !out) return NOVA_E_INVAL;
  Engine& E = e->e;
  if (!E.cfg.debug_keep_logits) return E.fail(NOVA_E_STATE, "debug_keep_logits is off");
  std::lock_guard<std::mutex> g(E.ctl_mu);
  auto it = E.reqs.find(id);
  if (it == E.reqs.end()) return NOVA_E_NOTFOUND;
  const auto& L = it->second->logits;
  if (index < 0 || index >= (int)L.size() || vocab != (int)L[index].size()) return NOVA_E_INVAL;
  std::memcpy(out, L[index].data(), (size_t)vocab * 4);
  return NOVA_OK;
}

int64_t nova_front_switches(nova_engine* e) { return e ? (int64_t)e->e.front_switches.load() : -1; }

nova_status nova_debug_read_buffer(nova_engine* e, const char* name, void* out, uint64_t bytes) {
  if (!e || !name || !out) return NOVA_E_INVAL;
  Engine& E = e->e;
  if (E.sim || !E.finalized) return E.fail(NOVA_E_STATE, "no device buffers");
  const auto& m = E.dims.m;
  const uint64_t B = E.cfg.max_decode_batch, D = m.llm_dim;
  const std::string n(name);
  const void* src = nullptr;
  uint64_t cap = 0;
  if (n == "dec_hid") src = E.dw.hid, cap = B * D * 4;
  else if (n == "dec_xg") src = E.dw.xb, cap = B * D * 2;
  else if (n == "dec_xlo") src = E.dw.xlo, cap = B * D * 2;
  else if (n == "dec_qkvf") src = E.dw.qkvf, cap = B * E.dims.llm_qkv_n * 4;
  else if (n == "dec_attn") src = E.dw.attn, cap = B * m.llm_heads * m.head_dim * 2;
  else if (n == "dec_act") src = E.dw.act, cap = B * m.llm_ffn * 2;
  else if (n == "dec_ss") src = E.dw.ss, cap = B * ((D / 64 + 3) / 4 * 4) * 4;
  else if (n == "dec_dbg") src = E.dw.logits + (size_t)15 * m.vocab, cap = (uint64_t)m.vocab * 4;
  else if (n == "w_o0") src = E.W.llm[0].o_w, cap = D * m.llm_heads * m.head_dim * 2;
  else if (n == "w_ob0") src = E.W.llm[0].o_wb, cap = D * m.llm_heads * m.head_dim * 2;
  else if (n == "w_qkvb0") src = E.W.llm[0].qkv_wb, cap = (uint64_t)E.dims.llm_qkv_n * D * 2;
  else return NOVA_E_NOTFOUND;
  if (bytes > cap) return NOVA_E_INVAL;
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(out, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    return E.fail(NOVA_E_CUDA, "debug read");
  return NOVA_OK;
}

nova_status nova_debug_force_tokens(nova_engine* e, uint64_t id, const int32_t* tokens, int32_t n) {
  if (!e || (!tokens && n > 0) || n < 0) return NOVA_E_INVAL;
  Engine& E = e->e;
  std::lock_guard<std::mutex> g(E.ctl_mu);
  auto it = E.reqs.find(id);
  if (it == E.reqs.end()) return NOVA_E_NOTFOUND;
  for (int i = 0; i < n; ++i)
    if (tokens[i] < 0 || tokens[i] >= E.dims.m.vocab) return NOVA_E_INVAL;
  it->second->forced.assign(tokens, tokens + n);
  return NOVA_OK;
}

nova_status nova_time_pass(nova_engine* e, int32_t stage, int32_t s, int32_t gh, int32_t gw, int32_t n_prompt,
                           int32_t B, int32_t ctx, int32_t corun, int32_t iters, double* out_ms) {
  if (!e || !out_ms) return NOVA_E_INVAL;
  GUARD({ return e->e.time_pass(stage, s, gh, gw, n_prompt, B, ctx, corun, iters, out_ms); })
}

nova_status nova_kernel_timing(nova_engine* e, int32_t every_n) {
  if (!e || every_n < 0) return NOVA_E_INVAL;
  e->e.sample_every = every_n;
  return NOVA_OK;
}

nova_status nova_kernel_stats(nova_engine* e, int32_t cls, double* out3) {
  if (!e || !out3 || cls < 0 || cls >= NOVA_K_COUNT) return NOVA_E_INVAL;
  std::lock_guard<std::mutex> g(e->e.kmu);
  out3[0] = e->e.kstats[cls].ms;
  out3[1] = e->e.kstats[cls].work;
  out3[2] = (double)e->e.kstats[cls].launches;
  return NOVA_OK;
}

nova_status nova_kernel_stats_sm(nova_engine* e, int32_t cls, double* sm_ms) {
  if (!e || !sm_ms || cls < 0 || cls >= NOVA_K_COUNT) return NOVA_E_INVAL;
  std::lock_guard<std::mutex> g(e->e.kmu);
  *sm_ms = e->e.kstats[cls].sm_ms;
  return NOVA_OK;
}

uint64_t nova_launch_count(void) { return g_kernel_launches.load(); }

nova_status nova_kernel_stats_reset(nova_engine* e) {
  if (!e) return NOVA_E_INVAL;
  std::lock_guard<std::mutex> g(e->e.kmu);
  for (auto& k : e->e.kstats) k = KStat{};
  return NOVA_OK;
}

nova_status nova_sim_set_curves(nova_engine* e, const nova_sim_curves* c) {
  if (!e || !c || c->n <= 0 || !c->s || !c->t_v || !c->t_p || !c->t_d_dv || !c->t_d_dp) return NOVA_E_INVAL;
  Engine& E = e->e;
  if (!E.sim) return E.fail(NOVA_E_STATE, "sim curves on a GPU engine");
  E.sc = *c;
  E.sc_s.assign(c->s, c->s + c->n);
  E.sc_tv.assign(c->t_v, c->t_v + c->n);
  E.sc_tp.assign(c->t_p, c->t_p + c->n);
  E.sc_tdv.assign(c->t_d_dv, c->t_d_dv + c->n);
  E.sc_tdp.assign(c->t_d_dp, c->t_d_dp + c->n);
  E.alg.total_sms = c->total_sms > 0 ? c->total_sms : 148;
  E.alg.granularity = c->granularity > 0 ? c->granularity : 8;
  E.alg.max_split = E.alg.total_sms - E.alg.granularity;
  return NOVA_OK;
}

}  // extern "C"
