// L4 controller: Algorithm 1 (§III-D), the Eq. 5
// adaptive split, and the Eqs. 1-4 / Pareto / Eq. 3 planner
// as pure host code.  Readings where the paper is silent are listed
// in DESIGN.md (R9-R17); oracle/scheduler.py and oracle/planner.py state the
// same rules step by step and tests replay this controller's decision log
// against them.
#include <algorithm>
#include <cmath>
#include <time.h>

#include "engine.h"

namespace nova {

int64_t mono_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

// ---------------------------------------------------------------- Eq. 5
static int floor_g(double v, int g) { return (int)std::floor(v / g + 1e-9) * g; }

double Alg1::arrival_rate() const {
  if (arr_t.size() < 2 || arr_t.back() <= arr_t.front()) return 0.0;
  return (double)(arr_t.size() - 1) * 1e9 / (double)(arr_t.back() - arr_t.front());
}

// Frontier lookup: lowest Eq. 1 E2E among the Pareto points whose Eq. 4
// throughput covers the estimated arrival rate; ties -> more decode SMs (s_v, then s_p, as
// Eq. 3); if no point covers it, the highest throughput (ties -> lower E2E).
static const nova_plan_point* frontier_pick(const std::vector<nova_plan_point>& F, double lam) {
  const nova_plan_point* best = nullptr;
  for (const auto& p : F) {
    if (p.thr_rps < lam) continue;
    if (!best || p.e2e_ms < best->e2e_ms ||
        (p.e2e_ms == best->e2e_ms && (p.s_v > best->s_v || (p.s_v == best->s_v && p.s_p > best->s_p))))
      best = &p;
  }
  if (best) return best;
  for (const auto& p : F)
    if (!best || p.thr_rps > best->thr_rps || (p.thr_rps == best->thr_rps && p.e2e_ms < best->e2e_ms)) best = &p;
  return best;
}

int Alg1::split(int ctx, int n_pend) const {
  if (ctx == NOVA_CTX_SOLO) return total_sms;
  if (pol.mode == NOVA_MODE_STATIC) return ctx == NOVA_CTX_DV ? pol.sm_decode_dv : pol.sm_decode_dp;
  // offload-aware floor (f3): while vision co-runs, decode keeps at least sm_dv_floor SMs
  const int fl = ctx == NOVA_CTX_DV ? pol.sm_dv_floor : 0;
  if (pol.mode == NOVA_MODE_FRONTIER && !frontier.empty()) {
    const nova_plan_point* p = frontier_pick(frontier, arrival_rate());
    return std::max(fl, ctx == NOVA_CTX_DV ? p->s_v : p->s_p);
  }
  const int op = ctx == NOVA_CTX_DV ? pol.sm_op_dv : pol.sm_op_dp;
  const double a = ctx == NOVA_CTX_DV ? pol.alpha_dv : pol.alpha_dp;
  const int v = floor_g(op - a * (std::max(n_pend, 1) - 1), granularity);
  return std::max(fl, std::max(pol.sm_min, v));
}

int Alg1::n_pend() const {
  return (int)q_v.size() + (vision_running ? 1 : 0) + (int)prefill_wait.size() + (prefill_running ? 1 : 0) +
         (chunk_req ? 1 : 0);
}

void Alg1::decode_ready(Request* r) {
  if (r->join_seq < 0) r->join_seq = join_counter++;
  q_d.push_back(r);
  std::stable_sort(q_d.begin(), q_d.end(), [](Request* a, Request* b) { return a->join_seq < b->join_seq; });
}

void Alg1::emit(Request* r, std::vector<Decision>& out) {
  r->emitted += 1;
  if (r->emitted >= r->gen_len) {
    out.push_back(Decision{NOVA_DEC_FINISH, NOVA_CTX_SOLO, 0, {r}});
  } else {
    decode_ready(r);
  }
}

void Alg1::dispatch_front(std::vector<Decision>& out, bool corun, int npend, bool has_decode) {
  auto ctxs = [&](int c) -> std::pair<int, int> {
    if (!corun || !has_decode) return {NOVA_CTX_SOLO, 0};
    return {c, split(c, npend)};
  };
  if (!prefill_wait.empty()) {
    Request* r = prefill_wait.front();
    prefill_wait.pop_front();
    prefill_running = r;
    auto cs = ctxs(NOVA_CTX_DP);
    out.push_back(Decision{NOVA_DEC_PREFILL, cs.first, cs.second, {r}});
  } else if (!q_v.empty()) {
    Request* r = q_v.front();
    q_v.pop_front();
    vision_running = r;
    auto cs = ctxs(NOVA_CTX_DV);
    out.push_back(Decision{NOVA_DEC_VISION, cs.first, cs.second, {r}});
  }
}

void Alg1::dispatch_decode(std::vector<Decision>& out, int ctx, int s) {
  const int bmax = std::max(1, pol.b_max);
  const int n = std::min<int>((int)q_d.size(), bmax);
  std::vector<Request*> batch(q_d.begin(), q_d.begin() + n);
  q_d.erase(q_d.begin(), q_d.begin() + n);
  decode_running = batch;
  decode_busy = true;
  out.push_back(Decision{NOVA_DEC_DECODE, ctx, s, batch});
}

// CHUNK (the paper's chunked-prefill baseline; R26): one pass at a time on all SMs.
// An LLM step is a hybrid iteration: the next min(remaining, budget - B) prefill tokens of the
// request in chunked prefill (FIFO from the prefill queue) batched with the decode batch (B
// requests, join order, <= B_max); without a prefill in progress it is a plain decode iteration.
// Vision encode runs as its own pass (separate weights), alternating with LLM steps when
// both are ready, and only while no finished encode waits for its first chunk (one E_vis staging).
void Alg1::dispatch_chunk(std::vector<Decision>& out) {
  if (vision_running || decode_busy) return;
  const bool llm_ready = chunk_req || !prefill_wait.empty() || !q_d.empty();
  const bool vis_ready = !q_v.empty() && prefill_wait.empty();
  if (vis_ready && (!llm_ready || last_pass == 1)) {
    Request* r = q_v.front();
    q_v.pop_front();
    vision_running = r;
    out.push_back(Decision{NOVA_DEC_VISION, NOVA_CTX_SOLO, 0, {r}});
    return;
  }
  if (!llm_ready) return;
  if (!chunk_req && !prefill_wait.empty()) {
    chunk_req = prefill_wait.front();
    prefill_wait.pop_front();
  }
  const int bmax = std::max(1, pol.b_max);
  const int n = std::min<int>((int)q_d.size(), bmax);
  std::vector<Request*> batch(q_d.begin(), q_d.begin() + n);
  q_d.erase(q_d.begin(), q_d.begin() + n);
  decode_busy = true;
  if (chunk_req) {
    const int budget = pol.chunk_budget > 0 ? pol.chunk_budget : 128;
    chunk_req->chunk_c0 = chunk_req->pre_done;
    chunk_req->chunk_n = std::min(chunk_req->S() - chunk_req->pre_done, std::max(1, budget - n));
    std::vector<Request*> rs{chunk_req};
    rs.insert(rs.end(), batch.begin(), batch.end());
    decode_running = rs;
    out.push_back(Decision{NOVA_DEC_HYBRID, NOVA_CTX_SOLO, chunk_req->chunk_n, rs});
  } else {
    decode_running = batch;
    out.push_back(Decision{NOVA_DEC_DECODE, NOVA_CTX_SOLO, total_sms, batch});
  }
}

std::vector<Decision> Alg1::tick(std::vector<Event>& evs) {
  // completions before arrivals, then by request id (R13)
  std::stable_sort(evs.begin(), evs.end(), [](const Event& a, const Event& b) {
    const bool aa = a.kind == NOVA_EV_ARRIVAL, ba = b.kind == NOVA_EV_ARRIVAL;
    if (aa != ba) return !aa;
    if (a.key != b.key) return a.key < b.key;
    return a.kind < b.kind;
  });
  std::vector<Decision> out;
  for (Event& e : evs) {
    switch (e.kind) {
      case NOVA_EV_ARRIVAL:
        q_v.push_back(e.reqs[0]);
        arr_t.push_back(e.t);
        while ((int)arr_t.size() > std::max(2, lam_window)) arr_t.pop_front();
        break;
      case NOVA_EV_VISION_DONE:
        vision_running = nullptr;
        prefill_wait.push_back(e.reqs[0]);
        last_pass = 0;
        break;
      case NOVA_EV_PREFILL_DONE:
        prefill_running = nullptr;
        last_pass = 0;
        emit(e.reqs[0], out);
        break;
      case NOVA_EV_DECODE_DONE:
        decode_running.clear();
        decode_busy = false;
        last_pass = 1;
        for (Request* r : e.reqs) emit(r, out);
        break;
      case NOVA_EV_HYBRID_DONE: {  // reqs[0]: the chunked prefill (token 0 after its last chunk)
        decode_running.clear();
        decode_busy = false;
        last_pass = 1;
        Request* p = e.reqs[0];
        p->pre_done += p->chunk_n;
        if (p->pre_done >= p->S()) {
          chunk_req = nullptr;
          emit(p, out);
        }
        for (size_t i = 1; i < e.reqs.size(); ++i) emit(e.reqs[i], out);
        break;
      }
    }
  }
  const int npend = n_pend();
  if (pol.mode == NOVA_MODE_CHUNK) {
    dispatch_chunk(out);
  } else if (pol.mode == NOVA_MODE_SERIAL) {
    if (!front_running() && !decode_busy) {
      const bool front_ready = !prefill_wait.empty() || !q_v.empty();
      const bool dec_ready = !q_d.empty();
      if (front_ready && (!dec_ready || last_pass == 1))
        dispatch_front(out, false, npend, false);
      else if (dec_ready)
        dispatch_decode(out, NOVA_CTX_SOLO, total_sms);
    }
  } else if (pol.mode == NOVA_MODE_PF_LIMIT) {  // prefill-first with a decode-queue threshold
    if (!front_running() && !decode_busy) {
      const bool front_ready = !prefill_wait.empty() || !q_v.empty();
      const int thr = pol.pf_threshold > 0 ? pol.pf_threshold : 5;
      if (!q_d.empty() && ((int)q_d.size() > thr || !front_ready))
        dispatch_decode(out, NOVA_CTX_SOLO, total_sms);
      else if (front_ready)
        dispatch_front(out, false, npend, false);
    }
  } else if (pol.mode == NOVA_MODE_MULTI_STREAM) {  // co-run, every pass on all SMs
    if (!front_running()) dispatch_front(out, false, npend, false);
    if (!decode_busy && !q_d.empty()) dispatch_decode(out, NOVA_CTX_SOLO, total_sms);
  } else {
    if (!front_running()) {
      const bool has_decode = decode_busy || !q_d.empty();
      dispatch_front(out, true, npend, has_decode);
    }
    if (!decode_busy && !q_d.empty()) {
      const int ctx = vision_running ? NOVA_CTX_DV : (prefill_running ? NOVA_CTX_DP : NOVA_CTX_SOLO);
      dispatch_decode(out, ctx, split(ctx, npend));
    }
  }
  return out;
}

}  // namespace nova

// ---------------------------------------------------------------- planner (pure host, C ABI)
using namespace nova;

extern "C" {

int32_t nova_adaptive_sm(int32_t sm_op, int32_t sm_min, double alpha, int32_t n_pending, int32_t granularity) {
  const int v = floor_g(sm_op - alpha * (std::max(n_pending, 1) - 1), std::max(granularity, 1));
  return std::max(sm_min, v);
}

int32_t nova_next_logical_layer(int32_t cur, int32_t K, int32_t L) { return (cur + K) % L; }

int32_t nova_offload_floor(const int32_t* s, const double* t_v, int32_t n, double t_h2d_ms) {
  if (!s || !t_v || n <= 0) return 0;
  double tmin = t_v[0];
  for (int i = 1; i < n; ++i) tmin = std::min(tmin, t_v[i]);
  const double bound = std::max(t_h2d_ms, tmin) * 1.02;  // "no slower" within 2% (measurement noise)
  int32_t best = 0;
  for (int i = 0; i < n; ++i)
    if (t_v[i] <= bound) best = std::max(best, s[i]);
  return best;
}

double nova_required_bandwidth(double bytes, double forward_s, int32_t L, int32_t K) {
  return bytes / forward_s * (double)(L - K) / (double)(L - 2);
}

nova_status nova_plan(const nova_curves* c, double L, double tau, nova_plan_point* pts, int32_t cap, int32_t* n_out,
                      nova_plan_point* best, int32_t* sm_min_out, double* alpha_dv_out, double* alpha_dp_out) {
  if (!c || c->n <= 0 || !c->s || !c->t_v || !c->t_p || !c->t_d_dv || !c->t_d_dp) return NOVA_E_INVAL;
  const int n = c->n;
  for (int i = 0; i < n; ++i)
    if (!(c->t_v[i] > 0 && c->t_p[i] > 0 && c->t_d_dv[i] > 0 && c->t_d_dp[i] > 0)) return NOVA_E_INVAL;
  std::vector<nova_plan_point> all;
  all.reserve((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double tv = c->t_v[i], tp = c->t_p[j];
      const double pv = tv / (tv + tp), pp = tp / (tv + tp);                      // Eq. 2
      const double e2e = tv + tp + (pv * c->t_d_dv[i] + pp * c->t_d_dp[j]) * L;  // Eq. 1
      const double thr = 1000.0 / (tv + tp);                                       // Eq. 4 (req/s)
      all.push_back(nova_plan_point{c->s[i], c->s[j], e2e, thr, 0, 0});
    }
  // Eq. 3: argmin E2E, ties -> larger s_v, then larger s_p
  int bi = 0;
  for (int k = 1; k < (int)all.size(); ++k) {
    const auto &p = all[k], &b = all[bi];
    if (p.e2e_ms < b.e2e_ms || (p.e2e_ms == b.e2e_ms && (p.s_v > b.s_v || (p.s_v == b.s_v && p.s_p > b.s_p)))) bi = k;
  }
  // Pareto frontier: not dominated (<= e2e, >= thr, one strict)
  for (auto& p : all) {
    bool dom = false;
    for (const auto& q : all)
      if (q.e2e_ms <= p.e2e_ms && q.thr_rps >= p.thr_rps && (q.e2e_ms < p.e2e_ms || q.thr_rps > p.thr_rps)) {
        dom = true;
        break;
      }
    p.on_frontier = dom ? 0 : 1;
  }
  if (best) *best = all[bi];
  // SM_min: smallest split whose co-run decode stays within tau x t_d_full
  int smin = c->s[n - 1];
  const double tdf = c->t_d_full > 0 ? c->t_d_full : std::min(*std::min_element(c->t_d_dv, c->t_d_dv + n),
                                                                  *std::min_element(c->t_d_dp, c->t_d_dp + n));
  for (int i = 0; i < n; ++i)
    if (std::max(c->t_d_dv[i], c->t_d_dp[i]) <= tau * tdf) {
      smin = c->s[i];
      break;
    }
  smin = std::min(smin, std::min(all[bi].s_v, all[bi].s_p));
  if (sm_min_out) *sm_min_out = smin;
  if (alpha_dv_out) *alpha_dv_out = (all[bi].s_v - smin) / 3.0;
  if (alpha_dp_out) *alpha_dp_out = (all[bi].s_p - smin) / 3.0;
  const int cnt = std::min<int>(cap, (int)all.size());
  if (pts)
    for (int k = 0; k < cnt; ++k) pts[k] = all[k];
  if (n_out) *n_out = pts ? cnt : (int)all.size();
  return NOVA_OK;
}

}  // extern "C"
