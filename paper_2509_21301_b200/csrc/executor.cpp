// L3 partition executor and engine lifecycle.
//
// SM partitioning (§III-B, §IV: libsmctrl stream masks on
// sm_86) is realised with CUDA green contexts: ONE split of the device's SMs into
// 8-SM groups is made at finalize, and for every decode split k the pair
// (decode = groups[0:k], front = groups[k:] + remainder) is materialised as two
// green contexts with a stream each.  A repartition (Eq. 5, per forward pass,
// P:410) is only the choice of which pre-built stream the next pass is launched
// on: nothing is rebuilt or relaunched.  Two role workers (front: vision/prefill,
// decode) each issue one pass at a time, as the paper's model workers do
// (P:237); completion is observed host-side and handed to the Algorithm 1
// controller (nova_step).
#include <algorithm>
#include <chrono>
#include <cstring>

#include "engine.h"

namespace nova {

#define CU_OK(x) ((x) == CUDA_SUCCESS)

// Driver entry points resolved through the runtime, so libnova.so loads (and its
// Sim backend / planner run) on hosts without a GPU driver.
namespace drv {
template <typename F>
static F get(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
}  // namespace drv
#define DRV(name) static auto name = drv::get<decltype(&::name)>(#name)

std::string Partition::init(int device, bool use_green) {
  DRV(cuDeviceGet);
  DRV(cuDeviceGetDevResource);
  DRV(cuDevSmResourceSplitByCount);
  DRV(cuDevResourceGenerateDesc);
  DRV(cuGreenCtxCreate);
  DRV(cuGreenCtxStreamCreate);
  if (use_green && !(cuDeviceGet && cuDeviceGetDevResource && cuDevSmResourceSplitByCount &&
                     cuDevResourceGenerateDesc && cuGreenCtxCreate && cuGreenCtxStreamCreate))
    return "green-context driver entry points unavailable";
  if (cudaSetDevice(device) != cudaSuccess) return "cudaSetDevice failed";
  cudaFree(0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  total = sms;
  if (cudaStreamCreateWithFlags(&solo_front, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&solo_decode, cudaStreamNonBlocking) != cudaSuccess)
    return "stream creation failed";
  green = false;
  if (use_green) {
    CUdevice dev;
    CUdevResource all;
    unsigned nb = 0;
    if (CU_OK(cuDeviceGet(&dev, device)) && CU_OK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM)) &&
        CU_OK(cuDevSmResourceSplitByCount(nullptr, &nb, &all, nullptr, 0, 8)) && nb >= 2) {
      std::vector<CUdevResource> groups(nb);
      CUdevResource rem;
      if (!CU_OK(cuDevSmResourceSplitByCount(groups.data(), &nb, &all, &rem, 0, 8))) return "SM split failed";
      n_groups = (int)nb;
      granularity = (int)groups[0].sm.smCount;
      total = (int)all.sm.smCount;
      dec_stream.assign(n_groups, nullptr);
      front_stream.assign(n_groups, nullptr);
      for (int k = 1; k < n_groups; ++k) {
        std::vector<CUdevResource> dv(groups.begin(), groups.begin() + k), fv(groups.begin() + k, groups.end());
        if (rem.sm.smCount > 0) fv.push_back(rem);
        CUdevResourceDesc dd, fd;
        CUgreenCtx g1, g2;
        CUstream s1, s2;
        if (!CU_OK(cuDevResourceGenerateDesc(&dd, dv.data(), (unsigned)dv.size())) ||
            !CU_OK(cuDevResourceGenerateDesc(&fd, fv.data(), (unsigned)fv.size())) ||
            !CU_OK(cuGreenCtxCreate(&g1, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM)) ||
            !CU_OK(cuGreenCtxCreate(&g2, fd, dev, CU_GREEN_CTX_DEFAULT_STREAM)) ||
            !CU_OK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0)) ||
            !CU_OK(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0)))
          return "green context creation failed";
        gctx.push_back(g1);
        gctx.push_back(g2);
        dec_stream[k] = (cudaStream_t)s1;
        front_stream[k] = (cudaStream_t)s2;
      }
      green = true;
      return "";
    }
    // Partitioning was requested but the driver cannot split the SMs: fail loudly rather than
    // run every policy on one shared stream while reporting splits that isolate nothing.
    return "green-context SM split unavailable (fewer than 2 groups of 8 SMs); use_green_ctx = 0 runs unpartitioned";
  }
  // no partitioning: every role stream is a plain primary-context stream
  granularity = 8;
  n_groups = total / 8;
  dec_stream.assign(n_groups, solo_decode);
  front_stream.assign(n_groups, solo_front);
  return "";
}

void Partition::destroy() {
  DRV(cuGreenCtxDestroy);
  if (green) {
    for (auto s : dec_stream)
      if (s) cudaStreamDestroy(s);
    for (auto s : front_stream)
      if (s) cudaStreamDestroy(s);
    for (auto g : gctx) cuGreenCtxDestroy(g);
  }
  dec_stream.clear();
  front_stream.clear();
  gctx.clear();
  if (solo_front) cudaStreamDestroy(solo_front);
  if (solo_decode) cudaStreamDestroy(solo_decode);
  solo_front = solo_decode = nullptr;
}

cudaStream_t Engine::stream_for(int role, int ctx, int s_dec) {
  if (role == 0) {  // front
    if (s_dec <= 0) return part.solo_front;
    return part.front_stream[std::min(s_dec / part.granularity, part.n_groups - 1)];
  }
  if (ctx == NOVA_CTX_SOLO || s_dec >= part.total) return part.solo_decode;
  return part.dec_stream[std::max(1, std::min(s_dec / part.granularity, part.n_groups - 1))];
}

// ---------------------------------------------------------------- workers
void Worker::start(Engine* e, int r) {
  eng = e;
  role = r;
  stop = false;
  th = std::thread([this] { run(); });
}

void Worker::push(PassCmd&& c) {
  {
    std::lock_guard<std::mutex> g(mu);
    q.push_back(std::move(c));
  }
  cv.notify_one();
}

static void spin_wait(cudaEvent_t ev) {
  // low-latency completion detection (the pass is async; this thread only waits)
  int n = 0;
  while (cudaEventQuery(ev) == cudaErrorNotReady) {
    if (++n > 64) std::this_thread::sleep_for(std::chrono::microseconds(5));
  }
}

void Worker::run() {
  cudaSetDevice(eng->cfg.device);
  cudaEvent_t ev, p0, p1;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventCreate(&p0);
  cudaEventCreate(&p1);
  for (;;) {
    PassCmd c;
    {
      std::unique_lock<std::mutex> g(mu);
      cv.wait(g, [&] { return stop || !q.empty(); });
      if (stop && q.empty()) break;
      c = std::move(q.front());
      q.pop_front();
    }
    cudaStream_t s = eng->stream_for(role, c.ctx, c.s_dec);
    cudaError_t e = cudaSuccess;
    const bool timing = eng->sample_every > 0;
    eng->ktimer[role].on = timing && (eng->pass_count[role]++ % eng->sample_every == 0);
    {  // the pass's SM budget (partition-normalized rooflines)
      const int psms = role == 0 ? (c.kind == NOVA_DEC_HYBRID ? eng->part.total : eng->front_sms(c.s_dec))
                                 : eng->dec_sms(c.ctx, c.s_dec);
      eng->ktimer[role].share = (double)psms / (double)eng->part.total;
    }
    if (timing) cudaEventRecord(p0, s);
    Event done;
    done.reqs = c.reqs;
    done.key = c.reqs.empty() ? 0 : c.reqs[0]->id;
    Engine::FrontRG rg{c.s_dec, eng->regroup_layers.load()};
    Engine::FrontRG* rgp = (role == 0 && rg.group > 0) ? &rg : nullptr;
    if (c.kind == NOVA_DEC_VISION) {
      e = eng->run_encode(c.reqs[0], s, eng->front_sms(c.s_dec), rgp);  // may move s (f4)
      done.kind = NOVA_EV_VISION_DONE;
    } else if (c.kind == NOVA_DEC_PREFILL) {
      e = eng->run_prefill(c.reqs[0], s, eng->front_sms(c.s_dec), rgp);
      done.kind = NOVA_EV_PREFILL_DONE;
    } else if (c.kind == NOVA_DEC_HYBRID) {
      e = eng->run_hybrid(c.reqs, c.forced_tok, s, eng->part.total);
      done.kind = NOVA_EV_HYBRID_DONE;
      for (Request* r : c.reqs) done.key = std::min<uint64_t>(done.key, r->id);
    } else {
      e = eng->run_decode(c.reqs, c.forced_tok, s, eng->dec_sms(c.ctx, c.s_dec));
      done.kind = NOVA_EV_DECODE_DONE;
      for (Request* r : c.reqs) done.key = std::min<uint64_t>(done.key, r->id);
    }
    if (e == cudaSuccess && timing) e = cudaEventRecord(p1, s);
    if (e == cudaSuccess) e = cudaEventRecord(ev, s);
    if (e == cudaSuccess) {
      spin_wait(ev);
      e = cudaEventQuery(ev) == cudaSuccess ? cudaSuccess : cudaGetLastError();
    }
    done.t = mono_ns();
    if (e == cudaSuccess && timing) {
      float ms = 0;
      cudaEventElapsedTime(&ms, p0, p1);
      const int cls = c.kind == NOVA_DEC_VISION ? NOVA_K_VIT_PASS
                                                : ((c.kind == NOVA_DEC_PREFILL || c.kind == NOVA_DEC_HYBRID)
                                                       ? NOVA_K_PRE_PASS
                                                       : NOVA_K_DEC_PASS);
      {
        std::lock_guard<std::mutex> g(eng->kmu);
        eng->kstats[cls].ms += ms;
        eng->kstats[cls].work += eng->pass_work[role];
        eng->kstats[cls].launches += 1;
        eng->kstats[cls].sm_ms += ms * eng->ktimer[role].share;
      }
      eng->ktimer[role].harvest(eng->kstats, eng->kmu);
    }
    if (e != cudaSuccess) {
      eng->fail(NOVA_E_CUDA, std::string("CUDA error in stage pass: ") + cudaGetErrorString(e));
    } else {
      const int V = eng->dims.m.vocab;
      if (c.kind == NOVA_DEC_PREFILL) {
        done.tokens.push_back(eng->fw.h_tok[0]);
        if (eng->cfg.debug_keep_logits)
          c.reqs[0]->logits.emplace_back(eng->fw.h_logits, eng->fw.h_logits + V);
      } else if (c.kind == NOVA_DEC_DECODE) {
        for (size_t b = 0; b < c.reqs.size(); ++b) {
          done.tokens.push_back(eng->dw.h_tok[b]);
          if (eng->cfg.debug_keep_logits)
            c.reqs[b]->logits.emplace_back(eng->dw.h_logits + b * V, eng->dw.h_logits + (b + 1) * V);
        }
      } else if (c.kind == NOVA_DEC_HYBRID) {  // hw.h_tok[0]: the prefill token (last chunk); [1..]: decode rows
        for (size_t b = 0; b < c.reqs.size(); ++b) {
          done.tokens.push_back(eng->hw.h_tok[b]);
          const bool emits = b > 0 || c.reqs[0]->chunk_c0 + c.reqs[0]->chunk_n >= c.reqs[0]->S();
          if (eng->cfg.debug_keep_logits && emits)
            c.reqs[b]->logits.emplace_back(eng->hw.h_logits + b * V, eng->hw.h_logits + (b + 1) * V);
        }
      }
    }
    eng->post_completion(std::move(done));
  }
  cudaEventDestroy(ev);
  cudaEventDestroy(p0);
  cudaEventDestroy(p1);
}

void Engine::post_completion(Event&& e) {
  {
    std::lock_guard<std::mutex> g(wake_mu);
    completions.push_back(std::move(e));
  }
  wake.notify_all();
}

// ---------------------------------------------------------------- lifecycle
nova_status Engine::create(const nova_model_config* m, const nova_engine_config* c, const nova_buffers* b) {
  dims.init(*m);
  cfg = *c;
  sim = c->backend == NOVA_BACKEND_SIM;
  if (cfg.max_decode_batch <= 0 || cfg.max_decode_batch > 16) return fail(NOVA_E_INVAL, "max_decode_batch in 1..16");
  if (cfg.max_requests <= 0) return fail(NOVA_E_INVAL, "max_requests must be > 0");
  alg.pol = nova_partition_policy{NOVA_MODE_ADAPTIVE, 72, 72, 48, 48, 16, 8.f, 8.f, cfg.max_decode_batch, 5, 0, 128};
  free_slots.clear();
  for (int i = cfg.max_requests - 1; i >= 0; --i) free_slots.push_back(i);
  if (sim) {
    alg.total_sms = 148;
    alg.granularity = 8;
    return NOVA_OK;
  }
  if (!b || !b->weights_dev || !b->kv_dev || !b->workspace_dev) return fail(NOVA_E_INVAL, "device buffers required");
  if (dims.m.vit_dim % dims.m.vit_heads || dims.m.llm_heads % dims.m.llm_kv_heads)
    return fail(NOVA_E_INVAL, "head counts");
  buf = *b;
  const size_t wb = plan_weights(dims, cfg, nullptr, nullptr, nullptr);
  const size_t ws = plan_workspace(dims, cfg, nullptr, nullptr);
  const size_t kb = plan_kv(dims, cfg);
  if (b->weights_bytes < wb || b->workspace_bytes < ws || b->kv_bytes < kb)
    return fail(NOVA_E_NOMEM, "device buffers smaller than nova_query_memory");
  if (cudaSetDevice(cfg.device) != cudaSuccess) return fail(NOVA_E_CUDA, "cudaSetDevice");
  plan_weights(dims, cfg, &W, &vl, reinterpret_cast<uint8_t*>(b->weights_dev));
  plan_workspace(dims, cfg, this, reinterpret_cast<uint8_t*>(b->workspace_dev));
  vit_K = (cfg.vit_resident_layers > 0 && cfg.vit_resident_layers < dims.m.vit_depth) ? cfg.vit_resident_layers : 0;
  if (vit_K == 1) return fail(NOVA_E_INVAL, "offload needs K >= 2 physical layers (P:427)");
  if (vit_K > 0) {
    if (cudaHostAlloc(&host_vit, (size_t)dims.m.vit_depth * vl.elems * 2, cudaHostAllocDefault) != cudaSuccess)
      return fail(NOVA_E_NOMEM, "pinned offload arena");
  }
  const int S = s_max_of_public();
  const size_t B = cfg.max_decode_batch, V = dims.m.vocab;
  if (cudaHostAlloc(&fw.h_pos3, 3 * S * sizeof(int), 0) || cudaHostAlloc(&fw.h_tok, 64, 0) ||
      cudaHostAlloc(&fw.h_logits, V * 4, 0) || cudaHostAlloc(&dw.h_rows, B * sizeof(DecodeRow), 0) ||
      cudaHostAlloc(&dw.h_tok, B * 4, 0) || cudaHostAlloc(&dw.h_forced, B * 4, 0) ||
      cudaHostAlloc(&dw.h_logits, B * V * 4, 0) ||
      cudaHostAlloc(&hw.h_rows, (NOVA_CHUNK_MAX + 16) * sizeof(DecodeRow), 0) ||
      cudaHostAlloc(&hw.h_lm_rows, 17 * sizeof(DecodeRow), 0) || cudaHostAlloc(&hw.h_pos3, 3 * NOVA_CHUNK_MAX * 4, 0) ||
      cudaHostAlloc(&hw.h_tok, 17 * 4, 0) || cudaHostAlloc(&hw.h_forced, 16 * 4, 0) ||
      cudaHostAlloc(&hw.h_logits, 17 * V * 4, 0))
    return fail(NOVA_E_NOMEM, "pinned host buffers");
  free_pages.clear();
  for (int i = cfg.kv_pages - 1; i >= 0; --i) free_pages.push_back(i);
  return NOVA_OK;
}

int Engine::s_max_of_public() const {
  return cfg.max_patches / (dims.m.merge * dims.m.merge) + cfg.max_prompt;
}

nova_status Engine::finalize() {
  if (finalized) return fail(NOVA_E_STATE, "already finalized");
  if (sim) {
    finalized = true;
    return NOVA_OK;
  }
  std::string e = part.init(cfg.device, cfg.use_green_ctx != 0);
  if (!e.empty()) return fail(NOVA_E_CUDA, e);
  alg.total_sms = part.total;
  alg.granularity = part.granularity;
  alg.max_split = part.max_split();
  if (cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&upload_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(NOVA_E_CUDA, "streams");
  if (cudaEventCreateWithFlags(&regroup_ev, cudaEventDisableTiming) != cudaSuccess) return fail(NOVA_E_CUDA, "events");
  ev_upload.assign(n_slots_total, nullptr);
  for (auto& ev : ev_upload)
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return fail(NOVA_E_CUDA, "events");
  if (vit_K > 0) {  // preload logical layers 0..K-1 into the physical slots
    vit_slot_of.assign(dims.m.vit_depth, -1);
    for (int k = 0; k < vit_K; ++k) vit_slot_of[k] = k;
    ev_loaded.assign(vit_K, nullptr);
    ev_free.assign(vit_K, nullptr);
    for (int k = 0; k < vit_K; ++k) {
      cudaEventCreateWithFlags(&ev_loaded[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev_free[k], cudaEventDisableTiming);
      if (cudaMemcpyAsync(W.vit_dev[k], host_vit + (size_t)k * vl.elems, vl.elems * 2, cudaMemcpyHostToDevice,
                          copy_stream) != cudaSuccess)
        return fail(NOVA_E_CUDA, "offload preload");
      cudaEventRecord(ev_loaded[k], copy_stream);
    }
  }
  {  // decode copies of the LLM linears in the streaming layout (model.cpp plan_weights)
    const auto& m = dims.m;
    const int D = m.llm_dim, F = m.llm_ffn, HD = m.llm_heads * m.head_dim;
    cudaError_t e = cudaSuccess;
    for (int l = 0; l < m.llm_layers && e == cudaSuccess; ++l) {
      const LlmLayerW& L = W.llm[l];
      e = block_weights(L.qkv_w, L.qkv_wb, dims.llm_qkv_n, D, copy_stream);
      if (e == cudaSuccess) e = block_weights(L.o_w, L.o_wb, D, HD, copy_stream);
      if (e == cudaSuccess) e = block_weights(L.gu_w, L.gu_wb, 2 * F, D, copy_stream);
      if (e == cudaSuccess) e = block_weights(L.down_w, L.down_wb, D, F, copy_stream);
    }
    if (e == cudaSuccess) e = block_weights(W.lm_head, W.lm_head_b, m.vocab, D, copy_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(copy_stream);
    if (e != cudaSuccess) return fail(NOVA_E_CUDA, std::string("streaming weight layout: ") + cudaGetErrorString(e));
  }
  cudaMemset(d_pix, 0, pix_stride * 2 * n_slots_total);
  cudaMemset(d_prompt, 0, (size_t)n_slots_total * cfg.max_prompt * 4);
  cudaMemset(d_bt, 0, (size_t)n_slots_total * max_pages_per_req * 4);
  cudaMemset(d_last, 0, (size_t)n_slots_total * 4);
  cudaMemset(dw.tickets, 0, 8192 * 4);
  cudaMemset(dw.keys, 0, (size_t)cfg.max_decode_batch * 8);
  cudaMemset(dw.bar, 0, 512 * 8);
  dec_bar_base = 0;
  {  // fused decode iteration: tensor maps of the activation tiles and the paged pool
    const auto& m = dims.m;
    if (g_dec_fused && decode_fused_supported(m.llm_dim, m.llm_heads, m.llm_kv_heads, m.head_dim, m.llm_ffn, m.vocab)) {
      DecFusedSetup su;
      su.L = m.llm_layers, su.D = m.llm_dim, su.H = m.llm_heads, su.KV = m.llm_kv_heads, su.hd = m.head_dim;
      su.F = m.llm_ffn, su.V = m.vocab, su.bmax = cfg.max_decode_batch, su.n_pages = cfg.kv_pages;
      su.xg = dw.xb, su.xlo = dw.xlo, su.attn = dw.attn, su.act = dw.act;
      su.pool = reinterpret_cast<const bf16*>(buf.kv_dev);
      for (const LlmLayerW& L : W.llm) {
        su.ln1.push_back(L.ln1), su.ln2.push_back(L.ln2), su.qkv_b.push_back(L.qkv_b);
        su.qkv_wb.push_back(L.qkv_wb), su.o_wb.push_back(L.o_wb), su.gu_wb.push_back(L.gu_wb);
        su.down_wb.push_back(L.down_wb);
      }
      dfs = decode_fused_create(su);
      if (!dfs) return fail(NOVA_E_CUDA, "fused decode setup (tensor maps / layer table)");
    }
  }
  cudaMemset(fw.keys, 0, 16 * 8);
  cudaMemset(hw.keys, 0, 17 * 8);
  ktimer[0].init(512);
  ktimer[1].init(512);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(NOVA_E_CUDA, "finalize sync");
  front_w.start(this, 0);
  dec_w.start(this, 1);
  finalized = true;
  return NOVA_OK;
}

void Engine::shutdown() {
  if (!sim && finalized) {
    for (Worker* w : {&front_w, &dec_w}) {
      {
        std::lock_guard<std::mutex> g(w->mu);
        w->stop = true;
      }
      w->cv.notify_all();
      if (w->th.joinable()) w->th.join();
    }
    cudaDeviceSynchronize();
    ktimer[0].destroy();
    ktimer[1].destroy();
    decode_fused_destroy(dfs);
    dfs = nullptr;
    part.destroy();
    for (auto ev : ev_upload) cudaEventDestroy(ev);
    if (regroup_ev) cudaEventDestroy(regroup_ev);
    regroup_ev = nullptr;
    for (auto ev : ev_loaded) cudaEventDestroy(ev);
    for (auto ev : ev_free) cudaEventDestroy(ev);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (upload_stream) cudaStreamDestroy(upload_stream);
    ev_upload.clear();
    ev_loaded.clear();
    ev_free.clear();
    copy_stream = upload_stream = nullptr;
  }
  if (!sim) {
    for (void* p : {(void*)host_vit, (void*)fw.h_pos3, (void*)fw.h_tok, (void*)fw.h_logits, (void*)dw.h_rows,
                    (void*)dw.h_tok, (void*)dw.h_forced, (void*)dw.h_logits, (void*)hw.h_rows, (void*)hw.h_lm_rows,
                    (void*)hw.h_pos3, (void*)hw.h_tok, (void*)hw.h_forced, (void*)hw.h_logits})
      if (p) cudaFreeHost(p);
    hw.h_rows = hw.h_lm_rows = nullptr;
    hw.h_pos3 = hw.h_tok = hw.h_forced = nullptr;
    hw.h_logits = nullptr;
    host_vit = nullptr;
    fw.h_pos3 = fw.h_tok = nullptr;
    fw.h_logits = nullptr;
    dw.h_rows = nullptr;
    dw.h_tok = dw.h_forced = nullptr;
    dw.h_logits = nullptr;
  }
  finalized = false;
}

// ---------------------------------------------------------------- requests
nova_status Engine::submit(const nova_request* q, uint64_t* id) {
  if (failed) return fail(NOVA_E_STATE, "engine failed: " + last_error());
  if (!finalized) return fail(NOVA_E_STATE, "nova_finalize first");
  const auto& m = dims.m;
  const int unit = m.patch * m.merge;
  if (!q || q->height <= 0 || q->width <= 0 || q->height % unit || q->width % unit)
    return fail(NOVA_E_INVAL, "image height/width must be positive multiples of patch*merge");
  const int gh = q->height / m.patch, gw = q->width / m.patch;
  if (gh * gw > cfg.max_patches) return fail(NOVA_E_INVAL, "image has more patches than max_patches");
  if (q->n_prompt < 0 || q->n_prompt > cfg.max_prompt) return fail(NOVA_E_INVAL, "n_prompt out of range");
  if (q->gen_len < 1 || q->gen_len > cfg.max_gen) return fail(NOVA_E_INVAL, "gen_len out of range");
  if (!sim) {
    if (!q->pixels_bf16 || (q->n_prompt > 0 && !q->prompt_ids)) return fail(NOVA_E_INVAL, "null input");
    for (int i = 0; i < q->n_prompt; ++i)
      if (q->prompt_ids[i] < 0 || q->prompt_ids[i] >= m.vocab) return fail(NOVA_E_INVAL, "token id out of range");
  }
  auto r = std::make_unique<Request>();
  r->gh = gh;
  r->gw = gw;
  r->n_prompt = q->n_prompt;
  r->gen_len = q->gen_len;
  r->sim_vs = q->sim_vision_scale > 0 ? q->sim_vision_scale : 1.f;
  r->sim_ps = q->sim_prefill_scale > 0 ? q->sim_prefill_scale : 1.f;
  const int need_pages = (r->S() + r->gen_len - 1 + 63) / 64;
  {
    std::lock_guard<std::mutex> g(ctl_mu);
    if (free_slots.empty()) return fail(NOVA_E_AGAIN, "no free request slot");
    if (!sim) {
      if (need_pages > max_pages_per_req) return fail(NOVA_E_INVAL, "request exceeds max context");
      if ((int)free_pages.size() < need_pages) return fail(NOVA_E_AGAIN, "no free KV pages");
      for (int i = 0; i < need_pages; ++i) {
        r->pages.push_back(free_pages.back());
        free_pages.pop_back();
      }
    }
    r->slot = free_slots.back();
    free_slots.pop_back();
    r->id = next_id++;
  }
  if (!sim) {
    const size_t npix = (size_t)m.in_ch * q->height * q->width;
    // pixels may be host or device memory (UVA): H2D for host buffers, D2D for HBM-resident inputs
    cudaError_t e = cudaMemcpyAsync(d_pix + (size_t)r->slot * pix_stride, q->pixels_bf16, npix * 2, cudaMemcpyDefault,
                                    upload_stream);
    if (e == cudaSuccess && q->n_prompt > 0)
      e = cudaMemcpyAsync(d_prompt + (size_t)r->slot * cfg.max_prompt, q->prompt_ids, q->n_prompt * 4,
                          cudaMemcpyHostToDevice, upload_stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_bt + (size_t)r->slot * max_pages_per_req, r->pages.data(), r->pages.size() * 4,
                          cudaMemcpyHostToDevice, upload_stream);
    if (e == cudaSuccess) e = cudaEventRecord(ev_upload[r->slot], upload_stream);
    if (e != cudaSuccess) return fail(NOVA_E_CUDA, std::string("submit copy: ") + cudaGetErrorString(e));
  }
  r->arrival = sim ? q->arrival_ns : (q->arrival_ns > 0 ? q->arrival_ns : mono_ns());
  r->st.arrival = r->arrival;
  *id = r->id;
  Request* raw = r.get();
  {
    std::lock_guard<std::mutex> g(ctl_mu);
    reqs[r->id] = std::move(r);
  }
  {
    std::lock_guard<std::mutex> g(inbox_mu);
    inbox.push_back(raw);
  }
  { std::lock_guard<std::mutex> g(wake_mu); }  // no lost wake-up against step()'s predicate check
  wake.notify_all();
  return NOVA_OK;
}

void Engine::finish_request(Request* r) {
  r->st.finished = 1;
  finished++;
  std::lock_guard<std::mutex> g(ctl_mu);
  for (int p : r->pages) free_pages.push_back(p);
  r->pages.clear();
  free_slots.push_back(r->slot);
  // Bounded memory for a long-running server: keep the records of the last `retention` finished
  // requests (no pass or scheduler queue references a finished request any more).
  finished_ids.push_back(r->id);
  const int ret = cfg.finished_retention == 0 ? 4096 : cfg.finished_retention;
  if (ret > 0)
    while ((int)finished_ids.size() > ret) {
      reqs.erase(finished_ids.front());  // no-op if already released by nova_release_request
      finished_ids.pop_front();
    }
}

void Engine::log_push(const nova_log_record& r) {
  log.push_back(r);
  while (log.size() > (size_t)NOVA_LOG_CAPACITY) {
    log.pop_front();
    log_base++;
  }
}

void Engine::log_event(const Event& e) {
  nova_log_record rec{};
  rec.t_ns = e.t;
  rec.tick = tick_no;
  rec.is_event = 1;
  rec.kind = e.kind;
  rec.n_ids = (int)std::min<size_t>(16, e.reqs.size());
  for (int i = 0; i < rec.n_ids; ++i) rec.ids[i] = e.reqs[i]->id;
  log_push(rec);
}

void Engine::log_decision(const Decision& d, int64_t t) {
  nova_log_record rec{};
  rec.t_ns = t;
  rec.tick = tick_no;
  rec.is_event = 0;
  rec.kind = d.kind;
  rec.ctx = d.ctx;
  rec.s_dec = d.s_dec;
  rec.n_ids = (int)std::min<size_t>(16, d.reqs.size());
  for (int i = 0; i < rec.n_ids; ++i) rec.ids[i] = d.reqs[i]->id;
  log_push(rec);
}

static int64_t curve_at(const std::vector<int32_t>& s, const std::vector<int64_t>& t, int v) {
  for (size_t i = 0; i < s.size(); ++i)
    if (s[i] == v) return t[i];
  // nearest lower split
  int64_t best = t.empty() ? 0 : t[0];
  for (size_t i = 0; i < s.size(); ++i)
    if (s[i] <= v) best = t[i];
  return best;
}

void Engine::dispatch(const Decision& d) {
  const int64_t now = sim ? sim_now : mono_ns();
  if (d.kind == NOVA_DEC_FINISH) {
    finish_request(d.reqs[0]);
    return;
  }
  if (d.kind == NOVA_DEC_VISION) {
    d.reqs[0]->st.vis_start = now;
    d.reqs[0]->st.split_at_vis = d.s_dec;
  } else if (d.kind == NOVA_DEC_PREFILL) {
    d.reqs[0]->st.pre_start = now;
    d.reqs[0]->st.split_at_pre = d.s_dec;
  } else if (d.kind == NOVA_DEC_HYBRID && d.reqs[0]->chunk_c0 == 0) {
    d.reqs[0]->st.pre_start = now;
  }
  if (sim) {
    Event ev;
    ev.reqs = d.reqs;
    ev.key = d.reqs[0]->id;
    int64_t dur;
    if (d.kind == NOVA_DEC_VISION) {
      ev.kind = NOVA_EV_VISION_DONE;
      dur = (int64_t)llround((d.ctx == NOVA_CTX_SOLO ? sc.t_v_solo : curve_at(sc_s, sc_tv, d.s_dec)) * d.reqs[0]->sim_vs);
    } else if (d.kind == NOVA_DEC_PREFILL) {
      ev.kind = NOVA_EV_PREFILL_DONE;
      dur = (int64_t)llround((d.ctx == NOVA_CTX_SOLO ? sc.t_p_solo : curve_at(sc_s, sc_tp, d.s_dec)) * d.reqs[0]->sim_ps);
      ev.tokens.push_back(-1);
    } else if (d.kind == NOVA_DEC_HYBRID) {  // chunk share of the solo prefill + the decode batch
      ev.kind = NOVA_EV_HYBRID_DONE;
      for (Request* r : d.reqs) ev.key = std::min<uint64_t>(ev.key, r->id);
      Request* p = d.reqs[0];
      const double nb = (double)d.reqs.size() - 1;
      const double dd = nb > 0 ? (double)sc.t_d_solo * (1.0 + sc.beta * (nb - 1)) : 0.0;
      dur = (int64_t)llround((double)sc.t_p_solo * p->sim_ps * p->chunk_n / p->S() + dd);
      ev.tokens.assign(d.reqs.size(), -1);
    } else {
      ev.kind = NOVA_EV_DECODE_DONE;
      for (Request* r : d.reqs) ev.key = std::min<uint64_t>(ev.key, r->id);
      int64_t base = d.ctx == NOVA_CTX_SOLO ? sc.t_d_solo
                                             : curve_at(sc_s, d.ctx == NOVA_CTX_DV ? sc_tdv : sc_tdp, d.s_dec);
      dur = (int64_t)llround(base * (1.0 + sc.beta * ((double)d.reqs.size() - 1)));
      ev.tokens.assign(d.reqs.size(), -1);
    }
    ev.t = now + dur;
    sim_pending.push_back(SimPending{ev.t, std::move(ev)});
    return;
  }
  PassCmd c;
  c.kind = d.kind;
  c.ctx = d.ctx;
  c.s_dec = d.s_dec;
  c.reqs = d.reqs;
  if (d.kind == NOVA_DEC_DECODE || d.kind == NOVA_DEC_HYBRID) {
    c.forced_tok.assign(d.reqs.size(), -1);
    for (size_t b = d.kind == NOVA_DEC_HYBRID ? 1 : 0; b < d.reqs.size(); ++b) {
      Request* r = d.reqs[b];
      const int k = r->emitted;  // feeding token k-1
      if ((int)r->forced.size() >= k && k >= 1) c.forced_tok[b] = r->forced[k - 1];
    }
    dec_w.push(std::move(c));
  } else {
    front_w.push(std::move(c));
  }
}

nova_status Engine::step(int64_t max_wait_us, nova_step_info* out) {
  if (failed) return fail(NOVA_E_STATE, "engine failed: " + last_error());
  if (!finalized) return fail(NOVA_E_STATE, "nova_finalize first");
  std::vector<Event> evs;
  int64_t now;
  if (sim) {
    int64_t t = INT64_MAX;
    for (auto& p : sim_pending) t = std::min(t, p.t);
    {
      std::lock_guard<std::mutex> g(inbox_mu);
      for (Request* r : inbox) t = std::min(t, r->arrival);
    }
    if (t == INT64_MAX) {
      if (out) *out = last_info, out->events = 0, out->dispatched = 0;
      return NOVA_OK;
    }
    sim_now = std::max(sim_now, t);
    now = sim_now;
    for (size_t i = 0; i < sim_pending.size();) {
      if (sim_pending[i].t == t) {
        evs.push_back(std::move(sim_pending[i].ev));
        sim_pending.erase(sim_pending.begin() + i);
      } else {
        ++i;
      }
    }
    std::lock_guard<std::mutex> g(inbox_mu);
    for (auto it = inbox.begin(); it != inbox.end();) {
      if ((*it)->arrival <= t) {
        evs.push_back(Event{NOVA_EV_ARRIVAL, (*it)->id, {*it}, (*it)->arrival, {}});
        it = inbox.erase(it);
      } else {
        ++it;
      }
    }
  } else {
    auto gather = [&] {
      {
        std::lock_guard<std::mutex> g(wake_mu);
        while (!completions.empty()) {
          evs.push_back(std::move(completions.front()));
          completions.pop_front();
        }
      }
      std::lock_guard<std::mutex> g(inbox_mu);
      while (!inbox.empty()) {
        Request* r = inbox.front();
        inbox.pop_front();
        evs.push_back(Event{NOVA_EV_ARRIVAL, r->id, {r}, r->arrival, {}});
      }
    };
    gather();
    if (evs.empty() && max_wait_us > 0) {
      std::unique_lock<std::mutex> g(wake_mu);
      wake.wait_for(g, std::chrono::microseconds(max_wait_us), [&] {
        std::lock_guard<std::mutex> g2(inbox_mu);
        return !completions.empty() || !inbox.empty() || failed;
      });
      g.unlock();
      gather();
    }
    if (failed) return fail(NOVA_E_STATE, "engine failed: " + last_error());
    now = mono_ns();
  }
  // completions: stamp stats, emit tokens
  for (Event& e : evs) {
    log_event(e);
    if (e.kind == NOVA_EV_VISION_DONE) {
      e.reqs[0]->st.vis_end = e.t;
    } else if (e.kind == NOVA_EV_PREFILL_DONE || e.kind == NOVA_EV_DECODE_DONE || e.kind == NOVA_EV_HYBRID_DONE) {
      for (size_t b = 0; b < e.reqs.size(); ++b) {
        Request* r = e.reqs[b];
        const int idx = r->emitted;  // index of this token
        const bool first = e.kind == NOVA_EV_PREFILL_DONE || (e.kind == NOVA_EV_HYBRID_DONE && b == 0);
        if (e.kind == NOVA_EV_HYBRID_DONE && b == 0 && r->pre_done + r->chunk_n < r->S()) continue;  // mid-prefill chunk
        if (first) {
          r->st.pre_end = e.t;
          r->st.first_tok = e.t;
        }
        r->st.last_tok = e.t;
        r->st.n_tokens = idx + 1;
        const int tok = b < e.tokens.size() ? e.tokens[b] : -1;
        r->tokens.push_back(tok);
        nova_token t{r->id, idx, tok, e.t, (idx == 0 ? NOVA_TOK_FIRST : 0) | (idx + 1 >= r->gen_len ? NOVA_TOK_LAST : 0), 0};
        std::lock_guard<std::mutex> g(tok_mu);
        tok_q.push_back(t);
      }
    }
  }
  std::vector<Decision> ds = alg.tick(evs);
  int dispatched = 0;
  for (const Decision& d : ds) {
    log_decision(d, now);
    dispatch(d);
    if (d.kind != NOVA_DEC_FINISH) dispatched++;
    if (d.kind == NOVA_DEC_DECODE) {
      last_info.sm_decode = d.s_dec;
      last_info.context = d.ctx;
      last_info.decode_batch = (int)d.reqs.size();
    }
  }
  if (regroup_layers.load(std::memory_order_relaxed) > 0) {  // f4: the split the policy gives now
    int hint = -1;
    if (alg.vision_running || alg.prefill_running) {
      const int ctx = alg.vision_running ? NOVA_CTX_DV : NOVA_CTX_DP;
      hint = (alg.decode_busy || !alg.q_d.empty()) ? alg.split(ctx, alg.n_pend()) : 0;
    }
    front_hint.store(hint, std::memory_order_relaxed);
  }
  tick_no++;
  last_info.events = (int)evs.size();
  last_info.dispatched = dispatched;
  last_info.n_pending = alg.n_pend();
  last_info.finished = finished;
  {
    std::lock_guard<std::mutex> g(ctl_mu);
    last_info.active = (int)reqs.size() - finished;
  }
  last_info.now_ns = now;
  if (out) *out = last_info;
  return NOVA_OK;
}

}  // namespace nova
