// Latency-vs-SM curve profiler: t_v(s), t_p(s), t_d(s, B)
// solo and co-run, the inputs of the Eq. 1-3 planner ("profiling
// the forward durations under different SM partitions ... O(N)").
#include <algorithm>

#include "engine.h"

namespace nova {

nova_status Engine::time_pass(int stage, int s, int gh, int gw, int n_prompt, int B, int ctx, int corun, int iters,
                              double* out) {
  if (sim || !finalized) return fail(NOVA_E_STATE, "time_pass needs a finalized GPU engine");
  if (s < 0 || (s > 0 && (s % part.granularity || s > part.max_split())))
    return fail(NOVA_E_PARTITION, "split must be 0 or a multiple of the granularity <= max split");
  if (stage < 0 || stage > 2 || iters < 1 || B < 1 || B > cfg.max_decode_batch) return fail(NOVA_E_INVAL, "args");
  const auto& m = dims.m;
  if (gh * gw > cfg.max_patches || n_prompt > cfg.max_prompt || gh % m.merge || gw % m.merge)
    return fail(NOVA_E_INVAL, "shape exceeds engine maxima");
  const int ps0 = cfg.max_requests;  // profiling slots follow the user slots
  Request front;
  front.slot = ps0;
  front.gh = gh;
  front.gw = gw;
  front.n_prompt = n_prompt;
  front.gen_len = 2;
  std::vector<Request> dec(B);
  std::vector<Request*> dptr;
  std::vector<int> forced(B, -1);
  int need = 0;
  const int fpages = (front.S() + 63) / 64;
  const int dpages = (ctx + 1 + 63) / 64;
  if (ctx + 1 > max_pages_per_req * 64) return fail(NOVA_E_INVAL, "ctx exceeds max context");
  need = fpages + B * dpages;
  std::vector<int> pages;
  {
    std::lock_guard<std::mutex> g(ctl_mu);
    if ((int)free_pages.size() < need) return fail(NOVA_E_AGAIN, "not enough free KV pages to profile");
    for (int i = 0; i < need; ++i) {
      pages.push_back(free_pages.back());
      free_pages.pop_back();
    }
  }
  std::vector<int> bt((size_t)(B + 1) * max_pages_per_req, 0);
  for (int i = 0; i < fpages; ++i) bt[i] = pages[i];
  for (int b = 0; b < B; ++b) {
    dec[b].slot = ps0 + 1 + b;
    dec[b].gh = dec[b].gw = m.merge;  // one vision token, one prompt token: S = 2
    dec[b].n_prompt = 1;
    dec[b].gen_len = ctx + 2;
    dec[b].emitted = ctx - 1;  // -> cache index S + e - 1 = ctx
    for (int i = 0; i < dpages; ++i) bt[(size_t)(b + 1) * max_pages_per_req + i] = pages[fpages + b * dpages + i];
    dptr.push_back(&dec[b]);
  }
  cudaError_t e = cudaMemcpy(d_bt + (size_t)ps0 * max_pages_per_req, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaEventRecord(ev_upload[ps0], upload_stream);
  const int fsms = front_sms(s);
  cudaStream_t fs = stream_for(0, NOVA_CTX_DV, s);
  cudaStream_t ds = stream_for(1, s == 0 ? NOVA_CTX_SOLO : NOVA_CTX_DV, s == 0 ? part.total : s);
  const int dsms = dec_sms(s == 0 ? NOVA_CTX_SOLO : NOVA_CTX_DV, s == 0 ? part.total : s);
  cudaEvent_t a, b, c, d;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventCreate(&c);
  cudaEventCreate(&d);
  auto run_front = [&](cudaStream_t st) {
    return stage == 0 ? run_encode(&front, st, fsms) : run_prefill(&front, st, fsms);
  };
  if (e == cudaSuccess && !corun) {
    cudaStream_t st = stage == 2 ? ds : fs;
    for (int it = 0; it <= iters && e == cudaSuccess; ++it) {  // iteration 0 = warm-up
      if (it == 1) e = cudaEventRecord(a, st);
      if (e == cudaSuccess) e = stage == 2 ? run_decode(dptr, forced, st, dsms) : run_front(st);
    }
    if (e == cudaSuccess) e = cudaEventRecord(b, st);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    float ms = 0;
    if (e == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    out[0] = ms / iters;
    out[1] = 0;
  } else if (e == cudaSuccess) {
    if (stage == 2) e = cudaErrorInvalidValue;
    double fsum = 0, dsum = 0;
    int dn = 0;
    for (int it = 0; it <= iters && e == cudaSuccess; ++it) {
      e = run_decode(dptr, forced, ds, dsms);  // warm decode on its partition
      if (e == cudaSuccess) e = cudaStreamSynchronize(ds);
      if (e == cudaSuccess) e = cudaEventRecord(a, fs);
      if (e == cudaSuccess) e = run_front(fs);
      if (e == cudaSuccess) e = cudaEventRecord(b, fs);
      if (e != cudaSuccess) break;
      int n = 0;
      e = cudaEventRecord(c, ds);
      while (e == cudaSuccess && n < 100000) {
        e = run_decode(dptr, forced, ds, dsms);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ds);
        ++n;
        if (cudaEventQuery(b) == cudaSuccess) break;
      }
      if (e == cudaSuccess) e = cudaEventRecord(d, ds);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      float fm = 0, dm = 0;
      cudaEventElapsedTime(&fm, a, b);
      cudaEventElapsedTime(&dm, c, d);
      if (it > 0) {
        fsum += fm;
        dsum += dm;
        dn += n;
      }
    }
    out[0] = fsum / iters;
    out[1] = dn ? dsum / dn : 0;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaEventDestroy(c);
  cudaEventDestroy(d);
  {
    std::lock_guard<std::mutex> g(ctl_mu);
    for (int p : pages) free_pages.push_back(p);
  }
  if (e != cudaSuccess) return fail(NOVA_E_CUDA, std::string("time_pass: ") + cudaGetErrorString(e));
  return NOVA_OK;
}

}  // namespace nova
