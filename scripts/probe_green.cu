// Probe: green-context SM partitions on this GPU (B200 validation of the executor).
// Checks (1) split granularity, (2) runtime-API kernels launched on a green-context
// stream run only on that partition's SMs, (3) primary-context allocations are
// usable there, (4) two disjoint partitions run concurrently.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <vector>
#include <set>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

__global__ void smid_kernel(int* out, unsigned long long* t, long long spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) {
    out[blockIdx.x] = s;
    long long c0 = clock64();
    while (clock64() - c0 < spin) {}
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    t[2 * blockIdx.x] = t0;
    t[2 * blockIdx.x + 1] = t1;
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("total SMs %u\n", all.sm.smCount);
  unsigned nb = 0;
  CK(cuDevSmResourceSplitByCount(NULL, &nb, &all, NULL, 0, 8));
  std::vector<CUdevResource> groups(nb);
  CUdevResource rem;
  CK(cuDevSmResourceSplitByCount(groups.data(), &nb, &all, &rem, 0, 8));
  printf("groups %u of %u SMs, remainder %u\n", nb, groups[0].sm.smCount, rem.sm.smCount);
  // decode = groups[0:3] (24 SMs), front = rest + remainder
  int k = 3;
  std::vector<CUdevResource> d(groups.begin(), groups.begin() + k), f(groups.begin() + k, groups.end());
  f.push_back(rem);
  CUdevResourceDesc dd, fd;
  CK(cuDevResourceGenerateDesc(&dd, d.data(), d.size()));
  CK(cuDevResourceGenerateDesc(&fd, f.data(), f.size()));
  CUgreenCtx gd, gf;
  CK(cuGreenCtxCreate(&gd, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gf, fd, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sd, sf;
  CK(cuGreenCtxStreamCreate(&sd, gd, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&sf, gf, CU_STREAM_NON_BLOCKING, 0));
  int *od, *of;
  unsigned long long *td, *tf;
  RK(cudaMalloc(&od, 4096 * 4));
  RK(cudaMalloc(&of, 4096 * 4));
  RK(cudaMalloc(&td, 8192 * 8));
  RK(cudaMalloc(&tf, 8192 * 8));
  const int nblk = 1000;
  long long spin = 2000000;  // ~1 ms
  smid_kernel<<<nblk, 64, 0, (cudaStream_t)sd>>>(od, td, spin);
  cudaError_t e1 = cudaGetLastError();
  smid_kernel<<<nblk, 64, 0, (cudaStream_t)sf>>>(of, tf, spin);
  cudaError_t e2 = cudaGetLastError();
  printf("launch on green streams (primary current): %s / %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
  RK(cudaDeviceSynchronize());
  std::vector<int> hd(nblk), hf(nblk);
  std::vector<unsigned long long> htd(2 * nblk), htf(2 * nblk);
  RK(cudaMemcpy(hd.data(), od, nblk * 4, cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(hf.data(), of, nblk * 4, cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(htd.data(), td, 2 * nblk * 8, cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(htf.data(), tf, 2 * nblk * 8, cudaMemcpyDeviceToHost));
  std::set<int> sdset(hd.begin(), hd.end()), sfset(hf.begin(), hf.end());
  int overlap = 0;
  for (int s : sdset) overlap += sfset.count(s);
  printf("decode partition used %zu SMs, front used %zu SMs, overlap %d\n", sdset.size(), sfset.size(), overlap);
  unsigned long long d0 = ~0ull, d1 = 0, f0 = ~0ull, f1 = 0;
  for (int i = 0; i < nblk; ++i) {
    d0 = std::min(d0, htd[2 * i]); d1 = std::max(d1, htd[2 * i + 1]);
    f0 = std::min(f0, htf[2 * i]); f1 = std::max(f1, htf[2 * i + 1]);
  }
  printf("decode span %.3f ms, front span %.3f ms, concurrent overlap %.3f ms\n", (d1 - d0) / 1e6, (f1 - f0) / 1e6,
         ((double)std::min(d1, f1) - (double)std::max(d0, f0)) / 1e6);
  // switching cost: record an event in one green stream and make another wait
  cudaEvent_t ev;
  RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  RK(cudaEventRecord(ev, (cudaStream_t)sd));
  RK(cudaStreamWaitEvent((cudaStream_t)sf, ev, 0));
  RK(cudaStreamSynchronize((cudaStream_t)sf));
  printf("cross-green-stream event wait OK\n");
  // create the full family: 17 splits x 2 ctxs, time it
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto t0 = clock();
  int made = 0;
  for (int s = 1; s < (int)nb; ++s) {
    std::vector<CUdevResource> dv(groups.begin(), groups.begin() + s), fv(groups.begin() + s, groups.end());
    fv.push_back(rem);
    CUdevResourceDesc x, y;
    CK(cuDevResourceGenerateDesc(&x, dv.data(), dv.size()));
    CK(cuDevResourceGenerateDesc(&y, fv.data(), fv.size()));
    CUgreenCtx g1, g2;
    CK(cuGreenCtxCreate(&g1, x, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&g2, y, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    made += 2;
  }
  printf("created %d more green contexts in %.1f ms (cpu)\n", made, 1000.0 * (clock() - t0) / CLOCKS_PER_SEC);
  printf("PROBE OK\n");
  return 0;
}
