// Probe: HBM streaming bandwidth of green-context SM partitions on this GPU, as a function of
// WHICH 8-SM groups form the partition (contiguous groups vs groups striped across the
// driver's group order).  Motivation: Nova gives decode (memory-bound) a small SM slice
// (PAPER.md P:358-365); on B200 a slice's bandwidth may be capped by the GPC <-> L2 ports it
// spans rather than by its SM count.  Prints one JSON line per configuration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_bw scripts/probe_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include <set>
#include <string>
#include <vector>

#define CK(x)                                                   \
  do {                                                          \
    CUresult r = (x);                                           \
    if (r != CUDA_SUCCESS) {                                    \
      const char* s;                                            \
      cuGetErrorString(r, &s);                                  \
      printf("FAIL %s: %s\n", #x, s);                           \
      return 1;                                                 \
    }                                                           \
  } while (0)

__global__ void smid_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
  long long c0 = clock64();
  while (clock64() - c0 < 200000) {
  }
}

// each thread streams 16-byte loads, 8 in flight, grid-strided over n uint4
__global__ void __launch_bounds__(512) read_kernel(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// strided tile pattern of a row-major [N][K] bf16 weight (K = 3584): each warp reads 64-row x
// 128-byte tiles (row stride 7168 B), 8 lanes per row, 16 B per lane, 8 loads in flight
__global__ void __launch_bounds__(512) read_tiles_kernel(const uint8_t* __restrict__ p, size_t rows, int row_bytes,
                                                         unsigned* sink) {
  unsigned acc = 0;
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarp = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t tiles_per_rowblock = row_bytes / 128;
  const size_t ntiles = (rows / 64) * tiles_per_rowblock;
  for (size_t t = warp; t < ntiles; t += nwarp) {
    const size_t rb = t / tiles_per_rowblock, kc = t % tiles_per_rowblock;
    const uint8_t* base = p + (rb * 64) * row_bytes + kc * 128;
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {  // 16 x 4 rows = 64 rows
      const int r = u * 4 + (lane >> 3);
      v[u] = __ldcs(reinterpret_cast<const uint4*>(base + (size_t)r * row_bytes + (lane & 7) * 16));
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// TMA bulk-copy streaming with a trivial consumer: the per-SM ceiling of a bulk-copy ring
// (STG stages of 8 KB, one producer lane, one consumer warp that releases slots immediately)
template <int STG>
__global__ void __launch_bounds__(64) bulk_ring_kernel(const uint8_t* __restrict__ p, size_t ntiles, unsigned* sink,
                                                       int tile_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STG * tile_bytes);
  uint64_t* empty = full + STG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STG; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto wait = [](uint64_t* b, unsigned ph) {
    unsigned ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
  };
  size_t j = 0;
  if (warp == 0 && lane == 0) {
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const int st = j % STG;
      if (j >= STG) wait(&empty[st], ((j / STG) & 1) ^ 1);
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tile_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"((unsigned)__cvta_generic_to_shared(sm + st * tile_bytes)), "l"(p + t * tile_bytes),
                   "r"(tile_bytes), "r"(bar) : "memory");
    }
  } else if (warp == 1) {
    unsigned acc = 0;
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const int st = j % STG;
      wait(&full[st], (j / STG) & 1);
      acc ^= reinterpret_cast<const unsigned*>(sm + st * tile_bytes)[lane];
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&empty[st]))
                     : "memory");
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  cudaSetDevice(0);
  cudaFree(0);
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned nb = 0;
  CK(cuDevSmResourceSplitByCount(NULL, &nb, &all, NULL, 0, 8));
  std::vector<CUdevResource> groups(nb);
  CUdevResource rem;
  CK(cuDevSmResourceSplitByCount(groups.data(), &nb, &all, &rem, 0, 8));
  int* dsm;
  cudaMalloc(&dsm, 4096 * 4);
  const size_t bytes = (size_t)2 << 30;
  uint4* buf;
  unsigned* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, bytes);
  auto make = [&](const std::vector<int>& gi, CUstream* st, int* nsm) -> int {
    std::vector<CUdevResource> v;
    for (int g : gi) v.push_back(g < (int)nb ? groups[g] : rem);
    CUdevResourceDesc d;
    CK(cuDevResourceGenerateDesc(&d, v.data(), (unsigned)v.size()));
    CUgreenCtx gc;
    CK(cuGreenCtxCreate(&gc, d, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxStreamCreate(st, gc, CU_STREAM_NON_BLOCKING, 0));
    *nsm = 0;
    for (auto& r : v) *nsm += r.sm.smCount;
    return 0;
  };
  // 1. SM ids of every group
  for (int g = 0; g <= (int)nb; ++g) {
    CUstream st;
    int n;
    if (make({g}, &st, &n)) return 1;
    smid_kernel<<<4 * n, 32, 0, (cudaStream_t)st>>>(dsm);
    cudaStreamSynchronize((cudaStream_t)st);
    std::vector<int> h(4 * n);
    cudaMemcpy(h.data(), dsm, 4 * n * 4, cudaMemcpyDeviceToHost);
    std::set<int> s(h.begin(), h.end());
    std::string ids;
    for (int x : s) ids += std::to_string(x) + ",";
    printf("{\"group\": %d, \"sms\": %d, \"smid\": [%s]}\n", g, n, ids.substr(0, ids.size() - 1).c_str());
  }
  // 2. bandwidth of partitions
  std::vector<std::pair<std::string, std::vector<int>>> cfgs = {
      {"g0", {0}}, {"g0-2", {0, 1, 2}}, {"g0,5,10", {0, 5, 10}}, {"g0,7,14", {0, 7, 14}},
      {"g0-4", {0, 1, 2, 3, 4}}, {"g0,3,6,9,12", {0, 3, 6, 9, 12}}, {"g0-9", {0, 1, 2, 3, 4, 5, 6, 7, 8, 9}},
      {"g_even", {0, 2, 4, 6, 8, 10, 12, 14}}, {"g0-7", {0, 1, 2, 3, 4, 5, 6, 7}}};
  std::vector<int> allg;
  for (int g = 0; g <= (int)nb; ++g) allg.push_back(g);
  cfgs.push_back({"all", allg});
  for (auto& c : cfgs) {
    CUstream st;
    int n;
    if (make(c.second, &st, &n)) return 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t nv = bytes / 16;
    read_kernel<<<n * 4, 512, 0, (cudaStream_t)st>>>(buf, nv, sink);
    cudaEventRecord(a, (cudaStream_t)st);
    for (int it = 0; it < 5; ++it) read_kernel<<<n * 4, 512, 0, (cudaStream_t)st>>>(buf, nv, sink);
    cudaEventRecord(b, (cudaStream_t)st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double gbs = 5.0 * bytes / (ms / 1e3) / 1e9;
    // same partition, row-major weight tile pattern
    const int rowb = 7168;
    const size_t rows = bytes / rowb / 64 * 64;
    read_tiles_kernel<<<n * 4, 512, 0, (cudaStream_t)st>>>((const uint8_t*)buf, rows, rowb, sink);
    cudaEventRecord(a, (cudaStream_t)st);
    for (int it = 0; it < 5; ++it)
      read_tiles_kernel<<<n * 4, 512, 0, (cudaStream_t)st>>>((const uint8_t*)buf, rows, rowb, sink);
    cudaEventRecord(b, (cudaStream_t)st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double gbt = 5.0 * rows * rowb / (ms / 1e3) / 1e9;
    // bulk-copy rings (~192 KB in flight per SM): CTAs/SM x stages x tile bytes
    const int vc[5][3] = {{1, 24, 8192}, {2, 12, 8192}, {4, 6, 8192}, {2, 3, 32768}, {4, 3, 16384}};
    std::string out;
    for (int v = 0; v < 5; ++v) {
      const int per = vc[v][0], stg = vc[v][1], tb = vc[v][2];
      const size_t nt = bytes / tb;
      const int smem = stg * tb + 1024;
      auto kern = stg == 24 ? bulk_ring_kernel<24> : stg == 12 ? bulk_ring_kernel<12> : stg == 6 ? bulk_ring_kernel<6>
                                                                                                    : bulk_ring_kernel<3>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEventRecord(a, (cudaStream_t)st);
      for (int it = 0; it < 5; ++it) kern<<<per * n, 64, smem, (cudaStream_t)st>>>((const uint8_t*)buf, nt, sink, tb);
      cudaEventRecord(b, (cudaStream_t)st);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      char tmp[128];
      snprintf(tmp, sizeof tmp, ", \"bulk_%dx%dx%dK\": %.1f", per, stg, tb / 1024, 5.0 * nt * tb / (ms / 1e3) / 1e9);
      out += tmp;
    }
    printf("{\"cfg\": \"%s\", \"sms\": %d, \"GB/s\": %.1f, \"tiles_GB/s\": %.1f%s}\n", c.first.c_str(), n, gbs,
           gbt, out.c_str());
  }
  printf("PROBE OK %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
