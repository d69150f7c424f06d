// Decode GEMV, TMA-streamed (SURVEY.md §8(a) row a7, §7 hard part 3: "decode must
// saturate HBM from a minority of SMs ... requires deep TMA-bulk smem pipelines").
//
//   Y[b][n] (epilogue) = sum_k X[b][k] W[n][k] + bias[n],   B <= 16 rows (bf16 X)
//
// One CTA = 64 weight rows x one K slice.  Warp 0 (one lane) streams [64 rows x 64 k]
// weight tiles (8 KB, SWIZZLE_128B) plus the matching [16 x 64] x tile through an
// 8-stage mbarrier ring with TMA; four consumer warps (one m16 tile each) run swap-AB
// mma.sync m16n8k16 from shared memory (ldmatrix on the swizzled tiles).  Up to ~160 KB
// of weights are in flight per SM with two CTAs resident, independent of how many SMs the
// decode partition owns.  Small-N shapes split K over P CTAs; partials go to a workspace
// and the last CTA of a row block (atomic ticket) adds them in split order 0..P-1, so the
// result is deterministic.  P depends only on (N, K).
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"

namespace nova {

bool g_use_tma_gemv = true;

namespace {

constexpr int RB = 64;         // weight rows per CTA
constexpr int KC = 64;         // k per stage (128 B rows -> SWIZZLE_128B)
constexpr int XR = 16;         // x rows per stage tile (batch padded to 16)
constexpr int STAGES = 8;
constexpr int W_BYTES = RB * KC * 2;   // 8 KB
constexpr int X_BYTES = XR * KC * 2;   // 2 KB
constexpr int SMEM = 1024 + STAGES * (W_BYTES + X_BYTES) + 8 * (2 * STAGES) + 64 + 4 * 32 * 2 * 4 * 4;

NOVA_DEV float silu_t(float z) { return __fdividef(z, 1.0f + __expf(-z)); }

// address of the 16-byte chunk `c16` of row `r` in a [rows][64] bf16 SWIZZLE_128B tile
NOVA_DEV uint32_t sw128(uint32_t base, int r, int c16) { return base + r * 128 + ((c16 ^ (r & 7)) << 4); }

struct TmaGemvArgs {
  void* Y;
  const bf16* bias;
  float* ws;       // [P][B][N] partials (P > 1)
  int* tickets;    // [N / RB] (P > 1), zero on entry, restored to zero by the last CTA
  int N, K, B, ldy, ks, P;
};

template <int NT, int EPI>
__global__ void __launch_bounds__(160) gemv_tma_kernel(const __grid_constant__ CUtensorMap tmW,
                                                       const __grid_constant__ CUtensorMap tmX, TmaGemvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * W_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + STAGES * X_BYTES);
  uint64_t* empty = full + STAGES;
  int* s_last = reinterpret_cast<int*>(empty + STAGES);
  float* red = reinterpret_cast<float*>(s_last + 16);  // [4 warps][NT][32][4]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x, p = blockIdx.y;
  const int r0 = rb * RB;
  const int kbeg = p * a.ks;
  const int kend = min(a.K, kbeg + a.ks);
  const int nk = (kend - kbeg + KC - 1) / KC;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer: W tiles may stream before the previous kernel ends
      const int pre = nk < STAGES ? nk : STAGES;
      for (int i = 0; i < pre; ++i) {  // PDL prologue: weights only
        mbar_arrive_expect_tx(&full[i], W_BYTES + X_BYTES);
        tma_load_2d(sW + i * W_BYTES, &tmW, &full[i], kbeg + i * KC, r0);
      }
      pdl_launch_dependents();
      pdl_wait();  // x is written by the previous kernel
      for (int i = 0; i < pre; ++i) tma_load_2d(sX + i * X_BYTES, &tmX, &full[i], kbeg + i * KC, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = pre; i < nk; ++i) {
        stage = i % STAGES;
        phase = (i / STAGES) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], W_BYTES + X_BYTES);
        tma_load_2d(sW + stage * W_BYTES, &tmW, &full[stage], kbeg + i * KC, r0);
        tma_load_2d(sX + stage * X_BYTES, &tmX, &full[stage], kbeg + i * KC, 0);
      }
    }
    return;
  }
  // ---------------- consumers: warp (1..4) owns m16 tile t = warp - 1
  pdl_launch_dependents();
  const int t = warp - 1;
  float acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
  for (int i = 0; i < nk; ++i) {
    const int stage = i % STAGES;
    mbar_wait(&full[stage], (i / STAGES) & 1);
    const uint32_t wb = smem_u32(sW + stage * W_BYTES), xb = smem_u32(sX + stage * X_BYTES);
#pragma unroll
    for (int kk = 0; kk < KC / 16; ++kk) {
      uint32_t af[4];
      ldmatrix_x4(af, sw128(wb, t * 16 + (lane & 15), kk * 2 + (lane >> 4)));
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t bfr[2];
        ldmatrix_x2(bfr, sw128(xb, nt * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)));
        mma_bf16_16816(acc[nt], af, bfr);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
  }
  // acc[nt]: c0:(row g, batch 2c) c1:(g, 2c+1) c2:(g+8, 2c) c3:(g+8, 2c+1)
  const int g = lane >> 2, c = lane & 3;
  if (a.P > 1) {  // ---------------- split-K: partials, then the last CTA of the row block reduces
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = nt * 8 + 2 * c + (j & 1);
        if (b < a.B) a.ws[((size_t)p * a.B + b) * a.N + r0 + t * 16 + g + ((j >> 1) << 3)] = acc[nt][j];
      }
    __threadfence();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 32) *s_last = (atomicAdd(&a.tickets[rb], 1) == a.P - 1);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (!*s_last) return;
    __threadfence();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = nt * 8 + 2 * c + (j & 1);
        float s = 0.f;
        if (b < a.B)
          for (int q = 0; q < a.P; ++q)
            s += __ldcg(&a.ws[((size_t)q * a.B + b) * a.N + r0 + t * 16 + g + ((j >> 1) << 3)]);
        acc[nt][j] = s;
      }
    if (threadIdx.x == 32) a.tickets[rb] = 0;
  }
  if constexpr (EPI == EPI_BF16_SILUMUL) {  // rows [32u, 32u+16) gate, [32u+16, 32u+32) up
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[((t * NT + nt) * 32 + lane) * 4 + j] = acc[nt][j];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (t & 1) return;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = nt * 8 + 2 * c + (j & 1);
        if (b >= a.B) continue;
        const float up = red[(((t + 1) * NT + nt) * 32 + lane) * 4 + j];
        const int n = r0 / 2 + (t / 2) * 16 + g + ((j >> 1) << 3);
        reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + n] = __float2bfloat16_rn(silu_t(acc[nt][j]) * up);
      }
  } else {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = nt * 8 + 2 * c + (j & 1);
        if (b >= a.B) continue;
        const int n = r0 + t * 16 + g + ((j >> 1) << 3);
        float v = acc[nt][j];
        if (a.bias != nullptr) v += __bfloat162float(a.bias[n]);
        if constexpr (EPI == EPI_BF16) {
          reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + n] = __float2bfloat16_rn(v);
        } else if constexpr (EPI == EPI_F32_RESID) {
          reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + n] += v;
        } else {
          reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + n] = v;
        }
      }
  }
}

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool encode(CUtensorMap* m, const void* ptr, int rows, int cols, int ld, int box_rows) {
  static PFN_enc enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_enc>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// weight tensor maps are reused every decode iteration: cache by (pointer, N, K)
std::mutex g_map_mu;
std::unordered_map<uint64_t, CUtensorMap>* g_maps = nullptr;

bool weight_map(CUtensorMap* m, const bf16* W, int N, int K) {
  const uint64_t key = reinterpret_cast<uint64_t>(W) ^ ((uint64_t)N << 48) ^ ((uint64_t)K << 32);
  std::lock_guard<std::mutex> g(g_map_mu);
  if (!g_maps) g_maps = new std::unordered_map<uint64_t, CUtensorMap>();
  auto it = g_maps->find(key);
  if (it != g_maps->end()) {
    *m = it->second;
    return true;
  }
  if (!encode(m, W, N, K, K, RB)) return false;
  (*g_maps)[key] = *m;
  return true;
}

template <int NT, int EPI>
cudaError_t launch(const CUtensorMap& mw, const CUtensorMap& mx, const TmaGemvArgs& a, cudaStream_t s) {
  auto kern = gemv_tma_kernel<NT, EPI>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    set = true;
  }
  return launch_k(kern, dim3(a.N / RB, a.P), dim3(160), SMEM, s, true, mw, mx, a);
}

}  // namespace

// Split factor from the shape only: aim at ~2 CTAs per SM of the whole GPU, >= 4 k-stages each.
int gemv_tma_splits(int N, int K) {
  const int blocks = N / RB;
  int P = (2 * 148 + blocks - 1) / blocks;
  const int maxp = K / (4 * KC);
  if (P > maxp) P = maxp;
  if (P < 1) P = 1;
  const int ks = ((K + P - 1) / P + KC - 1) / KC * KC;
  return (K + ks - 1) / ks;
}

cudaError_t gemv_tma(const bf16* X, int ldx, const bf16* W, int N, int K, void* Y, int ldy, const bf16* bias, int B,
                     int epi, float* ws, int* tickets, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (B > 16 || N % RB || K % KC || ldx % 8) return cudaErrorInvalidValue;
  CUtensorMap mw, mx;
  if (!weight_map(&mw, W, N, K) || !encode(&mx, X, B, K, ldx, XR)) return cudaErrorInvalidValue;
  const int P = gemv_tma_splits(N, K);
  const int ks = ((K + P - 1) / P + KC - 1) / KC * KC;
  if (P > 1 && (!ws || !tickets)) return cudaErrorInvalidValue;
  TmaGemvArgs a{Y, bias, ws, tickets, N, K, B, ldy, ks, P};
  const bool two = B > 8;
  switch (epi) {
    case EPI_BF16: return two ? launch<2, EPI_BF16>(mw, mx, a, s) : launch<1, EPI_BF16>(mw, mx, a, s);
    case EPI_BF16_SILUMUL:
      return two ? launch<2, EPI_BF16_SILUMUL>(mw, mx, a, s) : launch<1, EPI_BF16_SILUMUL>(mw, mx, a, s);
    case EPI_F32_RESID: return two ? launch<2, EPI_F32_RESID>(mw, mx, a, s) : launch<1, EPI_F32_RESID>(mw, mx, a, s);
    case EPI_F32_STORE: return two ? launch<2, EPI_F32_STORE>(mw, mx, a, s) : launch<1, EPI_F32_STORE>(mw, mx, a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nova
