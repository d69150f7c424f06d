// Decode GEMV on the 5th-generation tensor cores (DESIGN.md §5 "gemv_umma").
//
//   Y[b][n] (epilogue) = sum_k X[b][k] W[n][k] + bias[n],   B <= 16 rows (bf16 X, or f32 X as hi + lo)
//
// Decode is memory-bound and Nova runs it on a SLICE of the SMs (Eq. 5,
// P:358-365), so what matters is how many bytes one SM streams.  The mma.sync GEMV (gemv_tma.cu)
// keeps four consumer warps in the loop: each 8 KB tile costs a ldmatrix / HMMA dependency chain
// before the slot is released, and a 32-SM slice streamed ~56 GB/s per SM (84 GB/s with the math
// removed), against ~210 GB/s per SM for a bulk-copy ring with a trivial consumer
// (profiles/r01_probe_bw.jsonl, 4 CTAs x 48 KB in flight).  Here nothing but the tensor core
// touches a stage:
//  * warp 0 / lane 0: TMA producer -- per 64-k step one stage = the two 64x64 pre-swizzled weight
//    tiles of a 128-row block (A operand, M = 128, K-major SWIZZLE_128B, one 8 KB bulk copy each)
//    + the 16 x 64 activation tile (B operand, N = 16; rows >= B zero-filled by the tensor map);
//    weight tiles of the first stages are requested before griddepcontrol.wait;
//  * warp 1: one elected lane issues 4 tcgen05.mma (K = 16 each; 8 for an f32 x given as hi + lo)
//    into a TMEM accumulator [128 lanes = rows][16 columns = batch] and tcgen05.commit releases the
//    stage straight back to the producer -- the release latency is the MMA's, not a warp's;
//  * warps 2-5: epilogue, one output row per thread (tcgen05.ld 32x32b.x16), double-buffered
//    accumulators so unit i's epilogue overlaps unit i+1's MMAs;
//  * 3 stages x 16 KB of weights per CTA, 4 CTAs per SM (3 for the hi/lo lm_head) = 192 KB in
//    flight per SM;
//  * work decomposition (128-row block x K split P) from the shape only; split partials summed in
//    split order (in registers for whole-block units, through the workspace + ticket otherwise), so
//    the result is bitwise independent of the grid (the partition) and of the batch composition.
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace nova {

int g_dec_umma = getenv("NOVA_DEC_UMMA") ? atoi(getenv("NOVA_DEC_UMMA")) : 1;

namespace {

constexpr int RB = 128;              // rows per block (UMMA M)
constexpr int KC = 64;               // k per stage (one 128-byte swizzle atom row)
constexpr int W_BYTES = RB * KC * 2; // 16 KB
constexpr int X_BYTES = 16 * KC * 2; // 2 KB (UMMA N = 16)
constexpr int NTHR = 192;            // producer, MMA, 4 epilogue warps
constexpr int TMEM_COLS = 32;        // two 16-column accumulators

template <int XHL>
struct UCfg {
  static constexpr int ST = 3;
  static constexpr int CPS = XHL ? 3 : 4;                     // CTAs per SM of the partition
  static constexpr int STAGE = W_BYTES + (1 + XHL) * X_BYTES;
  static constexpr int SMEM = 1024 + ST * STAGE + 512;
};

NOVA_DEV float silu_u(float z) { return __fdividef(z, 1.0f + __expf(-z)); }

// 32 lanes x 16 consecutive f32 columns: thread t gets lane (base_lane + t), columns col..col+15
NOVA_DEV void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

struct UArgs {
  void* Y;
  const bf16* wblk;  // streaming layout [N/64][K/64] x 64x64 tiles
  const bf16* bias;
  float* ws;         // [P][B][N] split partials
  int* tickets;      // [N / 128] (zero on entry, left zero)
  int N, K, B, ldy, ks, P, blocks;
  unsigned long long* keys;  // EPI_F32_ARGMAX
  const float* nhid;         // RMSNorm folded (R25): residual rows [B][K] (null = off)
  float neps;
};

// unit i of this CTA: whole-block rounds first (split partials summed in registers), then split units
NOVA_DEV bool uunit(int i, int blocks, int P, int G, int bx, int& blk, int& p, bool& local) {
  const int R = P > 1 ? blocks / G : 0;
  if (i < R * P) {
    blk = (i / P) * G + bx;
    p = i % P;
    local = true;
    return true;
  }
  const int u = bx + (i - R * P) * G;
  if (u >= (blocks - R * G) * P) return false;
  blk = R * G + u / P;
  p = u % P;
  local = false;
  return true;
}

template <int EPI, int XHL>
__global__ void __launch_bounds__(NTHR, UCfg<XHL>::CPS)
    gemv_umma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmX2, UArgs a) {
  using C = UCfg<XHL>;
  constexpr int ST = C::ST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * C::STAGE);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  float* s_inv = reinterpret_cast<float*>(s_last + 3);  // [16] RMSNorm row scales (16-byte aligned)
  float* s_red = s_inv + 16;                             // [4][16] warp partials

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x, bx = blockIdx.x;
  const int kblocks = a.K / KC;
  auto unit_kb = [&](int p) { return (min(a.K, (p + 1) * a.ks) - p * a.ks) / KC; };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmX);
    if constexpr (XHL) tma_prefetch_desc(&tmX2);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer
      auto load_w = [&](int st, int blk, int k) {
        uint8_t* dst = smem + st * C::STAGE;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          bulk_load(dst + h * 8192, a.wblk + ((size_t)(2 * blk + h) * kblocks + k / KC) * (64 * KC), 8192, &full[st]);
      };
      auto load_x = [&](int st, int k) {
        uint8_t* dst = smem + st * C::STAGE + W_BYTES;
        tma_load_2d(dst, &tmX, &full[st], k, 0);
        if constexpr (XHL) tma_load_2d(dst + X_BYTES, &tmX2, &full[st], k, 0);
      };
      // pass 1 (before griddepcontrol.wait): weights of the first ST stages (never written upstream)
      int ui = 0, blk = 0, p = 0, kb = 0, i = 0;
      bool loc;
      bool have = uunit(ui, a.blocks, a.P, G, bx, blk, p, loc);
      int nkb = have ? unit_kb(p) : 0;
      while (have && i < ST) {
        mbar_arrive_expect_tx(&full[i], C::STAGE);
        load_w(i, blk, p * a.ks + kb * KC);
        ++i;
        if (++kb == nkb) {
          kb = 0;
          have = uunit(++ui, a.blocks, a.P, G, bx, blk, p, loc);
          nkb = have ? unit_kb(p) : 0;
        }
      }
      pdl_launch_dependents();
      pdl_wait();  // x is written by the previous kernel
      ui = 0, kb = 0;
      have = uunit(ui, a.blocks, a.P, G, bx, blk, p, loc);
      nkb = have ? unit_kb(p) : 0;
      int j = 0;
      for (; have; ++j) {
        const int st = j % ST;
        const int k = p * a.ks + kb * KC;
        if (j < ST) {
          load_x(st, k);
        } else {
          mbar_wait(&empty[st], ((j / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], C::STAGE);
          load_w(st, blk, k);
          load_x(st, k);
        }
        if (++kb == nkb) {
          kb = 0;
          have = uunit(++ui, a.blocks, a.P, G, bx, blk, p, loc);
          nkb = have ? unit_kb(p) : 0;
        }
      }
      // tail: every stage released by its MMA commit before this CTA may exit
      for (int jj = j > ST ? j - ST : 0; jj < j; ++jj) mbar_wait(&empty[jj % ST], (jj / ST) & 1);
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, elected lane issues)
    constexpr uint32_t idesc = umma_idesc_bf16(RB, 16);
    const uint64_t da0 = umma_desc_sw128(smem_u32(smem));
    const uint64_t db0 = umma_desc_sw128(smem_u32(smem + W_BYTES));
    int j = 0, acc = 0;
    uint32_t aphase = 0;
    int blk, p;
    bool loc;
    for (int ui = 0; uunit(ui, a.blocks, a.P, G, bx, blk, p, loc); ++ui) {
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * 16;
      const int nkb = unit_kb(p);
      for (int kb = 0; kb < nkb; ++kb, ++j) {
        const int st = j % ST;
        mbar_wait(&full[st], (j / ST) & 1);
        tc_fence_after();
        const uint64_t a0 = da0 + (uint64_t)(st * (C::STAGE >> 4));
        const uint64_t b0 = db0 + (uint64_t)(st * (C::STAGE >> 4));
#pragma unroll
        for (int k = 0; k < KC / 16; ++k) {  // +32 B along K inside the 128-B swizzle atom
          umma_bf16_ss_warp(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          if constexpr (XHL) umma_bf16_ss_warp(d, a0 + 2 * k, b0 + (X_BYTES >> 4) + 2 * k, idesc, 1u);
        }
        umma_commit_warp(&empty[st]);
      }
      umma_commit_warp(&tfull[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  } else {  // ---------------- epilogue: warps 2..5 -> TMEM lane quarters 2, 3, 0, 1
    pdl_launch_dependents();
    pdl_wait();  // epilogues read / write activations of the previous kernels
    const int quarter = warp & 3, et = threadIdx.x - 64;  // et: epilogue thread 0..127
    const int r = quarter * 32 + lane;                     // row within the block
    if (a.nhid) {
      // RMSNorm row scales (R25), while the first MMAs run: thread et sums float4 chunks et, et + 128,
      // ... in order, xor butterfly per warp, warps combined ((w0 + w1) + w2) + w3 -- one fixed order
      const int nch = a.K / 4, ew = et >> 5;
      for (int b = 0; b < a.B; ++b) {
        const float4* hr = reinterpret_cast<const float4*>(a.nhid + (size_t)b * a.K);
        float sq = 0.f;
        for (int q = et; q < nch; q += 128) {
          const float4 h4 = __ldcg(hr + q);
          sq += (h4.x * h4.x + h4.y * h4.y) + (h4.z * h4.z + h4.w * h4.w);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) s_red[ew * 16 + b] = sq;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et < a.B)
        s_inv[et] = rsqrtf((((s_red[et] + s_red[16 + et]) + s_red[32 + et]) + s_red[48 + et]) / (float)a.K + a.neps);
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    int acc = 0;
    uint32_t aphase = 0;
    float sum[16];
    int blk, p;
    bool local;
    for (int ui = 0; uunit(ui, a.blocks, a.P, G, bx, blk, p, local); ++ui) {
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      float v[16];
      tmem_ld16(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * 16, v);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
      const int n = blk * RB + r;
      if (local) {  // split partials summed in split order in registers (== the workspace reduction)
#pragma unroll
        for (int b = 0; b < 16; ++b) sum[b] = (p == 0 ? 0.f : sum[b]) + v[b];
        if (p < a.P - 1) continue;
#pragma unroll
        for (int b = 0; b < 16; ++b) v[b] = sum[b];
      } else if (a.P > 1) {
#pragma unroll
        for (int b = 0; b < 16; ++b)
          if (b < a.B) a.ws[((size_t)p * a.B + b) * a.N + n] = v[b];
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) *s_last = (atomicAdd(&a.tickets[blk], 1) == a.P - 1);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const bool last = *s_last;
        asm volatile("bar.sync 1, 128;" ::: "memory");  // s_last is reused by the next unit
        if (!last) continue;
        __threadfence();
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          float q8[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) q8[q] = (b < a.B && q < a.P) ? __ldcg(&a.ws[((size_t)q * a.B + b) * a.N + n]) : 0.f;
          float s = 0.f;
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q < a.P) s += q8[q];
          v[b] = s;
        }
        if (et == 0) a.tickets[blk] = 0;
      }
      // ---- epilogues (row n, batch columns b < B)
      if constexpr (EPI == EPI_BF16_SILUMUL) {
        if (a.nhid) {
#pragma unroll
          for (int b = 0; b < 16; ++b) v[b] *= b < a.B ? s_inv[b] : 0.f;
        }
        // rows interleave 16 gate | 16 up: lane l < 16 (gate) pairs with lane l + 16 (up)
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          const float up = __shfl_down_sync(0xffffffffu, v[b], 16);
          if (lane < 16 && b < a.B)
            reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + blk * (RB / 2) + quarter * 16 + lane] =
                __float2bfloat16_rn(silu_u(v[b]) * up);
        }
      } else if constexpr (EPI == EPI_F32_ARGMAX) {
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          if (b < a.B) reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + n] = v[b];
          uint32_t uu = __float_as_uint(v[b]);
          uu = (uu & 0x80000000u) ? ~uu : (uu | 0x80000000u);
          unsigned long long best = ((unsigned long long)uu << 32) | (0xFFFFFFFFu - (uint32_t)n);
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long ot = __shfl_xor_sync(0xffffffffu, best, o);
            best = ot > best ? ot : best;
          }
          if (lane == 0 && b < a.B) atomicMax(a.keys + b, best);
        }
      } else {
        const float bi = a.bias ? __bfloat162float(a.bias[n]) : 0.f;
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          if (b >= a.B) continue;
          const float y = v[b] + bi;
          if constexpr (EPI == EPI_BF16) {
            reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + n] = __float2bfloat16_rn(y);
          } else if constexpr (EPI == EPI_F32_RESID) {
            reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + n] += y;
          } else {
            reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + n] = y;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool encx(CUtensorMap* m, const void* ptr, int rows, int cols, int ld) {
  static PFN_enc enc = nullptr;
  if (!enc) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_enc>(f);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)KC, 16};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

std::mutex g_u_mu;

template <int EPI, int XHL>
cudaError_t ulaunch(const CUtensorMap& mx, const CUtensorMap& mx2, const UArgs& a, int sms, cudaStream_t s) {
  using C = UCfg<XHL>;
  auto kern = gemv_umma_kernel<EPI, XHL>;
  static bool set = false;
  {
    std::lock_guard<std::mutex> g(g_u_mu);
    if (!set) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      if (e != cudaSuccess) return e;
      set = true;
    }
  }
  int grid = C::CPS * (sms > 0 ? sms : 148);
  if (grid > a.blocks * a.P) grid = a.blocks * a.P;
  return launch_k(kern, dim3(grid), dim3(NTHR), C::SMEM, s, true, mx, mx2, a);
}

}  // namespace

// Shape-only decomposition: 128-row blocks and the smallest K split P (<= 8, chunks >= 256 k) that
// gives >= ~128 units -- one wave at the 32-SM (128-CTA) slices decode mostly runs on; bigger grids
// then take whole blocks first and split units for the rest (a split costs a partial round trip +
// ticket, so wide matrices are not split at all).  env NOVA_UMMA_UNITS overrides the 128.
GemvTmaPlan gemv_umma_plan(int N, int K, int epi) {
  GemvTmaPlan pl;
  pl.RB = RB;
  const int blocks = N / RB;
  static const int target = getenv("NOVA_UMMA_UNITS") ? atoi(getenv("NOVA_UMMA_UNITS")) : 128;
  int bestP = 1;
  static const int maxp = getenv("NOVA_UMMA_MAXP") ? atoi(getenv("NOVA_UMMA_MAXP")) : 8;
  if (epi != EPI_F32_ARGMAX) {
    for (int P = 1; P <= maxp; ++P) {
      const int ks = ((K + P - 1) / P + KC - 1) / KC * KC;
      if ((K + ks - 1) / ks != P || (P > 1 && ks < 256)) continue;
      bestP = P;
      if (blocks * P >= target) break;
    }
  }
  pl.P = bestP;
  pl.ks = ((K + bestP - 1) / bestP + KC - 1) / KC * KC;
  pl.units = blocks * bestP;
  return pl;
}

bool gemv_umma_supported(int N, int K, int epi) {
  return N % RB == 0 && K % KC == 0 &&
         (epi == EPI_BF16 || epi == EPI_BF16_SILUMUL || epi == EPI_F32_RESID || epi == EPI_F32_STORE ||
          epi == EPI_F32_ARGMAX);
}

cudaError_t gemv_umma(const bf16* X, int ldx, const bf16* W_blocked, int N, int K, void* Y, int ldy, const bf16* bias,
                      int B, int epi, float* ws, int* tickets, cudaStream_t s, int sms, unsigned long long* keys,
                      const bf16* X_lo, const float* norm_hid, float norm_eps) {
  if (B <= 0) return cudaSuccess;
  if (B > 16 || !gemv_umma_supported(N, K, epi) || ldx % 8 || !W_blocked) return cudaErrorInvalidValue;
  if (epi == EPI_F32_ARGMAX && (!keys || !X_lo)) return cudaErrorInvalidValue;
  const GemvTmaPlan pl = gemv_umma_plan(N, K, epi);
  if (pl.P > 1 && (!ws || !tickets)) return cudaErrorInvalidValue;
  CUtensorMap mx, mx2;
  if (!encx(&mx, X, B, K, ldx)) return cudaErrorInvalidValue;
  if (X_lo) {
    if (!encx(&mx2, X_lo, B, K, ldx)) return cudaErrorInvalidValue;
  } else {
    mx2 = mx;
  }
  if (norm_hid && (epi != EPI_BF16_SILUMUL || K % 4)) return cudaErrorInvalidValue;
  UArgs a{Y, W_blocked, bias, ws, tickets, N, K, B, ldy, pl.ks, pl.P, N / RB, keys, norm_hid, norm_eps};
  if (X_lo) {
    if (epi == EPI_F32_ARGMAX) return ulaunch<EPI_F32_ARGMAX, 1>(mx, mx2, a, sms, s);
    if (epi == EPI_F32_STORE) return ulaunch<EPI_F32_STORE, 1>(mx, mx2, a, sms, s);
    return cudaErrorInvalidValue;
  }
  switch (epi) {
    case EPI_BF16: return ulaunch<EPI_BF16, 0>(mx, mx2, a, sms, s);
    case EPI_BF16_SILUMUL: return ulaunch<EPI_BF16_SILUMUL, 0>(mx, mx2, a, sms, s);
    case EPI_F32_RESID: return ulaunch<EPI_F32_RESID, 0>(mx, mx2, a, sms, s);
    case EPI_F32_STORE: return ulaunch<EPI_F32_STORE, 0>(mx, mx2, a, sms, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nova
