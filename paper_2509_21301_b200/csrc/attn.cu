// Attention kernels (PAPER.md P:139-141 Table resource_stage "Attention" row; the
// paper used FlashInfer on sm_86).
//
// flash_attn: ViT bidirectional MHA (a5) and LLM prefill causal GQA (a6) over a
//   fused qkv buffer, FA2-style online softmax with warp-level mma.sync
//   (m16n8k16, bf16 in / f32 accumulate).  64 query rows per CTA (16 per warp),
//   64-key K/V tiles double-buffered through cp.async.
// decode_attn: paged GQA decode attention (a7): one CTA per (request, KV head,
//   256-token chunk); the GQA group shares every K/V load; chunk partials are
//   merged by a second kernel in fixed chunk order (deterministic; the chunking
//   depends only on the context length).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace nova {
namespace {

constexpr float LOG2E = 1.4426950408889634f;
}  // namespace
bool g_decode_attn_tc = true;
namespace {

template <int HD>
struct FaCfg {
  static constexpr int BQ = 64, BKV = 64, HDP = HD + 8;
  static constexpr int SMEM = (BQ + 4 * BKV) * HDP * 2;
};

template <int HD, bool CAUSAL>
__global__ void __launch_bounds__(128) flash_attn_kernel(const bf16* __restrict__ qkv, int ld, bf16* __restrict__ out,
                                                         int ldo, int S, int H, int KV, float scale_log2) {
  using C = FaCfg<HD>;
  constexpr int HDP = C::HDP, BKV = C::BKV;
  constexpr int KT = HD / 16;  // k-steps of QK^T
  constexpr int DT = HD / 8;   // n-tiles of O
  extern __shared__ __align__(16) uint8_t fa_smem[];
  bf16* sQ = reinterpret_cast<bf16*>(fa_smem);
  bf16* sK = sQ + C::BQ * HDP;  // [2][BKV][HDP]
  bf16* sV = sK + 2 * BKV * HDP;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, c = lane & 3;
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (H / KV);
  const int q0 = qt * C::BQ;
  const bf16* qbase = qkv + (size_t)h * HD;
  const bf16* kbase = qkv + (size_t)(H + kvh) * HD;
  const bf16* vbase = qkv + (size_t)(H + KV + kvh) * HD;
  constexpr int CH = HD / 8;  // 16-byte chunks per row

  for (int i = tid; i < C::BQ * CH; i += 128) {
    const int r = i / CH, cc = i % CH;
    const int row = q0 + r;
    cp_async16(sQ + r * HDP + cc * 8, qbase + (size_t)(row < S ? row : 0) * ld + cc * 8, row < S);
  }
  auto load_kv = [&](int tile, int buf) {
    const int k0 = tile * BKV;
    for (int i = tid; i < BKV * CH; i += 128) {
      const int r = i / CH, cc = i % CH;
      const int row = k0 + r;
      const size_t off = (size_t)(row < S ? row : 0) * ld + cc * 8;
      cp_async16(sK + (buf * BKV + r) * HDP + cc * 8, kbase + off, row < S);
      cp_async16(sV + (buf * BKV + r) * HDP + cc * 8, vbase + off, row < S);
    }
  };
  const int n_tiles_all = (S + BKV - 1) / BKV;
  const int n_tiles = CAUSAL ? min(n_tiles_all, (q0 + C::BQ + BKV - 1) / BKV) : n_tiles_all;
  load_kv(0, 0);
  cp_async_commit();

  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-1e30f, -1e30f}, l_r[2] = {0.f, 0.f};
  uint32_t qa[KT][4];
  const int row_a = q0 + warp * 16 + g, row_b = row_a + 8;

  for (int t = 0; t < n_tiles; ++t) {
    if (t + 1 < n_tiles) load_kv(t + 1, (t + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int kk = 0; kk < KT; ++kk)
        ldmatrix_x4(qa[kk], smem_u32(sQ + (warp * 16 + (lane & 15)) * HDP + kk * 16 + (lane >> 4) * 8));
    }
    const bf16* kt = sK + (t & 1) * BKV * HDP;
    const bf16* vt = sV + (t & 1) * BKV * HDP;
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        uint32_t b[2];
        ldmatrix_x2(b, smem_u32(kt + (nt * 8 + (lane & 7)) * HDP + kk * 16 + ((lane >> 3) & 1) * 8));
        mma_bf16_16816(s[nt], qa[kk], b);
      }
    }
    // mask + online softmax (rows row_a: s[.][0..1], row_b: s[.][2..3])
    const int k0 = t * BKV;
    float mx[2] = {-1e30f, -1e30f};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int key = k0 + nt * 8 + 2 * c + (j & 1);
        const int row = (j < 2) ? row_a : row_b;
        bool valid = key < S;
        if (CAUSAL) valid = valid && key <= row;
        const float v = valid ? s[nt][j] * scale_log2 : -1e30f;
        s[nt][j] = v;
        mx[j >> 1] = fmaxf(mx[j >> 1], v);
      }
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r]);
      corr[r] = exp2f(m_r[r] - mn);
      m_r[r] = mn;
    }
    float ls[2] = {0.f, 0.f};
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - m_r[0]), p1 = exp2f(s[nt][1] - m_r[0]);
      const float p2 = exp2f(s[nt][2] - m_r[1]), p3 = exp2f(s[nt][3] - m_r[1]);
      ls[0] += p0 + p1;
      ls[1] += p2 + p3;
      const int kk = nt >> 1, hi = nt & 1;
      pa[kk][hi * 2 + 0] = pack_bf16(p0, p1);
      pa[kk][hi * 2 + 1] = pack_bf16(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_r[r] = l_r[r] * corr[r] + ls[r];
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      o[dt][0] *= corr[0];
      o[dt][1] *= corr[0];
      o[dt][2] *= corr[1];
      o[dt][3] *= corr[1];
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // A fragment order a0:(g, k0-7) a1:(g+8, k0-7) a2:(g, k8-15) a3:(g+8, k8-15)
      const uint32_t a[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        uint32_t b[2];
        ldmatrix_x2_trans(b, smem_u32(vt + (kk * 16 + (lane & 15)) * HDP + dt * 8));
        mma_bf16_16816(o[dt], a, b);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
#pragma unroll
  for (int r = 0; r < 2; ++r) l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  const float inv_a = 1.f / l_r[0], inv_b = 1.f / l_r[1];
#pragma unroll
  for (int dt = 0; dt < DT; ++dt) {
    const int col = h * HD + dt * 8 + 2 * c;
    if (row_a < S)
      *reinterpret_cast<uint32_t*>(out + (size_t)row_a * ldo + col) = pack_bf16(o[dt][0] * inv_a, o[dt][1] * inv_a);
    if (row_b < S)
      *reinterpret_cast<uint32_t*>(out + (size_t)row_b * ldo + col) = pack_bf16(o[dt][2] * inv_b, o[dt][3] * inv_b);
  }
}

template <int HD>
cudaError_t fa_launch(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, int causal, cudaStream_t s) {
  const float sl2 = LOG2E / sqrtf((float)HD);
  dim3 grid((S + 63) / 64, H), block(128);
  const int smem = FaCfg<HD>::SMEM;
  count_launch();
  if (causal) {
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(flash_attn_kernel<HD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      set = true;
    }
    flash_attn_kernel<HD, true><<<grid, block, smem, s>>>(qkv, ld, out, ldo, S, H, KV, sl2);
  } else {
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(flash_attn_kernel<HD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      set = true;
    }
    flash_attn_kernel<HD, false><<<grid, block, smem, s>>>(qkv, ld, out, ldo, S, H, KV, sl2);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- chunked-prefill attention
// CHUNK mode (the paper's chunked-prefill baseline): the C query rows of one prefill chunk
// (cache indices c0 .. c0 + C - 1 of request `slot`, already appended) attend to every cached key
// j <= their own index -- the prefix of earlier chunks and the causal part of the chunk -- read
// straight from the paged pool: a 64-key tile is one KV page (bt[slot][tile]).  Same online-softmax
// structure as flash_attn_kernel (64 query rows x one query head per CTA, mma.sync m16n8k16).
template <int HD>
__global__ void __launch_bounds__(128) chunk_attn_kernel(const bf16* __restrict__ qkv, int ld, bf16* __restrict__ out,
                                                         int ldo, int C, int c0, int H, int KV,
                                                         const bf16* __restrict__ pool, int layer, int n_pages,
                                                         const int* __restrict__ btr, float scale_log2) {
  using Cf = FaCfg<HD>;
  constexpr int HDP = Cf::HDP, BKV = Cf::BKV;
  constexpr int KT = HD / 16, DT = HD / 8, CH = HD / 8;
  extern __shared__ __align__(16) uint8_t fa_smem[];
  bf16* sQ = reinterpret_cast<bf16*>(fa_smem);
  bf16* sK = sQ + Cf::BQ * HDP;
  bf16* sV = sK + 2 * BKV * HDP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, c = lane & 3;
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (H / KV);
  const int q0 = qt * Cf::BQ;
  const bf16* qbase = qkv + (size_t)h * HD;
  // launched with programmatic dependent launch: q and this chunk's K/V are written by the
  // preceding RoPE / KV-append kernel
  pdl_launch_dependents();
  pdl_wait();
  for (int i = tid; i < Cf::BQ * CH; i += 128) {
    const int r = i / CH, cc = i % CH;
    const int row = q0 + r;
    cp_async16(sQ + r * HDP + cc * 8, qbase + (size_t)(row < C ? row : 0) * ld + cc * 8, row < C);
  }
  const int Lk = c0 + min(C, q0 + Cf::BQ);  // keys this tile of queries can see
  const size_t page_elems = (size_t)2 * KV * 64 * HD;
  auto load_kv = [&](int tile, int buf) {
    const bf16* kb = pool + ((size_t)layer * n_pages + btr[tile]) * page_elems + (size_t)kvh * 64 * HD;
    const bf16* vb = kb + (size_t)KV * 64 * HD;
    const int k0 = tile * BKV;
    for (int i = tid; i < BKV * CH; i += 128) {
      const int r = i / CH, cc = i % CH;
      const bool ok = k0 + r < Lk;
      cp_async16(sK + (buf * BKV + r) * HDP + cc * 8, kb + (size_t)(ok ? r : 0) * HD + cc * 8, ok);
      cp_async16(sV + (buf * BKV + r) * HDP + cc * 8, vb + (size_t)(ok ? r : 0) * HD + cc * 8, ok);
    }
  };
  const int n_tiles = (Lk + BKV - 1) / BKV;
  load_kv(0, 0);
  cp_async_commit();
  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-1e30f, -1e30f}, l_r[2] = {0.f, 0.f};
  uint32_t qa[KT][4];
  const int row_a = q0 + warp * 16 + g, row_b = row_a + 8;  // chunk rows; cache index c0 + row
  for (int t = 0; t < n_tiles; ++t) {
    if (t + 1 < n_tiles) load_kv(t + 1, (t + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int kk = 0; kk < KT; ++kk)
        ldmatrix_x4(qa[kk], smem_u32(sQ + (warp * 16 + (lane & 15)) * HDP + kk * 16 + (lane >> 4) * 8));
    }
    const bf16* kt = sK + (t & 1) * BKV * HDP;
    const bf16* vt = sV + (t & 1) * BKV * HDP;
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        uint32_t b[2];
        ldmatrix_x2(b, smem_u32(kt + (nt * 8 + (lane & 7)) * HDP + kk * 16 + ((lane >> 3) & 1) * 8));
        mma_bf16_16816(s[nt], qa[kk], b);
      }
    }
    const int k0 = t * BKV;
    float mx[2] = {-1e30f, -1e30f};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int key = k0 + nt * 8 + 2 * c + (j & 1);
        const int row = (j < 2) ? row_a : row_b;
        const float v = (key <= c0 + row && key < Lk) ? s[nt][j] * scale_log2 : -1e30f;
        s[nt][j] = v;
        mx[j >> 1] = fmaxf(mx[j >> 1], v);
      }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r]);
      corr[r] = exp2f(m_r[r] - mn);
      m_r[r] = mn;
    }
    float ls[2] = {0.f, 0.f};
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - m_r[0]), p1 = exp2f(s[nt][1] - m_r[0]);
      const float p2 = exp2f(s[nt][2] - m_r[1]), p3 = exp2f(s[nt][3] - m_r[1]);
      ls[0] += p0 + p1;
      ls[1] += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_r[r] = l_r[r] * corr[r] + ls[r];
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      o[dt][0] *= corr[0];
      o[dt][1] *= corr[0];
      o[dt][2] *= corr[1];
      o[dt][3] *= corr[1];
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        uint32_t b[2];
        ldmatrix_x2_trans(b, smem_u32(vt + (kk * 16 + (lane & 15)) * HDP + dt * 8));
        mma_bf16_16816(o[dt], pa[kk], b);
      }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  const float inv_a = 1.f / l_r[0], inv_b = 1.f / l_r[1];
#pragma unroll
  for (int dt = 0; dt < DT; ++dt) {
    const int col = h * HD + dt * 8 + 2 * c;
    if (row_a < C)
      *reinterpret_cast<uint32_t*>(out + (size_t)row_a * ldo + col) = pack_bf16(o[dt][0] * inv_a, o[dt][1] * inv_a);
    if (row_b < C)
      *reinterpret_cast<uint32_t*>(out + (size_t)row_b * ldo + col) = pack_bf16(o[dt][2] * inv_b, o[dt][3] * inv_b);
  }
}

template <int HD>
cudaError_t ca_launch(const bf16* qkv, int ld, bf16* out, int ldo, int C, int c0, int H, int KV, const bf16* pool,
                      int layer, int n_pages, const int* btr, cudaStream_t s) {
  const float sl2 = LOG2E / sqrtf((float)HD);
  const int smem = FaCfg<HD>::SMEM;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(chunk_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    set = true;
  }
  return launch_k(chunk_attn_kernel<HD>, dim3((C + 63) / 64, H), dim3(128), smem, s, true, qkv, ld, out, ldo, C, c0, H,
                  KV, pool, layer, n_pages, btr, sl2);
}

// ---------------------------------------------------------------- decode attention
constexpr int DCHUNK = 256;
constexpr int MAXG = 8;  // max GQA group size

template <int HD>
__global__ void __launch_bounds__(DCHUNK) decode_attn_partial(const bf16* __restrict__ qkv, int ld,
                                                              const bf16* __restrict__ pool, int layer, int n_pages,
                                                              int H, int KV, const int* __restrict__ bt, int max_pages,
                                                              const DecodeRow* __restrict__ rows, float* __restrict__ ws,
                                                              int n_chunks, float scale_log2) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int SEG = HD / 4;            // phase 1: 4 lanes per key, SEG elements each
  const int b = blockIdx.x, kvh = blockIdx.y, ch = blockIdx.z;
  const int G = H / KV;
  const DecodeRow rr = rows[b];
  const int L = rr.ctx + 1;
  const int j0 = ch * DCHUNK;
  if (j0 >= L) return;
  const int nj = min(DCHUNK, L - j0);
  __shared__ float sq[MAXG][4][SEG + 1];  // padded: the 4 lane segments fall in different banks
  __shared__ float sp[MAXG][DCHUNK];
  __shared__ float smax[MAXG], ssum[MAXG];
  __shared__ float sred[DCHUNK / 32][MAXG][HD];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < G * HD; i += DCHUNK) {
    const int gg = i / HD, d = i % HD;
    sq[gg][d / SEG][d % SEG] = __bfloat162float(qkv[(size_t)b * ld + (size_t)(kvh * G + gg) * HD + d]) * scale_log2;
  }
  __syncthreads();
  const size_t page_stride = (size_t)2 * KV * 64 * HD;
  const bf16* lbase = pool + (size_t)layer * n_pages * page_stride;
  const int* btr = bt + (size_t)rr.slot * max_pages;
  // phase 1: scores; 8 keys per warp per pass, each key's row read by 4 lanes (coalesced)
  const int sub = lane & 3, tk = lane >> 2;
  constexpr int PASSES = DCHUNK / (8 * (DCHUNK / 32));  // 4: every key of the chunk in one unrolled sweep
  uint4 kv[PASSES][SEG / 8];
#pragma unroll
  for (int ps = 0; ps < PASSES; ++ps) {  // issue every K load of this thread first (memory-level parallelism)
    const int j = warp * 8 + tk + ps * 8 * (DCHUNK / 32);
    if (j < nj) {
      const int jj = j0 + j;
      const bf16* kp = lbase + (size_t)btr[jj >> 6] * page_stride + ((size_t)kvh * 64 + (jj & 63)) * HD + sub * SEG;
#pragma unroll
      for (int e = 0; e < SEG / 8; ++e) kv[ps][e] = *reinterpret_cast<const uint4*>(kp + 8 * e);
    }
  }
#pragma unroll
  for (int ps = 0; ps < PASSES; ++ps) {
    const int j = warp * 8 + tk + ps * 8 * (DCHUNK / 32);
    float acc[MAXG];
#pragma unroll
    for (int gg = 0; gg < MAXG; ++gg) acc[gg] = 0.f;
    if (j < nj) {
#pragma unroll
      for (int e = 0; e < SEG; e += 8) {
        const uint4 u = kv[ps][e / 8];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = unpack_bf16(w[q]);
#pragma unroll
          for (int gg = 0; gg < MAXG; ++gg)
            if (gg < G) acc[gg] += f.x * sq[gg][sub][e + 2 * q] + f.y * sq[gg][sub][e + 2 * q + 1];
        }
      }
    }
#pragma unroll
    for (int gg = 0; gg < MAXG; ++gg) {
      acc[gg] += __shfl_xor_sync(0xffffffffu, acc[gg], 1);
      acc[gg] += __shfl_xor_sync(0xffffffffu, acc[gg], 2);
    }
    if (j < nj && sub == 0) {
#pragma unroll
      for (int gg = 0; gg < MAXG; ++gg)
        if (gg < G) sp[gg][j] = acc[gg];
    }
  }
  __syncthreads();
  // phase 2: softmax statistics per head (one warp per head)
  for (int gg = warp; gg < G; gg += DCHUNK / 32) {
    float m = -1e30f;
    for (int j = lane; j < nj; j += 32) m = fmaxf(m, sp[gg][j]);
    m = warp_max(m);
    float sum = 0.f;
    for (int j = lane; j < nj; j += 32) {
      const float p = exp2f(sp[gg][j] - m);
      sp[gg][j] = p;
      sum += p;
    }
    sum = warp_sum(sum);
    if (lane == 0) {
      smax[gg] = m;
      ssum[gg] = sum;
    }
  }
  __syncthreads();
  // phase 3: o[g][d] = sum_j p[g][j] v[j][d].  Thread owns 8 columns (one 16-byte load per key)
  // of token group tg; all V loads of the chunk are issued before any FMA.
  constexpr int CG = HD / 8;           // column groups per row
  constexpr int TG = DCHUNK / CG;      // token groups
  constexpr int TPT = DCHUNK / TG;     // keys per thread (= CG)
  const int cg = tid % CG, tg = tid / CG;
  uint4 vr[TPT];
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int j = tg + u * TG;
    if (j < nj) {
      const int jj = j0 + j;
      vr[u] = *reinterpret_cast<const uint4*>(lbase + (size_t)btr[jj >> 6] * page_stride +
                                              ((size_t)(KV + kvh) * 64 + (jj & 63)) * HD + 8 * cg);
    } else {
      vr[u] = make_uint4(0, 0, 0, 0);
    }
  }
  float o[MAXG][8];
#pragma unroll
  for (int gg = 0; gg < MAXG; ++gg)
#pragma unroll
    for (int e = 0; e < 8; ++e) o[gg][e] = 0.f;
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int j = tg + u * TG;
    if (j >= nj) break;
    const uint32_t w4[4] = {vr[u].x, vr[u].y, vr[u].z, vr[u].w};
    float v[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = unpack_bf16(w4[q]);
      v[2 * q] = f.x;
      v[2 * q + 1] = f.y;
    }
#pragma unroll
    for (int gg = 0; gg < MAXG; ++gg)
      if (gg < G) {
        const float p = sp[gg][j];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[gg][e] += p * v[e];
      }
  }
  // token groups inside a warp share cg when lane % CG matches: butterfly over those lanes (fixed order)
#pragma unroll
  for (int off = CG; off < 32; off <<= 1)
#pragma unroll
    for (int gg = 0; gg < MAXG; ++gg)
#pragma unroll
      for (int e = 0; e < 8; ++e) o[gg][e] += __shfl_xor_sync(0xffffffffu, o[gg][e], off);
  if (lane < CG) {
#pragma unroll
    for (int gg = 0; gg < MAXG; ++gg)
      if (gg < G)
#pragma unroll
        for (int e = 0; e < 8; ++e) sred[warp][gg][8 * cg + e] = o[gg][e];
  }
  __syncthreads();
  const size_t wbase = ((size_t)b * H + kvh * G) * n_chunks + ch;
  for (int i = tid; i < G * HD; i += DCHUNK) {
    const int gg = i / HD, d = i % HD;
    float acc = 0.f;
#pragma unroll
    for (int t = 0; t < DCHUNK / 32; ++t) acc += sred[t][gg][d];  // fixed order over warps
    float* w = ws + (wbase + (size_t)gg * n_chunks) * (HD + 2);
    w[2 + d] = acc;
    if (d == 0) {
      w[0] = smax[gg];
      w[1] = ssum[gg];
    }
  }
}

// Tensor-core decode attention, one launch, merged through a thread-block cluster (DSMEM).
// Cluster = CL = da_cluster(KV) CTAs per (request, KV head); CTA = DA_W warps; the context is cut into 32-key
// blocks and warp w of cluster rank r owns blocks (r*DA_W + w), (r*DA_W + w) + DA_W*CL, ...  A warp
// streams its blocks through a 2-stage cp.async ring in its own smem slice (pages gathered
// through the block table), and keeps an online softmax over them: S = Q K^T with the G query
// heads sharing the KV head as the M side of mma.sync m16n8k16 (padded to 16 rows), keys the
// N side; O += P V.  The DA_W warp states are merged in smem in warp order, then rank 0 reads the
// CL CTA states from the peers' shared memory (mapa + ld.shared::cluster) and merges them in
// rank order.  Every reduction order depends only on the context length -> deterministic,
// batch- and SM-budget-invariant; no global workspace, no second kernel.
constexpr int TKW = 32;   // keys per block
// CTAs per (request, KV head): 8 when the model has <= 2 KV heads (2B: B x 2 x 4 CTAs leave most
// of a decode slice idle at the paper's small batches), else 4.  Depends on the model shape only, so
// a request's result does not depend on the batch or the partition.
inline int da_cluster(int KV) { return KV <= 2 ? 8 : 4; }
constexpr int DA_W = 6;   // warps per CTA (smem: 6 x NST stages x 17 KB): DA_W x CL block streams per (request, KV head)
// NST = K/V ring stages per warp: 2 (one CTA per SM at hd 128) or 1 (two CTAs per SM; blocks are
// gathered one at a time, from L2 after the pre-wait prefetch).  The sums do not depend on NST, so the
// launcher picks it from the partition size.
template <int HD, int NST = 2>
struct DtcCfg {
  static constexpr int HDP = HD + 8;                       // padded row (conflict-free ldmatrix)
  static constexpr int BLK = 2 * TKW * HDP * 2;            // one K+V block (bytes)
  static constexpr int Q_BYTES = 16 * HDP * 2;
  static constexpr int RING = DA_W * NST * BLK;            // DA_W warps x NST stages
  // after the ring drains: warp states [DA_W][16][HD + 2] f32, then the CTA state [16][HD + 2] f32
  static constexpr int ST_OFF = Q_BYTES + DA_W * 16 * (HD + 2) * 4;
  static constexpr int SMEM = Q_BYTES + (RING > ST_OFF - Q_BYTES + 16 * (HD + 2) * 4 ? RING : ST_OFF - Q_BYTES + 16 * (HD + 2) * 4);
};

NOVA_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
NOVA_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
NOVA_DEV float ld_dsmem_f32(uint32_t local_saddr, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_saddr), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// One 32-key block of the tensor-core decode attention for one warp: scores of the (<= 16) GQA rows
// against keys k0..k0+31 (K rows wK, V rows wV in shared memory, padded pitch HDP), online softmax
// (running max mx, sum ls per row pair) and P.V into o.  Shared by both decode-attention kernels.
template <int HD>
NOVA_DEV void da_block(const bf16* wK, const bf16* wV, int k0, int L, const uint32_t (&qa)[HD / 16][4],
                       float (&mx)[2], float (&ls)[2], float (&o)[HD / 8][4], float scale_log2, int lane) {
  constexpr int HDP = HD + 8, KT = HD / 16, DT = HD / 8;
  const int c = lane & 3;
  float sc[4][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      uint32_t bb[2];
      ldmatrix_x2(bb, smem_u32(wK + (nt * 8 + (lane & 7)) * HDP + kk * 16 + ((lane >> 3) & 1) * 8));
      mma_bf16_16816(sc[nt], qa[kk], bb);
    }
  }
  // rows g (sc[.][0..1]) and g+8 (sc[.][2..3]); keys k0 + nt*8 + 2c + (j&1)
  float bm[2] = {-1e30f, -1e30f};
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool ok = k0 + nt * 8 + 2 * c + (j & 1) < L;
      sc[nt][j] = ok ? sc[nt][j] * scale_log2 : -1e30f;
      bm[j >> 1] = fmaxf(bm[j >> 1], sc[nt][j]);
    }
  float corr[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    bm[r] = fmaxf(bm[r], __shfl_xor_sync(0xffffffffu, bm[r], 1));
    bm[r] = fmaxf(bm[r], __shfl_xor_sync(0xffffffffu, bm[r], 2));
    const float mn = fmaxf(mx[r], bm[r]);
    corr[r] = exp2f(mx[r] - mn);
    mx[r] = mn;
  }
  float ps[2] = {0.f, 0.f};
  uint32_t pa[2][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const float p0 = exp2f(sc[nt][0] - mx[0]), p1 = exp2f(sc[nt][1] - mx[0]);
    const float p2 = exp2f(sc[nt][2] - mx[1]), p3 = exp2f(sc[nt][3] - mx[1]);
    ps[0] += p0 + p1;
    ps[1] += p2 + p3;
    pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
    pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    ps[r] += __shfl_xor_sync(0xffffffffu, ps[r], 1);
    ps[r] += __shfl_xor_sync(0xffffffffu, ps[r], 2);
    ls[r] = ls[r] * corr[r] + ps[r];
  }
#pragma unroll
  for (int dt = 0; dt < DT; ++dt) {
    o[dt][0] *= corr[0];
    o[dt][1] *= corr[0];
    o[dt][2] *= corr[1];
    o[dt][3] *= corr[1];
  }
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      uint32_t bb[2];
      ldmatrix_x2_trans(bb, smem_u32(wV + (kk * 16 + (lane & 15)) * HDP + dt * 8));
      mma_bf16_16816(o[dt], pa[kk], bb);
    }
  }
}

template <int HD, int CL, int NST>
__global__ void __launch_bounds__(32 * DA_W) decode_attn_tc_kernel(const bf16* __restrict__ qkv, int ld,
                                                             const bf16* __restrict__ pool, int layer, int n_pages,
                                                             int H, int KV, const int* __restrict__ bt, int max_pages,
                                                             const DecodeRow* __restrict__ rows, bf16* __restrict__ out,
                                                             int ldo, float scale_log2) {
  using Cf = DtcCfg<HD, NST>;
  constexpr int HDP = Cf::HDP, CH = HD / 8, KT = HD / 16, DT = HD / 8, PW = HD + 2;
  extern __shared__ __align__(16) uint8_t dsm[];
  bf16* sQ = reinterpret_cast<bf16*>(dsm);
  float* sW = reinterpret_cast<float*>(dsm + Cf::Q_BYTES);  // warp states [DA_W][16][PW] (after the ring drains)
  float* sS = reinterpret_cast<float*>(dsm + Cf::ST_OFF);   // CTA state [16][PW]
  pdl_launch_dependents();
  const int rank = (int)cluster_rank();
  const int kvh = blockIdx.y, b = blockIdx.z;
  const int G = H / KV;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    // Before griddepcontrol.wait: the rows / block table (uploaded ahead of the pass's first
    // kernel) and the cached K/V of earlier tokens (written by earlier passes) are final, so warm
    // this warp's K/V rows into L2 while the qkv linear still runs.  Only the appended token
    // (written by that linear) may be stale in the prefetch; L2 is coherent, so the real loads
    // after the wait see it.
    const DecodeRow r0 = rows[b];
    const int L0 = r0.ctx + 1, nb = (L0 + TKW - 1) / TKW;
    const size_t ps = (size_t)2 * KV * 64 * HD;
    const bf16* lb = pool + (size_t)layer * n_pages * ps;
    const int* bt0 = bt + (size_t)r0.slot * max_pages;
    for (int blk = rank * DA_W + warp; blk < nb; blk += DA_W * CL) {
      const int j = blk * TKW + lane;
      if (j < L0) {
        const bf16* kp = lb + (size_t)bt0[j >> 6] * ps + ((size_t)kvh * 64 + (j & 63)) * HD;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp + 64));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp + (size_t)KV * 64 * HD));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp + (size_t)KV * 64 * HD + 64));
      }
    }
  }
  pdl_wait();
  const DecodeRow rr = rows[b];
  const int L = rr.ctx + 1;
  for (int i = tid; i < 16 * CH; i += 32 * DA_W) {  // Q rows g < G (rows >= G zero)
    const int r = i / CH, c = i % CH;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < G) v = *reinterpret_cast<const uint4*>(qkv + (size_t)b * ld + (size_t)(kvh * G + r) * HD + c * 8);
    *reinterpret_cast<uint4*>(sQ + r * HDP + c * 8) = v;
  }
  const size_t page_stride = (size_t)2 * KV * 64 * HD;
  const bf16* lbase = pool + (size_t)layer * n_pages * page_stride;
  const int* btr = bt + (size_t)rr.slot * max_pages;
  const int nblk = (L + TKW - 1) / TKW;
  const int wg = rank * DA_W + warp, wstride = DA_W * CL;
  bf16* ring = reinterpret_cast<bf16*>(dsm + Cf::Q_BYTES) + (size_t)warp * NST * (Cf::BLK / 2);
  auto issue = [&](int blk, int stage) {  // gather K and V rows of block blk into stage
    bf16* wK = ring + (size_t)stage * (Cf::BLK / 2);
    bf16* wV = wK + TKW * HDP;
    const int k0 = blk * TKW;
    for (int i = lane; i < TKW * CH; i += 32) {
      const int r = i / CH, c = i % CH;
      const int j = k0 + r;
      const bool ok = j < L;
      const int jj = ok ? j : k0;
      const bf16* kp = lbase + (size_t)btr[jj >> 6] * page_stride + ((size_t)kvh * 64 + (jj & 63)) * HD + c * 8;
      cp_async16(wK + r * HDP + c * 8, kp, ok);
      cp_async16(wV + r * HDP + c * 8, kp + (size_t)KV * 64 * HD, ok);
    }
  };
  if (wg < nblk) issue(wg, 0);
  cp_async_commit();
  __syncthreads();  // Q in smem
  const int g = lane >> 2, c = lane & 3;
  uint32_t qa[KT][4];
#pragma unroll
  for (int kk = 0; kk < KT; ++kk) ldmatrix_x4(qa[kk], smem_u32(sQ + (lane & 15) * HDP + kk * 16 + (lane >> 4) * 8));
  float mx[2] = {-1e30f, -1e30f}, ls[2] = {0.f, 0.f};
  float o[DT][4];
#pragma unroll
  for (int dt = 0; dt < DT; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
  int it = 0;
  for (int blk = wg; blk < nblk; blk += wstride, ++it) {
    const int nxt = blk + wstride;
    if constexpr (NST == 2) {
      if (nxt < nblk) issue(nxt, (it + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const bf16* wK = ring + (size_t)(NST == 2 ? (it & 1) : 0) * (Cf::BLK / 2);
    const bf16* wV = wK + TKW * HDP;
    const int k0 = blk * TKW;
    da_block<HD>(wK, wV, k0, L, qa, mx, ls, o, scale_log2, lane);
    __syncwarp();  // this stage is refilled NST blocks later
    if constexpr (NST == 1) {
      if (nxt < nblk) issue(nxt, 0);
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // every warp is done with the ring: reuse it for the warp states
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = g + 8 * r;
    if (row >= G) continue;
    float* w = sW + (warp * 16 + row) * PW;
    if (c == 0) {
      w[0] = mx[r];
      w[1] = ls[r];
    }
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      w[2 + dt * 8 + 2 * c] = o[dt][2 * r];
      w[2 + dt * 8 + 2 * c + 1] = o[dt][2 * r + 1];
    }
  }
  __syncthreads();
  // CTA state = merge of the DA_W warp states in warp order (warps without blocks: m = -1e30, l = 0)
  for (int i = tid; i < G * (HD + 2); i += 32 * DA_W) {
    const int row = i / PW, d = i % PW;
    float M = -1e30f;
#pragma unroll
    for (int w = 0; w < DA_W; ++w) M = fmaxf(M, sW[(w * 16 + row) * PW]);
    float acc = 0.f;
    if (d == 0) {
      acc = M;
    } else {
#pragma unroll
      for (int w = 0; w < DA_W; ++w) {
        const float* pw = sW + (w * 16 + row) * PW;
        acc += exp2f(pw[0] - M) * pw[d];
      }
    }
    sS[row * PW + d] = acc;
  }
  cluster_sync_all();  // CTA states visible cluster-wide
  {  // every rank merges HD / CL of the columns (the same operations per element as one merging rank)
    const uint32_t base = smem_u32(sS);
    constexpr int DW = HD / CL;
    for (int i = tid; i < G * DW; i += 32 * DA_W) {
      const int row = i / DW, d = rank * DW + i % DW;
      float m[CL], l[CL], v[CL];
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        const uint32_t a = base + (uint32_t)(row * PW) * 4u;
        m[q] = ld_dsmem_f32(a, q);
        l[q] = ld_dsmem_f32(a + 4u, q);
        v[q] = ld_dsmem_f32(a + (uint32_t)(2 + d) * 4u, q);
      }
      float M = m[0];
#pragma unroll
      for (int q = 1; q < CL; ++q) M = fmaxf(M, m[q]);
      float num = 0.f, den = 0.f;
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        const float f = exp2f(m[q] - M);
        den += f * l[q];
        num += f * v[q];
      }
      out[(size_t)b * ldo + (size_t)(kvh * G + row) * HD + d] = __float2bfloat16_rn(num / den);
    }
  }
  cluster_sync_all();  // peers keep their shared memory alive until every rank has read it
}

// The same decode attention with CLP < VC physical CTAs per (request, KV head) (session 3): the
// VC = da_cluster(KV) "virtual" CTAs of the cluster kernel above keep their block streams (virtual
// rank v, warp w: blocks v DA_W + w, + DA_W VC, ...), physical rank p runs the virtual ranks p, p + CLP,
// ... one after another through one continuous cp.async ring, and every (virtual rank, warp) state goes
// to the workspace; after a cluster barrier the CLP CTAs merge disjoint column ranges: per virtual rank
// the warp states in warp order, then the virtual ranks in rank order -- the cluster kernel's
// operations in its order, so the output is bitwise the same.  Fewer, longer CTAs for large batches
// on a small partition (one wave instead of B KV VC / (2 SMs) of them).  ws: B KV VC DA_W G (HD + 2) floats.
template <int HD, int VC, int NST>
__global__ void __launch_bounds__(32 * DA_W) decode_attn_v_kernel(const bf16* __restrict__ qkv, int ld,
                                                            const bf16* __restrict__ pool, int layer, int n_pages,
                                                            int H, int KV, const int* __restrict__ bt, int max_pages,
                                                            const DecodeRow* __restrict__ rows, bf16* __restrict__ out,
                                                            int ldo, float scale_log2, float* __restrict__ ws) {
  using Cf = DtcCfg<HD, NST>;
  constexpr int HDP = Cf::HDP, CH = HD / 8, KT = HD / 16, DT = HD / 8, PW = HD + 2;
  extern __shared__ __align__(16) uint8_t dsm[];
  bf16* sQ = reinterpret_cast<bf16*>(dsm);
  float* sML = reinterpret_cast<float*>(dsm + Cf::Q_BYTES);  // phase 2: [VC][DA_W][16] (m, l) (the ring is free)
  pdl_launch_dependents();
  const int CLP = gridDim.x;
  const int rank = (int)cluster_rank();
  const int kvh = blockIdx.y, b = blockIdx.z;
  const int G = H / KV;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {  // L2 warm-up before griddepcontrol.wait, as in the cluster kernel
    const DecodeRow r0 = rows[b];
    const int L0 = r0.ctx + 1, nb = (L0 + TKW - 1) / TKW;
    const size_t ps = (size_t)2 * KV * 64 * HD;
    const bf16* lb = pool + (size_t)layer * n_pages * ps;
    const int* bt0 = bt + (size_t)r0.slot * max_pages;
    for (int v = rank; v < VC; v += CLP)
      for (int blk = v * DA_W + warp; blk < nb; blk += DA_W * VC) {
        const int j = blk * TKW + lane;
        if (j < L0) {
          const bf16* kp = lb + (size_t)bt0[j >> 6] * ps + ((size_t)kvh * 64 + (j & 63)) * HD;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp + 64));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp + (size_t)KV * 64 * HD));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp + (size_t)KV * 64 * HD + 64));
        }
      }
  }
  pdl_wait();
  const DecodeRow rr = rows[b];
  const int L = rr.ctx + 1;
  for (int i = tid; i < 16 * CH; i += 32 * DA_W) {  // Q rows g < G (rows >= G zero)
    const int r = i / CH, c = i % CH;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < G) v = *reinterpret_cast<const uint4*>(qkv + (size_t)b * ld + (size_t)(kvh * G + r) * HD + c * 8);
    *reinterpret_cast<uint4*>(sQ + r * HDP + c * 8) = v;
  }
  const size_t page_stride = (size_t)2 * KV * 64 * HD;
  const bf16* lbase = pool + (size_t)layer * n_pages * page_stride;
  const int* btr = bt + (size_t)rr.slot * max_pages;
  const int nblk = (L + TKW - 1) / TKW;
  const int wstride = DA_W * VC;
  bf16* ring = reinterpret_cast<bf16*>(dsm + Cf::Q_BYTES) + (size_t)warp * NST * (Cf::BLK / 2);
  auto issue = [&](int blk, int stage) {
    bf16* wK = ring + (size_t)stage * (Cf::BLK / 2);
    bf16* wV = wK + TKW * HDP;
    const int k0 = blk * TKW;
    for (int i = lane; i < TKW * CH; i += 32) {
      const int r = i / CH, c = i % CH;
      const int j = k0 + r;
      const bool ok = j < L;
      const int jj = ok ? j : k0;
      const bf16* kp = lbase + (size_t)btr[jj >> 6] * page_stride + ((size_t)kvh * 64 + (jj & 63)) * HD + c * 8;
      cp_async16(wK + r * HDP + c * 8, kp, ok);
      cp_async16(wV + r * HDP + c * 8, kp + (size_t)KV * 64 * HD, ok);
    }
  };
  // this warp's blocks, virtual rank by virtual rank: (v, blk) -> the next one (v = VC: none)
  auto next = [&](int& v, int& blk) {
    blk += wstride;
    if (blk >= nblk) {
      v += CLP;
      blk = v * DA_W + warp;
      if (blk >= nblk) v = VC;  // later virtual ranks of this warp are empty too
    }
  };
  int v0 = rank, b0 = rank * DA_W + warp;
  if (b0 >= nblk) v0 = VC;
  if (v0 < VC) issue(b0, 0);
  cp_async_commit();
  __syncthreads();  // Q in smem
  const int g = lane >> 2, c = lane & 3;
  uint32_t qa[KT][4];
#pragma unroll
  for (int kk = 0; kk < KT; ++kk) ldmatrix_x4(qa[kk], smem_u32(sQ + (lane & 15) * HDP + kk * 16 + (lane >> 4) * 8));
  float* wsb = ws + (size_t)(b * KV + kvh) * VC * DA_W * G * PW;
  auto store_state = [&](int v, const float (&mx)[2], const float (&ls)[2], const float (&o)[DT][4]) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = g + 8 * r;
      if (row >= G) continue;
      float* w = wsb + ((size_t)(v * DA_W + warp) * G + row) * PW;
      if (c == 0) {
        w[0] = mx[r];
        w[1] = ls[r];
      }
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        w[2 + dt * 8 + 2 * c] = o[dt][2 * r];
        w[2 + dt * 8 + 2 * c + 1] = o[dt][2 * r + 1];
      }
    }
  };
  float mx[2] = {-1e30f, -1e30f}, ls[2] = {0.f, 0.f};
  float o[DT][4];
#pragma unroll
  for (int dt = 0; dt < DT; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
  int vs = rank;  // the virtual rank whose state is being accumulated (states of empty ones are stored too)
  int it = 0;
  for (int v = v0, blk = b0; v < VC; ++it) {
    int nv = v, nb = blk;
    next(nv, nb);
    if constexpr (NST == 2) {
      if (nv < VC) issue(nb, (it + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    while (vs < v) {  // virtual ranks finished (or empty) before this block's
      store_state(vs, mx, ls, o);
      mx[0] = mx[1] = -1e30f, ls[0] = ls[1] = 0.f;
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
      vs += CLP;
    }
    const bf16* wK = ring + (size_t)(NST == 2 ? (it & 1) : 0) * (Cf::BLK / 2);
    const bf16* wV = wK + TKW * HDP;
    da_block<HD>(wK, wV, blk * TKW, L, qa, mx, ls, o, scale_log2, lane);
    __syncwarp();
    if constexpr (NST == 1) {
      if (nv < VC) issue(nb, 0);
      cp_async_commit();
    }
    v = nv, blk = nb;
  }
  for (; vs < VC; vs += CLP) {  // the last accumulated state, then the empty ones
    store_state(vs, mx, ls, o);
    mx[0] = mx[1] = -1e30f, ls[0] = ls[1] = 0.f;
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
  }
  cp_async_wait<0>();
  __threadfence();
  __syncthreads();
  if (CLP > 1) cluster_sync_all();  // every warp state of the (request, KV head) is in ws
  // phase 2: (m, l) of all VC x DA_W states to smem, then this CTA's columns d in [d0, d1)
  for (int i = tid; i < VC * DA_W * G; i += 32 * DA_W) {
    const float* w = wsb + (size_t)i * PW;
    sML[2 * i] = __ldcg(w);
    sML[2 * i + 1] = __ldcg(w + 1);
  }
  __syncthreads();
  const int d0 = (rank * HD) / CLP, d1 = ((rank + 1) * HD) / CLP;
  for (int i = tid; i < G * (d1 - d0); i += 32 * DA_W) {
    const int row = i / (d1 - d0), d = d0 + i % (d1 - d0);
    float Mv[VC], Lv[VC], Av[VC];
#pragma unroll
    for (int q = 0; q < VC; ++q) {
      float M = -1e30f;
#pragma unroll
      for (int w = 0; w < DA_W; ++w) M = fmaxf(M, sML[2 * ((q * DA_W + w) * G + row)]);
      float accl = 0.f, acc = 0.f;
#pragma unroll
      for (int w = 0; w < DA_W; ++w) {
        const int k = (q * DA_W + w) * G + row;
        const float f = exp2f(sML[2 * k] - M);
        accl += f * sML[2 * k + 1];
        acc += f * __ldcg(wsb + (size_t)k * PW + 2 + d);
      }
      Mv[q] = M, Lv[q] = accl, Av[q] = acc;
    }
    float M = Mv[0];
#pragma unroll
    for (int q = 1; q < VC; ++q) M = fmaxf(M, Mv[q]);
    float num = 0.f, den = 0.f;
#pragma unroll
    for (int q = 0; q < VC; ++q) {
      const float f = exp2f(Mv[q] - M);
      den += f * Lv[q];
      num += f * Av[q];
    }
    out[(size_t)b * ldo + (size_t)(kvh * G + row) * HD + d] = __float2bfloat16_rn(num / den);
  }
}

template <int HD>
__global__ void decode_attn_combine(const float* __restrict__ ws, const DecodeRow* __restrict__ rows, bf16* out,
                                    int ldo, int H, int n_chunks, int keys_per_part) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const int L = rows[b].ctx + 1;
  const int nc = (L + keys_per_part - 1) / keys_per_part;
  const float* w = ws + ((size_t)b * H + h) * n_chunks * (HD + 2);
  float M = -1e30f;
  for (int c = 0; c < nc; ++c) M = fmaxf(M, w[c * (HD + 2)]);
  float num = 0.f, den = 0.f;
  for (int c = 0; c < nc; ++c) {
    const float f = exp2f(w[c * (HD + 2)] - M);
    den += f * w[c * (HD + 2) + 1];
    if (d < HD) num += f * w[c * (HD + 2) + 2 + d];
  }
  if (d < HD) out[(size_t)b * ldo + (size_t)h * HD + d] = __float2bfloat16_rn(num / den);
}

template <int HD>
cudaError_t da_launch(const bf16* qkv, int ld, bf16* out, int ldo, const bf16* pool, int layer, int n_pages, int H,
                      int KV, const int* bt, int max_pages, const DecodeRow* rows, int B, int max_ctx, float* ws,
                      int* tickets, int sms, cudaStream_t s) {
  if (H / KV > 16) return cudaErrorInvalidValue;
  const float sl2 = LOG2E / sqrtf((float)HD);
  cudaError_t e;
  if (g_decode_attn_tc) {  // tensor-core version: one cluster of da_cluster(KV) CTAs per (request, KV head)
    if (H / KV > 16) return cudaErrorInvalidValue;
    const int CLN = da_cluster(KV);
    // ring depth by the partition (never the sums): one stage and two CTAs per SM when the clusters
    // would take more than one wave of the partition at one CTA per SM (env NOVA_DA_NST forces 1 / 2)
    static const int force = getenv("NOVA_DA_NST") ? atoi(getenv("NOVA_DA_NST")) : 0;
    const int nsm = sms > 0 ? sms : 148;
    const int nst = force ? force : (CLN * KV * B > nsm ? 1 : 2);
    // more than three waves even at two CTAs per SM: CLP < CLN physical CTAs per (request, KV head) run the
    // CLN virtual ones (decode_attn_v_kernel, bitwise the same output; its workspace merge costs more
    // than one or two extra waves -- scripts/gpu_r2_dav.sh: 2B B = 16 on 16 / 24 / 32 SMs -12% / -4% / -7%,
    // 2B B = 8 on 32 SMs (two waves) +5%); env NOVA_DA_V = 0 disables, 2 = 2-stage ring
    static const int vmode = getenv("NOVA_DA_V") ? atoi(getenv("NOVA_DA_V")) : 1;
    if (vmode && ws && CLN * KV * B > 3 * 2 * nsm) {
      int clp = CLN / 2;
      while (clp > 1 && clp * KV * B > 2 * nsm) clp /= 2;
      const int vst = vmode == 2 ? 2 : 1;
      auto vk = CLN == 8 ? (vst == 1 ? decode_attn_v_kernel<HD, 8, 1> : decode_attn_v_kernel<HD, 8, 2>)
                         : (vst == 1 ? decode_attn_v_kernel<HD, 4, 1> : decode_attn_v_kernel<HD, 4, 2>);
      static bool vset = false;
      if (!vset) {
        cudaFuncSetAttribute(decode_attn_v_kernel<HD, 8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 1>::SMEM);
        cudaFuncSetAttribute(decode_attn_v_kernel<HD, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 1>::SMEM);
        cudaFuncSetAttribute(decode_attn_v_kernel<HD, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 2>::SMEM);
        cudaFuncSetAttribute(decode_attn_v_kernel<HD, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 2>::SMEM);
        vset = true;
      }
      cudaLaunchConfig_t vc = {};
      vc.gridDim = dim3(clp, KV, B);
      vc.blockDim = dim3(32 * DA_W);
      vc.dynamicSmemBytes = vst == 1 ? DtcCfg<HD, 1>::SMEM : DtcCfg<HD, 2>::SMEM;
      vc.stream = s;
      cudaLaunchAttribute va[2];
      va[0].id = cudaLaunchAttributeClusterDimension;
      va[0].val.clusterDim.x = clp;
      va[0].val.clusterDim.y = 1;
      va[0].val.clusterDim.z = 1;
      va[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      va[1].val.programmaticStreamSerializationAllowed = 1;
      vc.attrs = va;
      vc.numAttrs = g_use_pdl ? 2 : 1;
      count_launch();
      e = cudaLaunchKernelEx(&vc, vk, qkv, ld, pool, layer, n_pages, H, KV, bt, max_pages, rows, out, ldo, sl2, ws);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
    auto kern = CLN == 8 ? (nst == 1 ? decode_attn_tc_kernel<HD, 8, 1> : decode_attn_tc_kernel<HD, 8, 2>)
                         : (nst == 1 ? decode_attn_tc_kernel<HD, 4, 1> : decode_attn_tc_kernel<HD, 4, 2>);
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(decode_attn_tc_kernel<HD, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 2>::SMEM);
      cudaFuncSetAttribute(decode_attn_tc_kernel<HD, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 2>::SMEM);
      cudaFuncSetAttribute(decode_attn_tc_kernel<HD, 8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 1>::SMEM);
      cudaFuncSetAttribute(decode_attn_tc_kernel<HD, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, DtcCfg<HD, 1>::SMEM);
      set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CLN, KV, B);
    cfg.blockDim = dim3(32 * DA_W);
    cfg.dynamicSmemBytes = nst == 1 ? DtcCfg<HD, 1>::SMEM : DtcCfg<HD, 2>::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CLN;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_use_pdl ? 2 : 1;
    count_launch();
    e = cudaLaunchKernelEx(&cfg, kern, qkv, ld, pool, layer, n_pages, H, KV, bt, max_pages, rows,
                           out, ldo, sl2);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  if (H / KV > MAXG) return cudaErrorInvalidValue;
  const int n_chunks = (max_ctx + 1 + DCHUNK - 1) / DCHUNK;
  e = launch_k(decode_attn_partial<HD>, dim3(B, KV, n_chunks), dim3(DCHUNK), 0, s, true, qkv, ld, pool, layer,
               n_pages, H, KV, bt, max_pages, rows, ws, n_chunks, sl2);
  if (e != cudaSuccess) return e;
  e = launch_k(decode_attn_combine<HD>, dim3(B, H), dim3(HD), 0, s, true, ws, rows, out, ldo, H, n_chunks, DCHUNK);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

cudaError_t flash_attn(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, int hd, int causal,
                       int max_ctas, cudaStream_t s) {
  // tcgen05 persistent kernel (v3) for the bidirectional ViT attention and the causal GQA prefill
  // (longest-first snake schedule of the causal Q-tile pairs); mma.sync kernel for other head dims.
  if (hd == 80 || hd == 128) return flash_attn_tc(qkv, ld, out, ldo, S, H, KV, hd, causal, max_ctas, s);
  return flash_attn_mma(qkv, ld, out, ldo, S, H, KV, hd, causal, s);
}

cudaError_t flash_attn_mma(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, int hd, int causal,
                           cudaStream_t s) {
  if (S <= 0) return cudaSuccess;
  if (ld % 8 || H % KV) return cudaErrorInvalidValue;
  switch (hd) {
    case 16: return fa_launch<16>(qkv, ld, out, ldo, S, H, KV, causal, s);
    case 32: return fa_launch<32>(qkv, ld, out, ldo, S, H, KV, causal, s);
    case 64: return fa_launch<64>(qkv, ld, out, ldo, S, H, KV, causal, s);
    case 80: return fa_launch<80>(qkv, ld, out, ldo, S, H, KV, causal, s);
    case 128: return fa_launch<128>(qkv, ld, out, ldo, S, H, KV, causal, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t decode_attn(const bf16* qkv, int ld, bf16* out, int ldo, const bf16* pool, int layer, int n_pages, int H,
                        int KV, int hd, const int* bt, int max_pages, const DecodeRow* rows, int B, int max_ctx,
                        float* ws, int* tickets, cudaStream_t s, int sms) {
  if (B <= 0) return cudaSuccess;
  switch (hd) {
    case 32: return da_launch<32>(qkv, ld, out, ldo, pool, layer, n_pages, H, KV, bt, max_pages, rows, B, max_ctx, ws, tickets, sms, s);
    case 64: return da_launch<64>(qkv, ld, out, ldo, pool, layer, n_pages, H, KV, bt, max_pages, rows, B, max_ctx, ws, tickets, sms, s);
    case 128:
      return da_launch<128>(qkv, ld, out, ldo, pool, layer, n_pages, H, KV, bt, max_pages, rows, B, max_ctx, ws, tickets, sms, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t chunk_attn(const bf16* qkv, int ld, bf16* out, int ldo, int C, int c0, int H, int KV, int hd,
                       const bf16* kv_pool, int layer, int n_pages, const int* block_table_row, cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  if (H % KV || ld % 8) return cudaErrorInvalidValue;
  switch (hd) {
    case 32: return ca_launch<32>(qkv, ld, out, ldo, C, c0, H, KV, kv_pool, layer, n_pages, block_table_row, s);
    case 64: return ca_launch<64>(qkv, ld, out, ldo, C, c0, H, KV, kv_pool, layer, n_pages, block_table_row, s);
    case 128: return ca_launch<128>(qkv, ld, out, ldo, C, c0, H, KV, kv_pool, layer, n_pages, block_table_row, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nova
