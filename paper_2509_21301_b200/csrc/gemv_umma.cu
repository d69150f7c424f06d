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
//    flight per SM -- the bulk-copy probe's best ring (4 x 3 x 16 KB: 5.1 TB/s on a 24-SM slice);
//  * work decomposition: a 128-row block's K range is cut into P chunks of CK k-steps (CK, P from
//    the shape only) and the block's result is the LEFT FOLD of its chunk partials
//    c_0 + c_1 + ... + c_{P-1} (each c_q one TMEM accumulation).  The grid decides only who computes
//    what: each CTA takes R = blocks / G whole blocks (folded in registers) plus an equal contiguous
//    share of the remaining blocks' items (stream-K); a CTA writes its prefix fold (a share that
//    starts a block) or its single chunk partials (one that starts mid-block) to the workspace for a
//    block it shares, and the last contributor (ticket) completes the same left fold -- so the result
//    is bitwise independent of the grid (the partition) and of the batch composition.  Shared blocks
//    are processed first (their tickets hide behind the stream), whole blocks last.
#include <algorithm>
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
constexpr int NACC = 4;              // TMEM accumulators (16 columns each): MMAs run up to 3 items ahead
constexpr int TMEM_COLS = NACC * 16;

// ring shapes (same shared memory per SM): RING 0 = 3 stages x 4 CTAs per SM, 1 = 6 x 2, 2 = 12 x 1
// (hi/lo x: 3 x 3, 5 x 2, 10 x 1; with the 8 KB RoPE pair-exchange buffer of the qkv epilogue
// (XB): 3 x 3, 5 x 2, 11 x 1)
constexpr int XB_BYTES = RB * 16 * 4;  // [16 batch columns][128 rows] f32
template <int XHL, int RING, int XB = 0>
struct UCfg {
  static constexpr int ST = RING == 0 ? 3 : RING == 1 ? ((XHL || XB) ? 5 : 6) : (XHL ? 10 : XB ? 11 : 12);
  static constexpr int CPS = RING == 0 ? ((XHL || XB) ? 3 : 4) : RING == 1 ? 2 : 1;  // CTAs per SM of the partition
  static constexpr int STAGE = W_BYTES + (1 + XHL) * X_BYTES;
  static constexpr int XB_OFF = ST * STAGE + 512;
  static constexpr int SMEM = 1024 + ST * STAGE + 512 + (XB ? XB_BYTES : 0);
};

NOVA_DEV float silu_u(float z) { return __fdividef(z, 1.0f + __expf(-z)); }

// One ring stage on the tensor core, one elect for the whole stage: 4 MMAs (K = 16 each, +32 B
// along K = +2 in the descriptors' 16-byte address field) into the accumulator at tmem_d (the first
// one overwrites it when acc0 == 0), then the commit that frees the stage.  The per-MMA
// elect / collective / descriptor moves cost ~150 ns per 16 KB stage otherwise.
NOVA_DEV void umma_stage_x4(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0, uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred p, e;\n .reg .b64 a1, a2, a3, b1, b2, b3;\n"
      " setp.ne.b32 p, %4, 0;\n"
      " add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
      " add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n}\n" ::"r"(tmem_d),
      "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(smem_u32(bar))
      : "memory");
}
// hi / lo x (two B operands at b0 and b0 + lo): 8 MMAs
NOVA_DEV void umma_stage_x8(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint64_t lo, uint32_t idesc, uint32_t acc0,
                            uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred p, e;\n .reg .b64 a1, a2, a3, b1, b2, b3, c0, c1, c2, c3;\n"
      " setp.ne.b32 p, %4, 0;\n"
      " add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
      " add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
      " add.s64 c0, %2, %6;\n add.s64 c1, c0, 2;\n add.s64 c2, c0, 4;\n add.s64 c3, c0, 6;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, c0, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, c1, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, c2, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, c3, %3, 1;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n}\n" ::"r"(tmem_d),
      "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(smem_u32(bar)), "l"(lo)
      : "memory");
}

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

#ifdef NOVA_UMMA_TRACE
// per-CTA timeline (scripts/umma_trace.py; never in the product build): [cta][8] globaltimer ns
__device__ unsigned long long g_utrace[2048 * 8];
NOVA_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define UTRACE(k) (a.trace ? (void)(g_utrace[blockIdx.x * 8 + (k)] = gtime()) : (void)0)
#else
#define UTRACE(k) ((void)0)
#endif

struct UArgs {
  void* Y;
  const bf16* wblk;  // streaming layout [N/64][K/64] x 64x64 tiles
  const bf16* bias;
  float* ws;         // [blocks * P items][B][128] chunk partials / prefix folds of shared blocks
  int* tickets;      // [N / 128] (zero on entry, left zero)
  int N, K, B, ldy, CK, P, blocks, T;  // T = blocks * P items
  int R;                               // whole-block rounds: CTA c owns blocks [c R, c R + R)
  unsigned long long* keys;  // EPI_F32_ARGMAX
  const float* nhid;         // RMSNorm folded (R25): residual rows [B][K] (null = off)
  float neps;
  const bf16* ngamma;        // EPI_F32_RESID next-norm prep (R25): nxout[b][n] = bf16(Y_new[b][n] * ngamma[n])
  bf16* nxout;
  int ldnx;
  // EPI_QKV_ROPE_KV (hd = 128 = one block per head): bias + RoPE at rows[b].pos on q / k, q -> Y (bf16),
  // k / v -> the paged cache at rows[b].ctx
  const DecodeRow* rows;
  bf16* pool;
  const int* bt;
  int H, KV, layer, n_pages, max_pages;
  float log2_theta;
  int ef;  // weights with the L2 evict-first policy (env NOVA_UMMA_EF, default 1)
#ifdef NOVA_UMMA_TRACE
  int trace = 0;
#endif
};

// Work of CTA c out of G: R whole blocks [c R, c R + R), then an equal contiguous share of the
// remaining blocks' items (blocks R G .. blocks-1, P items each) -- the remainder is dealt stream-K.
struct IOrder {
  int rs, re;            // remainder items [rs, re) (global item numbers)
  int z0, nz, a0, na, m0, nrem, n, wb0, P;
  // Processing order: the remainder first -- its partial blocks at both ends (the one it ends in,
  // then the one it starts in), then its whole blocks -- and the R whole-block rounds last, so the
  // tickets and folds of shared blocks happen while the ring is still streaming and every CTA's
  // tail is a block it completes in registers.
  NOVA_DEV IOrder(int T, int blocks, int R, int G, int c, int P_) : P(P_) {
    const int base = R * G * P, trem = T - base;
    rs = base + (int)(((long long)c * trem) / G);
    re = base + (int)(((long long)(c + 1) * trem) / G);
    nrem = re - rs;
    wb0 = c * R;
    n = nrem + R * P;
    z0 = a0 = m0 = rs;
    nz = na = 0;
    (void)blocks;
    if (nrem <= 0 || rs / P == (re - 1) / P) return;
    const int bs = rs / P, be = (re - 1) / P;
    if (re % P) z0 = be * P, nz = re - z0;
    if (rs % P) a0 = rs, na = (bs + 1) * P - rs, m0 = (bs + 1) * P;
  }
  NOVA_DEV int at(int k) const {
    if (k < nrem) return k < nz ? z0 + k : k < nz + na ? a0 + (k - nz) : m0 + (k - nz - na);
    return wb0 * P + (k - nrem);
  }
};
// chunks [0, b0) of remainder block blk belong to the CTA whose share holds its chunk 0
NOVA_DEV int prefix_len(int blk, int P, int T, int R, int G) {
  const long long base = (long long)R * G * P, trem = T - base;
  const long long i0 = (long long)blk * P - base;
  const long long c = ((i0 + 1) * G - 1) / trem;  // owner of item i0
  const long long e = ((c + 1) * trem) / G;
  return (int)min(e - i0, (long long)P);
}

template <int EPI, int XHL, int RING>
__global__ void __launch_bounds__(NTHR, UCfg<XHL, RING, EPI == EPI_QKV_ROPE_KV>::CPS)
    gemv_umma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmX2, UArgs a) {
  using C = UCfg<XHL, RING, EPI == EPI_QKV_ROPE_KV>;
  constexpr int ST = C::ST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * C::STAGE);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  float* s_inv = reinterpret_cast<float*>(s_last + 3);  // [16] RMSNorm row scales (16-byte aligned)
  float* s_red = s_inv + 16;                             // [4][16] warp partials

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x, bx = blockIdx.x;
  const int kblocks = a.K / KC;
  const IOrder ord(a.T, a.blocks, a.R, G, bx, a.P);
  // k-steps [kb0, kb1) of item i
  auto item_kb = [&](int i, int& blk, int& kb0, int& kb1) {
    blk = i / a.P;
    kb0 = (i - blk * a.P) * a.CK;
    kb1 = min(kb0 + a.CK, kblocks);
  };

  if (threadIdx.x == 0) {
    UTRACE(0);
    tma_prefetch_desc(&tmX);
    if constexpr (XHL) tma_prefetch_desc(&tmX2);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NACC; ++s) {
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
    if (lane == 0) {  // ---------------- producer: the k-steps of the range's items, in processing order
      const uint64_t pol = l2_evict_first();
      auto load_w = [&](int st, int blk, int kb) {
        uint8_t* dst = smem + st * C::STAGE;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bf16* src = a.wblk + ((size_t)(2 * blk + h) * kblocks + kb) * (64 * KC);
          if (a.ef)
            bulk_load_hint(dst + h * 8192, src, 8192, &full[st], pol);
          else
            bulk_load(dst + h * 8192, src, 8192, &full[st]);
        }
      };
      auto load_x = [&](int st, int kb) {
        uint8_t* dst = smem + st * C::STAGE + W_BYTES;
        tma_load_2d(dst, &tmX, &full[st], kb * KC, 0);
        if constexpr (XHL) tma_load_2d(dst + X_BYTES, &tmX2, &full[st], kb * KC, 0);
      };
      // pass 1 (before griddepcontrol.wait): weights of the first ST stages (never written upstream)
      {
        int j = 0;
        for (int k = 0; k < ord.n && j < ST; ++k) {
          int blk, kb0, kb1;
          item_kb(ord.at(k), blk, kb0, kb1);
          for (int kb = kb0; kb < kb1 && j < ST; ++kb, ++j) {
            mbar_arrive_expect_tx(&full[j], C::STAGE);
            load_w(j, blk, kb);
          }
        }
      }
      pdl_launch_dependents();
      pdl_wait();  // x is written by the previous kernel
      UTRACE(1);
      int j = 0;
      for (int k = 0; k < ord.n; ++k) {
        int blk, kb0, kb1;
        item_kb(ord.at(k), blk, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++j) {
          const int st = j % ST;
          if (j >= ST) {
            mbar_wait(&empty[st], ((j / ST) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[st], C::STAGE);
            load_w(st, blk, kb);
          }
          load_x(st, kb);
        }
      }
      // tail: every stage released by its MMA commit before this CTA may exit
      for (int jj = j > ST ? j - ST : 0; jj < j; ++jj) mbar_wait(&empty[jj % ST], (jj / ST) & 1);
      UTRACE(3);
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, elected lane issues)
    constexpr uint32_t idesc = umma_idesc_bf16(RB, 16);
    const uint64_t da0 = umma_desc_sw128(smem_u32(smem));
    const uint64_t db0 = umma_desc_sw128(smem_u32(smem + W_BYTES));
    int j = 0;
    for (int n = 0; n < ord.n; ++n) {
      const int acc = n % NACC;
      mbar_wait(&tempty[acc], ((n / NACC) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * 16;
      int blk, kb0, kb1;
      item_kb(ord.at(n), blk, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb, ++j) {
        const int st = j % ST;
        mbar_wait(&full[st], (j / ST) & 1);
        tc_fence_after();
#ifdef NOVA_UMMA_TRACE
        if (j == 0 && lane == 0) UTRACE(2);
#endif
        const uint64_t a0 = da0 + (uint64_t)(st * (C::STAGE >> 4));
        const uint64_t b0 = db0 + (uint64_t)(st * (C::STAGE >> 4));
        if constexpr (XHL)
          umma_stage_x8(d, a0, b0, (uint64_t)(X_BYTES >> 4), idesc, kb != kb0 ? 1u : 0u, &empty[st]);
        else
          umma_stage_x4(d, a0, b0, idesc, kb != kb0 ? 1u : 0u, &empty[st]);
      }
      umma_commit_warp(&tfull[acc]);
    }
  } else {  // ---------------- epilogue: warps 2..5 -> TMEM lane quarters 2, 3, 0, 1
    pdl_launch_dependents();
    pdl_wait();  // epilogues read / write activations of the previous kernels
    const int quarter = warp & 3, et = threadIdx.x - 64;  // et: epilogue thread 0..127
    const int r = quarter * 32 + lane;                     // row within the block
    if (a.nhid) {
      // RMSNorm row scales (R25), while the first MMAs run: thread et sums float4 chunks et, et + 128,
      // ... in order, xor butterfly per warp, warps combined ((w0 + w1) + w2) + w3 -- one fixed order
      // (the loads of RJ rows x 4 chunks issued together: one L2 round trip per RJ rows, not per row)
      constexpr int RJ = C::CPS >= 3 ? 2 : 4;
      const int nch = a.K / 4, ew = et >> 5;
      for (int b0 = 0; b0 < a.B; b0 += RJ) {
        float sq[RJ];
#pragma unroll
        for (int j = 0; j < RJ; ++j) sq[j] = 0.f;
        for (int q = et; q < nch; q += 4 * 128) {
          float4 h4[RJ][4];
#pragma unroll
          for (int j = 0; j < RJ; ++j)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              h4[j][u] = (b0 + j < a.B && q + u * 128 < nch)
                             ? __ldcg(reinterpret_cast<const float4*>(a.nhid + (size_t)(b0 + j) * a.K) + q + u * 128)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < RJ; ++j)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (q + u * 128 < nch)
                sq[j] += (h4[j][u].x * h4[j][u].x + h4[j][u].y * h4[j][u].y) +
                         (h4[j][u].z * h4[j][u].z + h4[j][u].w * h4[j][u].w);
        }
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sq[j] += __shfl_xor_sync(0xffffffffu, sq[j], o);
          if (lane == 0 && b0 + j < a.B) s_red[ew * 16 + b0 + j] = sq[j];
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et < a.B)
        s_inv[et] = rsqrtf((((s_red[et] + s_red[16 + et]) + s_red[32 + et]) + s_red[48 + et]) / (float)a.K + a.neps);
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    const int B = a.B, P = a.P;
    auto slot = [&](size_t item, int b) { return a.ws + (item * B + b) * RB + r; };
    float sum[16];
    int nshared = 0;
    bool prefix = false;  // this CTA holds chunk 0 of the current block: sum = its left fold so far
    int q0 = 0;           // first chunk of the current block in this CTA's range
    int cur = -1;         // current block
    for (int n = 0; n < ord.n; ++n) {
      const int i = ord.at(n), acc = n % NACC;
      mbar_wait(&tfull[acc], (n / NACC) & 1);
      tc_fence_after();
      float v[16];
      tmem_ld16(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * 16, v);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      const int blk = i / P, q = i - blk * P;
      if (blk != cur) cur = blk, prefix = (q == 0), q0 = q;
      const bool last_here = n == ord.n - 1 || ord.at(n + 1) / P != blk;
      if (prefix) {  // c_0 + c_1 + ... in registers
#pragma unroll
        for (int b = 0; b < 16; ++b) sum[b] = q == 0 ? v[b] : sum[b] + v[b];
        if (!last_here) continue;
        if (q == P - 1) {  // the whole block in this CTA
#pragma unroll
          for (int b = 0; b < 16; ++b) v[b] = sum[b];
        } else {
#pragma unroll
          for (int b = 0; b < 16; ++b)
            if (b < B) __stcg(slot(i, b), sum[b]);
        }
      } else {  // a range that starts mid-block: single chunk partials
#pragma unroll
        for (int b = 0; b < 16; ++b)
          if (b < B) __stcg(slot(i, b), v[b]);
        if (!last_here) continue;
      }
      if (!(prefix && q == P - 1)) {  // shared block: the last contributor completes the fold
        // one release/acquire ticket per CTA: the barrier orders the epilogue threads' partial stores
        // before thread 0's atom (cumulativity), and its acquire before the other threads' loads
        const int cnt = q - q0 + 1;
        int* last_s = s_last + (nshared++ & 1);  // alternating flags: no third barrier
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          int old;
          asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(a.tickets + blk), "r"(cnt) : "memory");
          *last_s = old == P - cnt;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
#ifdef NOVA_UMMA_TRACE
        if (et == 0) UTRACE(5);
#endif
        if (!*last_s) continue;
        // c_0..c_{b0-1} folded by the prefix owner, then c_{b0}, ..., c_{P-1}: every load of a batch
        // column in flight at once, the fold in chunk order (P <= 16)
        const int b0 = prefix_len(blk, P, a.T, a.R, G);
        const size_t i0 = (size_t)blk * P;
        const size_t cs = (size_t)B * RB;  // chunk stride in the workspace
        if (B <= 2) {  // decode's usual batch: all <= 2 x 16 loads in flight, then the two folds
          const float* p0 = slot(i0, 0);
          float w0[16], w1[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const bool on = c >= b0 - 1 && c < P;
            w0[c] = on ? __ldcg(p0 + c * cs) : 0.f;
            w1[c] = (on && B == 2) ? __ldcg(p0 + RB + c * cs) : 0.f;
          }
          float f0 = 0.f, f1 = 0.f;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if (c == b0 - 1) {
              f0 = w0[c];
              f1 = w1[c];
            } else if (c >= b0 && c < P) {
              f0 += w0[c];
              f1 += w1[c];
            }
          }
#pragma unroll
          for (int b = 0; b < 16; ++b) v[b] = b == 0 ? f0 : b == 1 ? f1 : 0.f;
        } else {  // the batch columns of FD chunks per round trip (the prefix with the first), folded in order;
                  // FD = 2 where the register budget allows it (<= 2 CTAs per SM), else 1
          constexpr int FD = C::CPS >= 3 ? 1 : 2;
          for (int c = b0 - 1; c < P; c += FD) {
            float w[FD][16];
#pragma unroll
            for (int j = 0; j < FD; ++j)
#pragma unroll
              for (int b = 0; b < 16; ++b) w[j][b] = (b < B && c + j < P) ? __ldcg(slot(i0 + c + j, b)) : 0.f;
#pragma unroll
            for (int j = 0; j < FD; ++j) {
              if (c + j >= P) break;
#pragma unroll
              for (int b = 0; b < 16; ++b) v[b] = (c + j == b0 - 1) ? w[j][b] : v[b] + w[j][b];
            }
          }
        }
        if (et == 0) a.tickets[blk] = 0;
      }
      const int nrow = blk * RB + r;
      // ---- epilogues (row nrow, batch columns b < B)
      if constexpr (EPI == EPI_BF16_SILUMUL || EPI == EPI_QKV_ROPE_KV) {
        if (a.nhid) {
#pragma unroll
          for (int b = 0; b < 16; ++b) v[b] *= b < B ? s_inv[b] : 0.f;
        }
      }
      if constexpr (EPI == EPI_QKV_ROPE_KV) {
        // one block = one head (hd 128): row r pairs with r ^ 64 (rotate_half); rows 64..127 hand
        // their sums to rows 0..63 through shared memory, the owners rotate and store both
        float* xb = reinterpret_cast<float*>(smem + C::XB_OFF);
        const float bi = a.bias ? __bfloat162float(a.bias[nrow]) : 0.f;
        if (r >= 64) {
#pragma unroll
          for (int b = 0; b < 16; ++b) xb[b * RB + r] = v[b] + bi;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (r < 64) {
          const int hh = blk, hd = RB, half = 64;
          const float inv = exp2f(-(2.0f * r / hd) * a.log2_theta);
#pragma unroll
          for (int b = 0; b < 16; ++b) {
            if (b >= B) continue;
            float v1 = v[b] + bi, v2 = xb[b * RB + r + half];
            const DecodeRow rr = a.rows[b];
            if (hh < a.H + a.KV) {  // t = h = w = pos for generated text: plain RoPE at pos
              float sn, cs;
              sincosf((float)rr.pos * inv, &sn, &cs);
              const float o1 = v1 * cs - v2 * sn, o2 = v2 * cs + v1 * sn;
              v1 = o1;
              v2 = o2;
            }
            if (hh < a.H) {
              bf16* q = reinterpret_cast<bf16*>(a.Y) + (size_t)b * a.ldy + (size_t)hh * hd;
              q[r] = __float2bfloat16_rn(v1);
              q[r + half] = __float2bfloat16_rn(v2);
            } else {
              const int isv = hh >= a.H + a.KV;
              const int kvh = hh - a.H - (isv ? a.KV : 0);
              const size_t page_stride = (size_t)2 * a.KV * 64 * hd;
              bf16* pg = a.pool + ((size_t)a.layer * a.n_pages + a.bt[(size_t)rr.slot * a.max_pages + (rr.ctx >> 6)]) *
                                      page_stride;
              bf16* dst = pg + (((size_t)isv * a.KV + kvh) * 64 + (rr.ctx & 63)) * hd;
              dst[r] = __float2bfloat16_rn(v1);
              dst[r + half] = __float2bfloat16_rn(v2);
            }
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // xb is reused by the next block
      } else if constexpr (EPI == EPI_BF16_SILUMUL) {
        // rows interleave 16 gate | 16 up: lane l < 16 (gate) pairs with lane l + 16 (up)
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          const float up = __shfl_down_sync(0xffffffffu, v[b], 16);
          if (lane < 16 && b < B)
            reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + blk * (RB / 2) + quarter * 16 + lane] =
                __float2bfloat16_rn(silu_u(v[b]) * up);
        }
      } else if constexpr (EPI == EPI_F32_ARGMAX) {
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          if (b < B) reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + nrow] = v[b];
          uint32_t uu = __float_as_uint(v[b]);
          uu = (uu & 0x80000000u) ? ~uu : (uu | 0x80000000u);
          unsigned long long best = ((unsigned long long)uu << 32) | (0xFFFFFFFFu - (uint32_t)nrow);
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long ot = __shfl_xor_sync(0xffffffffu, best, o);
            best = ot > best ? ot : best;
          }
          if (lane == 0 && b < B) atomicMax(a.keys + b, best);
        }
      } else {
        const float bi = a.bias ? __bfloat162float(a.bias[nrow]) : 0.f;
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          if (b >= B) continue;
          const float y = v[b] + bi;
          if constexpr (EPI == EPI_BF16) {
            reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + nrow] = __float2bfloat16_rn(y);
          } else if constexpr (EPI == EPI_F32_RESID) {
            float* yp = reinterpret_cast<float*>(a.Y) + (size_t)b * a.ldy + nrow;
            const float hn = *yp + y;
            *yp = hn;
            if (a.nxout) a.nxout[(size_t)b * a.ldnx + nrow] = __float2bfloat16_rn(hn * __bfloat162float(a.ngamma[nrow]));
          } else {
            reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + nrow] = y;
          }
        }
      }
    }
  }
#ifdef NOVA_UMMA_TRACE
  if (threadIdx.x == 64) UTRACE(4);
  if (threadIdx.x == 0 && a.trace) g_utrace[blockIdx.x * 8 + 6] = ((unsigned long long)ord.rs << 32) | (unsigned)ord.n;
#endif
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

template <int EPI, int XHL, int RING>
cudaError_t ulaunch_r(const CUtensorMap& mx, const CUtensorMap& mx2, const UArgs& a, int sms, cudaStream_t s) {
  using C = UCfg<XHL, RING, EPI == EPI_QKV_ROPE_KV>;
  auto kern = gemv_umma_kernel<EPI, XHL, RING>;
  static bool set = false;
  {
    std::lock_guard<std::mutex> g(g_u_mu);
    if (!set) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      if (e != cudaSuccess) return e;
      set = true;
    }
  }
  // the grid (never the sums): whole blocks when there are enough of them to keep HBM busy
  // (>= NOVA_UMMA_WBMIN = 128 blocks x 48 KB in flight), the blocks x P items stream-K otherwise
  static const int wbmin = getenv("NOVA_UMMA_WBMIN") ? atoi(getenv("NOVA_UMMA_WBMIN")) : 128;
  int grid = C::CPS * (sms > 0 ? sms : 148);
  if (a.blocks < grid) grid = a.blocks >= wbmin ? a.blocks : std::min(grid, a.T);
  UArgs b = a;
  b.R = a.blocks / grid;
#ifdef NOVA_UMMA_TRACE
  static const int tn = getenv("NOVA_UMMA_TRACE_N") ? atoi(getenv("NOVA_UMMA_TRACE_N")) : -1;
  b.trace = tn < 0 || tn == a.N;
#endif
  return launch_k(kern, dim3(grid), dim3(NTHR), C::SMEM, s, true, mx, mx2, b);
}

// Ring shape by the SM budget (the grid, never the sums): on slices below 64 SMs four CTAs of 3
// stages per SM stream the most; on >= 64 SMs HBM saturates anyway and two CTAs of 6 stages
// prefetch more of each CTA's weights before griddepcontrol.wait (scripts/gpu_r2_x4.sh: 2B decode
// iteration 1.68 -> 1.51 ms on the full GPU, 24-SM slice 3.14 -> 2.99 ms with the 3 x 4 ring).
// env NOVA_UMMA_RING = 0 / 1 / 2 forces one.
template <int EPI, int XHL>
cudaError_t ulaunch(const CUtensorMap& mx, const CUtensorMap& mx2, const UArgs& a, int sms, cudaStream_t s) {
  static const int force = getenv("NOVA_UMMA_RING") ? atoi(getenv("NOVA_UMMA_RING")) : -1;
  const int ring = force >= 0 ? force : (sms <= 0 || sms >= 64) ? 1 : 0;
  if (ring == 1) return ulaunch_r<EPI, XHL, 1>(mx, mx2, a, sms, s);
  if (ring == 2) return ulaunch_r<EPI, XHL, 2>(mx, mx2, a, sms, s);
  return ulaunch_r<EPI, XHL, 0>(mx, mx2, a, sms, s);
}

}  // namespace

// Shape-only decomposition: 128-row blocks, each K range cut into P chunks of CK k-steps (the last
// may be shorter): CK >= 4 (NOVA_UMMA_CKMIN; 64 KB of weights per item -- 2 and 8 measured no
// better in decode iterations) and P <= 16 (NOVA_UMMA_PMAX: the length of the fold a
// shared block's last contributor completes), and N * P <= 2^20 (the workspace: P * B * N floats).
GemvTmaPlan gemv_umma_plan(int N, int K, int epi) {
  (void)epi;
  GemvTmaPlan pl;
  pl.RB = RB;
  const int kblocks = K / KC;
  static const int ckmin = getenv("NOVA_UMMA_CKMIN") ? atoi(getenv("NOVA_UMMA_CKMIN")) : 4;
  static const int pmax = std::min(16, getenv("NOVA_UMMA_PMAX") ? atoi(getenv("NOVA_UMMA_PMAX")) : 16);
  int ck = std::max(ckmin, (kblocks + pmax - 1) / pmax);
  while (ck < kblocks && (long long)N * ((kblocks + ck - 1) / ck) > (1LL << 20)) ++ck;
  ck = std::max(1, std::min(ck, kblocks));
  pl.P = (kblocks + ck - 1) / ck;
  pl.ks = ck * KC;
  pl.units = (N / RB) * pl.P;
  return pl;
}

bool gemv_umma_supported(int N, int K, int epi) {
  return N % RB == 0 && K % KC == 0 &&
         (epi == EPI_BF16 || epi == EPI_BF16_SILUMUL || epi == EPI_F32_RESID || epi == EPI_F32_STORE ||
          epi == EPI_F32_ARGMAX || epi == EPI_QKV_ROPE_KV);
}

cudaError_t gemv_umma(const bf16* X, int ldx, const bf16* W_blocked, int N, int K, void* Y, int ldy, const bf16* bias,
                      int B, int epi, float* ws, int* tickets, cudaStream_t s, int sms, unsigned long long* keys,
                      const bf16* X_lo, const float* norm_hid, float norm_eps, const bf16* ngamma,
                      bf16* nxout, int ldnx, const GemvAux* qa) {
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
  if (norm_hid && ((epi != EPI_BF16_SILUMUL && epi != EPI_QKV_ROPE_KV) || K % 4)) return cudaErrorInvalidValue;
  if (nxout && (epi != EPI_F32_RESID || !ngamma)) return cudaErrorInvalidValue;
  if (epi == EPI_QKV_ROPE_KV &&
      (!qa || qa->hd != RB || N != (qa->H + 2 * qa->KV) * RB || !qa->rows || !qa->pool || !qa->bt || X_lo))
    return cudaErrorInvalidValue;
  UArgs a{Y, W_blocked, bias, ws, tickets, N, K, B, ldy, pl.ks / KC, pl.P, N / RB, pl.units, 0, keys, norm_hid, norm_eps,
          ngamma, nxout, ldnx};
  static const int ef = getenv("NOVA_UMMA_EF") ? atoi(getenv("NOVA_UMMA_EF")) : 1;
  a.ef = ef;
  if (qa) {
    a.rows = qa->rows, a.pool = qa->pool, a.bt = qa->bt, a.H = qa->H, a.KV = qa->KV, a.layer = qa->layer;
    a.n_pages = qa->n_pages, a.max_pages = qa->max_pages, a.log2_theta = qa->log2_theta;
  }
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
    case EPI_QKV_ROPE_KV: return ulaunch<EPI_QKV_ROPE_KV, 0>(mx, mx2, a, sms, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nova

#ifdef NOVA_UMMA_TRACE
extern "C" int nova_debug_umma_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, nova::g_utrace, (size_t)n * 8 * 8);
}
#endif
