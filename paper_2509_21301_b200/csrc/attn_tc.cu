// tcgen05 / TMEM / TMA flash attention for the vision encoder (bidirectional MHA,
// SURVEY.md §8(a) row a5; PAPER.md Table resource_stage P:139 "Attention" row, the
// part of the encode pass the paper ran with FlashInfer on sm_86) and the LLM
// prefill (causal GQA, row a6).
//
// One CTA = 128 query rows of one head.  Warp roles:
//   w0: TMA producer -- Q once, then K_j / V_j tiles (128 keys) in a 2-stage ring;
//   w1: MMA issuer  -- S_j = Q K_j^T into TMEM (double-buffered, 2 x 128 columns),
//                      O += P_j V_j into TMEM (HD columns), one thread issues;
//   w4-w7: softmax  -- thread = query row = TMEM lane: tcgen05.ld S_j, online softmax
//                      in the exp2 domain with lazy rescaling (O is corrected in TMEM
//                      only when the row max grows by > 8, i.e. 2^8), P_j as bf16 into
//                      a SWIZZLE_128B smem tile (the A operand of the second MMA).
// Operands: Q, K K-major SW128 (64-column chunks of the fused qkv buffer, straight from
// TMA); V is used as an MN-major B operand (no transpose pass); P K-major SW128.
// Deterministic: per (row, head) the key order and every reduction are fixed.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace nova {
namespace {

constexpr int FBM = 128;   // query rows per CTA
constexpr int FBN = 128;   // keys per tile
constexpr int CHUNK = 64;  // columns per SW128 chunk (128 B)
constexpr float LOG2E_F = 1.4426950408889634f;

template <int HD>
struct FtCfg {
  static constexpr int NCH = (HD + CHUNK - 1) / CHUNK;          // 64-col chunks per row of a head
  static constexpr int TILE_BYTES = NCH * FBN * CHUNK * 2;       // one 128-row Q/K/V tile
  static constexpr int P_BYTES = FBM * FBN * 2;                  // P tile (2 chunks of 64 keys)
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + TILE_BYTES;               // 2 stages
  static constexpr int V_OFF = K_OFF + 2 * TILE_BYTES;           // 2 stages
  static constexpr int P_OFF = V_OFF + 2 * TILE_BYTES;
  static constexpr int BAR_OFF = P_OFF + P_BYTES;
  static constexpr int SMEM = 1024 + BAR_OFF + 256;
  static constexpr int TMEM_COLS = 512;                          // S0, S1, O
};

// MN-major SWIZZLE_128B descriptor (V as the B operand): LBO = stride between 64-element
// N groups (chunk stride), SBO = stride between 8-row K groups (1024 B).
NOVA_DEV uint64_t umma_desc_sw128_mn(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// tcgen05.st of 32 consecutive f32 columns for this thread's lane
NOVA_DEV void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
NOVA_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 16 consecutive f32 columns
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
NOVA_DEV void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}

template <int HD, bool CAUSAL>
__global__ void __launch_bounds__(256, 1)
    fmha_tc_kernel(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, int ldo, int S, int H, int KV,
                   float scale_log2) {
  using C = FtCfg<HD>;
  constexpr int NCH = C::NCH;
  constexpr uint32_t IDESC_S = umma_idesc_bf16(FBM, FBN);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(FBM, HD) | (1u << 16);  // B (V) MN-major
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_empty = bars + 11; // [2]
  uint64_t* p_full = bars + 13;
  uint64_t* pv_done = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (H / KV);
  const int q0 = qt * FBM;
  const int n_tiles_all = (S + FBN - 1) / FBN;
  const int n_tiles = CAUSAL ? min(n_tiles_all, (q0 + FBM + FBN - 1) / FBN) : n_tiles_all;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tS[2] = {tbase, tbase + FBN};
  const uint32_t tO = tbase + 2 * FBN;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      const int qcol = h * HD, kcol = (H + kvh) * HD, vcol = (H + KV + kvh) * HD;
      mbar_arrive_expect_tx(q_full, C::TILE_BYTES);
      for (int c = 0; c < NCH; ++c)
        tma_load_2d(smem + C::Q_OFF + c * FBN * 128, &tm, q_full, qcol + c * CHUNK, q0);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const uint32_t ph = ((j >> 1) & 1) ^ 1;
        mbar_wait(&k_empty[st], ph);
        mbar_arrive_expect_tx(&k_full[st], C::TILE_BYTES);
        for (int c = 0; c < NCH; ++c)
          tma_load_2d(smem + C::K_OFF + st * C::TILE_BYTES + c * FBN * 128, &tm, &k_full[st], kcol + c * CHUNK,
                      j * FBN);
        mbar_wait(&v_empty[st], ph);
        mbar_arrive_expect_tx(&v_full[st], C::TILE_BYTES);
        for (int c = 0; c < NCH; ++c)
          tma_load_2d(smem + C::V_OFF + st * C::TILE_BYTES + c * FBN * 128, &tm, &v_full[st], vcol + c * CHUNK,
                      j * FBN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t qa = smem_u32(smem + C::Q_OFF);
      const uint32_t pa = smem_u32(smem + C::P_OFF);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        mbar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t kb = smem_u32(smem + C::K_OFF + st * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k * 16 / CHUNK) * FBN * 128 + (k * 16 % CHUNK) * 2;
          umma_bf16_ss(tS[st], umma_desc_sw128(qa + off), umma_desc_sw128(kb + off), IDESC_S, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[st]);
        umma_commit(&k_empty[st]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) issue_s(j + 1);
        const int st = j & 1;
        mbar_wait(p_full, j & 1);
        mbar_wait(&v_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = smem_u32(smem + C::V_OFF + st * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < FBN / 16; ++k) {  // 16 keys per step
          const uint32_t aoff = (k * 16 / CHUNK) * FBM * 128 + (k * 16 % CHUNK) * 2;
          umma_bf16_ss(tO, umma_desc_sw128(pa + aoff), umma_desc_sw128_mn(vb + k * 16 * 128, FBN * 128), IDESC_O,
                       (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&v_empty[st]);
        umma_commit(pv_done);
      }
    }
  } else if (warp >= 4) {  // ---------------- softmax / correction / epilogue
    const int row = (warp - 4) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int qrow = q0 + row;
    float m = -1e30f, l = 0.f;
    uint8_t* P = smem + C::P_OFF;
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      const int k0 = j * FBN;
      const bool edge = (k0 + FBN > S) || (CAUSAL && k0 + FBN > q0);
      // keys >= lim are masked (tail of the sequence; causal diagonal); interior tiles skip the test
      const int lim = CAUSAL ? min(S, qrow + 1) : S;
      // pass 1: row max
      float mx = -1e30f;
#pragma unroll
      for (int c = 0; c < FBN / 32; ++c) {
        float v[32];
        tmem_ld32(tS[st] + lane_off + c * 32, v);
        if (edge) {
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, (k0 + c * 32 + i < lim) ? v[i] : -1e30f);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
        }
      }
      const float mnew = fmaxf(m, mx * scale_log2);
      const bool need = (mnew - m) > 8.0f;
      // PV_{j-1} must be complete before P is overwritten and before O is rescaled
      if (j > 0) mbar_wait(pv_done, (j - 1) & 1);
      if (__any_sync(0xffffffffu, need) && j > 0) {
        tc_fence_after();
        const float f = need ? fast_exp2(m - mnew) : 1.0f;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + lane_off + c * 16, o);
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] *= f;
          tmem_st16(tO + lane_off + c * 16, o);
        }
        tmem_st_wait();
      }
      if (need) {
        l *= fast_exp2(m - mnew);
        m = mnew;
      }
      // pass 2: P = exp2(s*scale - m) -> bf16 -> swizzled smem
      const float nm = -m;
      float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
      for (int c = 0; c < FBN / 32; ++c) {
        float v[32];
        tmem_ld32(tS[st] + lane_off + c * 32, v);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float p0 = fast_exp2(fmaf(v[i], scale_log2, nm));
          float p1 = fast_exp2(fmaf(v[i + 1], scale_log2, nm));
          if (edge) {
            const int key = k0 + c * 32 + i;
            p0 = key < lim ? p0 : 0.f;
            p1 = key + 1 < lim ? p1 : 0.f;
          }
          ls0 += p0;
          ls1 += p1;
          pk[i / 2] = pack_bf16(p0, p1);
        }
        // 32 keys = 64 B = four 16-byte chunks of row `row` in key chunk (c / 2)
        uint8_t* base = P + (c >> 1) * FBM * 128 + row * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int jj = (c & 1) * 4 + q;
          *reinterpret_cast<uint4*>(base + ((jj ^ (row & 7)) * 16)) =
              make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      const float ls = ls0 + ls1;
      l += ls;
      tc_fence_before();
      mbar_arrive(&s_empty[st]);
      fence_proxy_async();  // generic-proxy smem writes of P -> visible to the tensor core
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 rows
    mbar_wait(pv_done, (n_tiles - 1) & 1);
    tc_fence_after();
    const float inv = 1.0f / l;
    bf16* orow = out + (size_t)qrow * ldo + (size_t)h * HD;
#pragma unroll
    for (int c = 0; c < HD / 16; ++c) {
      float o[16];
      tmem_ld16(tO + lane_off + c * 16, o);
      if (qrow < S) {
        uint4 a = make_uint4(pack_bf16(o[0] * inv, o[1] * inv), pack_bf16(o[2] * inv, o[3] * inv),
                             pack_bf16(o[4] * inv, o[5] * inv), pack_bf16(o[6] * inv, o[7] * inv));
        uint4 b = make_uint4(pack_bf16(o[8] * inv, o[9] * inv), pack_bf16(o[10] * inv, o[11] * inv),
                             pack_bf16(o[12] * inv, o[13] * inv), pack_bf16(o[14] * inv, o[15] * inv));
        reinterpret_cast<uint4*>(orow + c * 16)[0] = a;
        reinterpret_cast<uint4*>(orow + c * 16)[1] = b;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------------
// v2: two CTAs per SM.  P stays in TMEM (bf16 pairs written over the S columns already read:
// the FA4 aliasing) and the P.V product is a TS MMA (A from TMEM), so shared memory holds only
// Q, K_j, V_j (single-buffered, 96 KB) and TMEM only S|P (128 cols) + O (<= 128 cols).  The two
// CTAs on an SM interleave: one CTA's softmax runs while the other's MMAs use the tensor core.
// In-CTA order per key tile: S_j (after PV_{j-1}, issue order) -> softmax_j -> PV_j.
template <int HD>
struct Ft2Cfg {
  static constexpr int NCH = (HD + CHUNK - 1) / CHUNK;
  static constexpr int TILE_BYTES = NCH * FBN * CHUNK * 2;
  static constexpr int Q_OFF = 0, K_OFF = TILE_BYTES, V_OFF = 2 * TILE_BYTES, BAR_OFF = 3 * TILE_BYTES;
  static constexpr int SMEM = 1024 + BAR_OFF + 128;
  static constexpr int TMEM_COLS = 256;
};

NOVA_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
NOVA_DEV void tmem_st16u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

template <int HD, bool CAUSAL>
__global__ void __launch_bounds__(256, 2)
    fmha2_kernel(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, int ldo, int S, int H, int KV,
                 float scale_log2) {
  using C = Ft2Cfg<HD>;
  constexpr int NCH = C::NCH;
  constexpr uint32_t IDESC_S = umma_idesc_bf16(FBM, FBN);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(FBM, HD) | (1u << 16);  // B (V) MN-major
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t *q_full = bars + 0, *k_full = bars + 1, *k_empty = bars + 2, *v_full = bars + 3, *v_empty = bars + 4;
  uint64_t *s_full = bars + 5, *p_full = bars + 6, *o_done = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (H / KV);
  const int q0 = qt * FBM;
  const int n_tiles_all = (S + FBN - 1) / FBN;
  const int n_tiles = CAUSAL ? min(n_tiles_all, (q0 + FBM + FBN - 1) / FBN) : n_tiles_all;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], i == 6 ? 128 : 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tS = tbase, tO = tbase + FBN;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (single-buffered K and V)
      const int qcol = h * HD, kcol = (H + kvh) * HD, vcol = (H + KV + kvh) * HD;
      mbar_arrive_expect_tx(q_full, C::TILE_BYTES);
      for (int c = 0; c < NCH; ++c) tma_load_2d(smem + C::Q_OFF + c * FBN * 128, &tm, q_full, qcol + c * CHUNK, q0);
      for (int j = 0; j < n_tiles; ++j) {
        const uint32_t ph = (j & 1) ^ 1;
        mbar_wait(k_empty, ph);
        mbar_arrive_expect_tx(k_full, C::TILE_BYTES);
        for (int c = 0; c < NCH; ++c)
          tma_load_2d(smem + C::K_OFF + c * FBN * 128, &tm, k_full, kcol + c * CHUNK, j * FBN);
        mbar_wait(v_empty, ph);
        mbar_arrive_expect_tx(v_full, C::TILE_BYTES);
        for (int c = 0; c < NCH; ++c)
          tma_load_2d(smem + C::V_OFF + c * FBN * 128, &tm, v_full, vcol + c * CHUNK, j * FBN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t qa = smem_u32(smem + C::Q_OFF), kb = smem_u32(smem + C::K_OFF), vb = smem_u32(smem + C::V_OFF);
      mbar_wait(q_full, 0);
      for (int j = 0; j < n_tiles; ++j) {
        mbar_wait(k_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k * 16 / CHUNK) * FBN * 128 + (k * 16 % CHUNK) * 2;
          umma_bf16_ss(tS, umma_desc_sw128(qa + off), umma_desc_sw128(kb + off), IDESC_S, k > 0 ? 1u : 0u);
        }
        umma_commit(s_full);   // also covers PV_{j-1}: O is stable once S_j is visible
        umma_commit(k_empty);
        mbar_wait(p_full, j & 1);
        mbar_wait(v_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < FBN / 16; ++k)  // P: 16 keys = 8 packed TMEM columns per step
          umma_bf16_ts(tO, tS + k * 8, umma_desc_sw128_mn(vb + k * 16 * 128, FBN * 128), IDESC_O,
                       (j > 0 || k > 0) ? 1u : 0u);
        umma_commit(v_empty);
      }
      umma_commit(o_done);
    }
  } else if (warp >= 4) {  // ---------------- softmax / correction / epilogue
    const int row = (warp - 4) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int qrow = q0 + row;
    float m = -1e30f, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      const int k0 = j * FBN;
      const bool edge = (k0 + FBN > S) || (CAUSAL && k0 + FBN > q0);
      const int lim = CAUSAL ? min(S, qrow + 1) : S;
      float mx = -1e30f;
#pragma unroll
      for (int c = 0; c < FBN / 32; ++c) {
        float v[32];
        tmem_ld32(tS + lane_off + c * 32, v);
        if (edge) {
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, (k0 + c * 32 + i < lim) ? v[i] : -1e30f);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
        }
      }
      const float mnew = fmaxf(m, mx * scale_log2);
      const bool need = (mnew - m) > 8.0f;
      if (__any_sync(0xffffffffu, need) && j > 0) {  // lazy rescale of O in TMEM (PV_{j-1} done: see s_full)
        const float f = need ? fast_exp2(m - mnew) : 1.0f;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + lane_off + c * 16, o);
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] *= f;
          tmem_st16(tO + lane_off + c * 16, o);
        }
      }
      if (need) {
        l *= fast_exp2(m - mnew);
        m = mnew;
      }
      const float nm = -m;
      float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
      for (int c = 0; c < FBN / 32; ++c) {
        // S chunk c (cols 32c..32c+31) is re-read; P chunk c lands in cols 16c..16c+15, i.e. over
        // S columns this thread has already read (chunks <= c), so the aliasing is safe
        float sv[32];
        tmem_ld32(tS + lane_off + c * 32, sv);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float p0 = fast_exp2(fmaf(sv[i], scale_log2, nm));
          float p1 = fast_exp2(fmaf(sv[i + 1], scale_log2, nm));
          if (edge) {
            const int key = k0 + c * 32 + i;
            p0 = key < lim ? p0 : 0.f;
            p1 = key + 1 < lim ? p1 : 0.f;
          }
          ls0 += p0;
          ls1 += p1;
          pk[i / 2] = pack_bf16(p0, p1);
        }
        tmem_st16u(tS + lane_off + c * 16, pk);  // P keys 32c..32c+31 -> packed columns 16c..16c+15
      }
      l += ls0 + ls1;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 rows
    mbar_wait(o_done, 0);
    tc_fence_after();
    const float inv = 1.0f / l;
    bf16* orow = out + (size_t)qrow * ldo + (size_t)h * HD;
#pragma unroll
    for (int c = 0; c < HD / 16; ++c) {
      float o[16];
      tmem_ld16(tO + lane_off + c * 16, o);
      if (qrow < S) {
        uint4 a = make_uint4(pack_bf16(o[0] * inv, o[1] * inv), pack_bf16(o[2] * inv, o[3] * inv),
                             pack_bf16(o[4] * inv, o[5] * inv), pack_bf16(o[6] * inv, o[7] * inv));
        uint4 b = make_uint4(pack_bf16(o[8] * inv, o[9] * inv), pack_bf16(o[10] * inv, o[11] * inv),
                             pack_bf16(o[12] * inv, o[13] * inv), pack_bf16(o[14] * inv, o[15] * inv));
        reinterpret_cast<uint4*>(orow + c * 16)[0] = a;
        reinterpret_cast<uint4*>(orow + c * 16)[1] = b;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------------
// v3: one CTA per SM, TWO 128-row Q tiles (A, B) of the same head sharing every K/V tile, the
// FA4 ping-pong: while softmax warpgroup A turns S_A(j) into P_A(j), the tensor core runs
// PV_B(j-1) / S_B(j), and vice versa, so the MUFU (exp) and the tensor pipe stay busy together.
//   w0: TMA (Q_A, Q_B once; K_j, V_j through a 2-stage ring)     w1: MMA issuer (one thread)
//   w2: TMEM alloc                                                w4-7 / w8-11: softmax A / B
// TMEM (512 cols): S_A | S_B | O_A | O_B.  P_X is written as packed bf16 over S_X (TS MMA).
// The softmax warpgroups take 224 registers (setmaxnreg; the producer group gives its share
// back) so the whole 128-column S row sits in registers: ONE TMEM read per tile and no
// second pass.  Per tile: 4 tcgen05.ld issued back to back, one wait.
// MMA issue order (in-order tensor pipe):  S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) ...
template <int HD>
struct Ft3Cfg {
  static constexpr int NCH = (HD + CHUNK - 1) / CHUNK;
  static constexpr int TILE_BYTES = NCH * FBN * CHUNK * 2;
  static constexpr int QA_OFF = 0, QB_OFF = TILE_BYTES;
  static constexpr int K_OFF = 2 * TILE_BYTES;   // 2 stages
  static constexpr int V_OFF = 4 * TILE_BYTES;   // 2 stages
  static constexpr int BAR_OFF = 6 * TILE_BYTES;
  static constexpr int SMEM = 1024 + BAR_OFF + 256;
};

template <int N>
NOVA_DEV void tmem_ld32_nw(uint32_t taddr, uint32_t* r) {  // no wait: pair with tmem_ld_wait32
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// tcgen05.wait::ld that the compiler must order before any use of r[0..31]
NOVA_DEV void tmem_ld_wait32(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// Work decomposition of the persistent v3 kernel, from the SHAPE only (never the grid): units
// are (head, Q-tile pair) in head-major order; the first `full` = floor(units / 148) * 148
// take every key tile; the remaining `rem` units are each cut into KC key-range chunks
// (KC = 148 / rem, >= 2 tiles per chunk) whose (m, l, O) partials are merged in chunk order by
// the last chunk to finish.  So the numerics are identical for any SM budget, and on the full
// GPU the tail wave is ~148 short chunks instead of `rem` full-length units.
constexpr int FMHA_WS_SLOTS = 320;  // partial slots (2 FBM rows each) in the split workspace
constexpr int FMHA_TICKETS = 256;
struct Fmha3Plan {
  int n_q2, n_tiles, units, full, rem, KC, total, causal, H, kt;
  int T = 0;  // causal split: target key tiles per chunk (0 = off)
  __host__ __device__ int len(int pr) const { return min(n_tiles, (2 * pr + 2) * FBM / kt); }
  __host__ __device__ int kc_of(int pr) const { return T ? min(4, max(1, (len(pr) + T - 1) / T)) : 1; }
  __host__ __device__ Fmha3Plan(int S, int H_, int split = 1, int causal_ = 0, int kt_ = FBN, int csplit = 0) {
    H = H_;
    causal = causal_;
    kt = kt_;
    n_q2 = (S + 2 * FBM - 1) / (2 * FBM);
    n_tiles = (S + kt - 1) / kt;
    units = n_q2 * H;
    full = (units / 148) * 148;
    rem = units - full;
    KC = 1;
    if (rem > 0) {
      KC = 148 / rem;
      if (KC > n_tiles / 2) KC = n_tiles / 2;
      if (KC > 16) KC = 16;
      if (KC < 1) KC = 1;
    }
    if (KC == 1 || !split || causal) {
      KC = 1;
      full = units;
      rem = 0;
    }
    total = full + rem * KC;
    if (causal && csplit && split) {
      int all = 0;
      for (int pr = 0; pr < n_q2; ++pr) all += H * len(pr);
      for (T = max(4, (all + 147) / 148);; ++T) {
        int slots = 0, groups = 0, tot = 0;
        for (int pr = 0; pr < n_q2; ++pr) {
          const int kc = kc_of(pr);
          tot += H * kc;
          if (kc > 1) slots += H * kc, groups += H;
        }
        if (slots <= FMHA_WS_SLOTS && groups <= FMHA_TICKETS) {
          total = tot;
          break;
        }
      }
    }
  }
  // unit -> (head, q pair, key tiles [t0, t1), split slot or -1, chunk index).
  // Causal: units run longest first (q pair n_q2-1 down to 0, heads fastest); the pair's key
  // range ends at its B tile's diagonal.
  __host__ __device__ void decode(int u, int& h, int& pr, int& t0, int& t1, int& slot, int& ch) const {
    int grp, kc;
    decode(u, h, pr, t0, t1, slot, ch, grp, kc);
  }
  __host__ __device__ void decode(int u, int& h, int& pr, int& t0, int& t1, int& slot, int& ch, int& grp,
                                  int& kc) const {
    grp = -1;
    kc = 1;
    if (causal && T) {
      int u0 = 0, s0 = 0, g0 = 0;
      for (pr = n_q2 - 1; pr >= 0; --pr) {
        const int k = kc_of(pr), n = H * k;
        if (u < u0 + n) {
          const int w = u - u0, L = len(pr);
          h = w / k;
          ch = w % k;
          t0 = (ch * L) / k;
          t1 = ((ch + 1) * L) / k;
          slot = -1;
          if (k > 1) slot = s0 + h * k + ch, grp = g0 + h, kc = k;
          return;
        }
        u0 += n;
        if (k > 1) s0 += n, g0 += H;
      }
      pr = 0, h = 0, t0 = t1 = 0, slot = -1, ch = 0;
      return;
    }
    if (causal) {
      pr = n_q2 - 1 - u / H;
      h = u % H;
      slot = -1;
      ch = 0;
      t0 = 0;
      t1 = min(n_tiles, (2 * pr + 2) * FBM / kt);
      return;
    }
    int base = u;
    ch = 0;
    slot = -1;
    if (u >= full) {
      base = full + (u - full) / KC;
      ch = (u - full) % KC;
      slot = u - full;
    }
    h = base / n_q2;
    pr = base % n_q2;
    t0 = slot < 0 ? 0 : (ch * n_tiles) / KC;
    t1 = slot < 0 ? n_tiles : ((ch + 1) * n_tiles) / KC;
    if (slot >= 0) grp = (u - full) / KC, kc = KC;
  }
  // k-th unit of CTA c out of G: snake order over rounds (c, then G-1-c, ...), so with units
  // sorted longest first the per-CTA sums even out; -1 = no unit this round, -2 = done.
  // Which CTA runs a unit never changes its numerics (a unit is computed whole or as fixed chunks).
  __host__ __device__ int unit_of(int k, int c, int G) const {
    if (k * G >= total) return -2;
    const int u = k * G + ((k & 1) ? G - 1 - c : c);
    return u < total ? u : -1;
  }
};

template <int HD, bool CAUSAL>
__global__ void __launch_bounds__(384, 1)
    fmha3_kernel(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, int ldo, int S, int H, int KV,
                 float scale_log2, float* __restrict__ ws, int* __restrict__ tickets, int split) {
  using C = Ft3Cfg<HD>;
  constexpr int NCH = C::NCH;
  constexpr int PW = HD + 4;  // split partial row: m, l, -, -, O[HD] (16-byte aligned rows)
  constexpr uint32_t IDESC_S = umma_idesc_bf16(FBM, FBN);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(FBM, HD) | (1u << 16);  // B (V) MN-major
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2] (A, B)
  uint64_t* p_full = bars + 11;  // [2] (A, B), 128 arrivals
  uint64_t* o_done = bars + 13;
  uint64_t* turn = bars + 14;    // [2] MUFU ping-pong token: A's exps, then B's, ... (128 arrivals)
  uint64_t* q_empty = bars + 16; // Q tiles and O of the unit consumed (256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  int* s_last = reinterpret_cast<int*>(bars + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Fmha3Plan plan(S, H, split, CAUSAL ? 1 : 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < 17; ++i) mbar_init(&bars[i], (i == 11 || i == 12 || i == 14 || i == 15) ? 128 : (i == 16 ? 256 : 1));
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 0 && lane == 0) {  // ---------------- TMA producer
      int it = 0, nu = 0;
      for (int k = 0, u; (u = plan.unit_of(k, blockIdx.x, gridDim.x)) != -2; ++k) {
        if (u < 0) continue;
        int h, pr, t0, t1, slot, ch;
        plan.decode(u, h, pr, t0, t1, slot, ch);
        const int kvh = h / (H / KV), q0 = pr * 2 * FBM;
        const int qcol = h * HD, kcol = (H + kvh) * HD, vcol = (H + KV + kvh) * HD;
        mbar_wait(q_empty, (nu & 1) ^ 1);  // previous unit's MMAs and epilogue are done with Q / O
        mbar_arrive_expect_tx(q_full, 2 * C::TILE_BYTES);
        for (int c = 0; c < NCH; ++c) {
          tma_load_2d(smem + C::QA_OFF + c * FBN * 128, &tm, q_full, qcol + c * CHUNK, q0);
          tma_load_2d(smem + C::QB_OFF + c * FBN * 128, &tm, q_full, qcol + c * CHUNK, q0 + FBM);
        }
        for (int j = t0; j < t1; ++j, ++it) {
          const int st = it & 1;
          const uint32_t ph = ((it >> 1) & 1) ^ 1;
          mbar_wait(&k_empty[st], ph);
          mbar_arrive_expect_tx(&k_full[st], C::TILE_BYTES);
          for (int c = 0; c < NCH; ++c)
            tma_load_2d(smem + C::K_OFF + st * C::TILE_BYTES + c * FBN * 128, &tm, &k_full[st], kcol + c * CHUNK,
                        j * FBN);
          mbar_wait(&v_empty[st], ph);
          mbar_arrive_expect_tx(&v_full[st], C::TILE_BYTES);
          for (int c = 0; c < NCH; ++c)
            tma_load_2d(smem + C::V_OFF + st * C::TILE_BYTES + c * FBN * 128, &tm, &v_full[st], vcol + c * CHUNK,
                        j * FBN);
        }
        ++nu;
      }
    } else if (warp == 1 && lane == 0) {  // ---------------- MMA issuer
      const uint32_t tS[2] = {tbase, tbase + FBN};
      const uint32_t tO[2] = {tbase + 2 * FBN, tbase + 3 * FBN};
      const uint32_t qa[2] = {smem_u32(smem + C::QA_OFF), smem_u32(smem + C::QB_OFF)};
      auto issue_s = [&](int x, int itx) {
        const uint32_t kb = smem_u32(smem + C::K_OFF + (itx & 1) * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k * 16 / CHUNK) * FBN * 128 + (k * 16 % CHUNK) * 2;
          umma_bf16_ss(tS[x], umma_desc_sw128(qa[x] + off), umma_desc_sw128(kb + off), IDESC_S, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[x]);
      };
      auto issue_pv = [&](int x, int itx, bool first) {
        const uint32_t vb = smem_u32(smem + C::V_OFF + (itx & 1) * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < FBN / 16; ++k)  // P: 16 keys = 8 packed TMEM columns per step
          umma_bf16_ts(tO[x], tS[x] + k * 8, umma_desc_sw128_mn(vb + k * 16 * 128, FBN * 128), IDESC_O,
                       (!first || k > 0) ? 1u : 0u);
      };
      int it = 0, nu = 0;
      for (int k = 0, u; (u = plan.unit_of(k, blockIdx.x, gridDim.x)) != -2; ++k) {
        if (u < 0) continue;
        int h, pr, t0, t1, slot, ch;
        plan.decode(u, h, pr, t0, t1, slot, ch);
        const int n = t1 - t0;
        mbar_wait(q_full, nu & 1);
        mbar_wait(&k_full[it & 1], (it >> 1) & 1);
        tc_fence_after();
        issue_s(0, it);
        issue_s(1, it);
        umma_commit(&k_empty[it & 1]);
        for (int j = 0; j < n; ++j, ++it) {
          const int st = it & 1;
          const uint32_t ph = (it >> 1) & 1;
          const bool more = j + 1 < n;
          mbar_wait(&v_full[st], ph);
          mbar_wait(&p_full[0], it & 1);
          tc_fence_after();
          issue_pv(0, it, j == 0);
          if (more) {
            mbar_wait(&k_full[st ^ 1], ((it + 1) >> 1) & 1);
            tc_fence_after();
            issue_s(0, it + 1);
          }
          mbar_wait(&p_full[1], it & 1);
          tc_fence_after();
          issue_pv(1, it, j == 0);
          umma_commit(&v_empty[st]);
          if (more) {
            issue_s(1, it + 1);
            umma_commit(&k_empty[st ^ 1]);
          }
        }
        umma_commit(o_done);
        ++nu;
      }
    }
  } else {  // ---------------- softmax warpgroups: x = 0 (warps 4-7, tile A), 1 (warps 8-11, tile B)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    const int x = (warp - 4) >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tbase + x * FBN + lane_off, tO = tbase + (2 + x) * FBN + lane_off;
    int it = 0, nu = 0;
    for (int k = 0, u; (u = plan.unit_of(k, blockIdx.x, gridDim.x)) != -2; ++k) {
      if (u < 0) continue;
      int h, pr, t0, t1, slot, ch;
      plan.decode(u, h, pr, t0, t1, slot, ch);
      const int qrow = pr * 2 * FBM + x * FBM + row;
      const int qlo = pr * 2 * FBM + x * FBM;  // first query row of this warpgroup's tile
      float m = -1e30f, l = 0.f;
      for (int j = t0; j < t1; ++j, ++it) {
        mbar_wait(&s_full[x], it & 1);
        tc_fence_after();
        uint32_t sv[FBN];
#pragma unroll
        for (int c = 0; c < FBN / 32; ++c) tmem_ld32_nw<32>(tS + c * 32, sv + c * 32);
#pragma unroll
        for (int c = 0; c < FBN / 32; ++c) tmem_ld_wait32(sv + c * 32);
        const int k0 = j * FBN;
        if (CAUSAL) {  // keys after the query row (and beyond S) are masked; interior tiles skip the test
          if (k0 + FBN - 1 > qlo || k0 + FBN > S) {
            const int lim = min(S, qrow + 1);
#pragma unroll
            for (int i = 0; i < FBN; ++i)
              if (k0 + i >= lim) sv[i] = __float_as_uint(-1e30f);
          }
        } else if (k0 + FBN > S) {  // keys beyond S (TMA zero-filled rows) must not contribute
#pragma unroll
          for (int i = 0; i < FBN; ++i)
            if (k0 + i >= S) sv[i] = __float_as_uint(-1e30f);
        }
        // row max with 8 independent accumulators (short dependency chains)
        float mxa[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mxa[a] = __uint_as_float(sv[a]);
#pragma unroll
        for (int i = 8; i < FBN; i += 8)
#pragma unroll
          for (int a = 0; a < 8; ++a) mxa[a] = fmaxf(mxa[a], __uint_as_float(sv[i + a]));
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        const float mnew = fmaxf(m, mx * scale_log2);
        const bool need = (mnew - m) > 8.0f;
        if (__any_sync(0xffffffffu, need) && j > t0) {  // lazy rescale of O (PV_x(j-1) done: s_full order)
          const float f = need ? fast_exp2(m - mnew) : 1.0f;
#pragma unroll
          for (int c = 0; c < HD / 16; ++c) {
            float o[16];
            tmem_ld16(tO + c * 16, o);
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= f;
            tmem_st16(tO + c * 16, o);
          }
        }
        if (need) {
          l *= fast_exp2(m - mnew);
          m = mnew;
        }
        // MUFU ping-pong: the two warpgroups take turns for the exponentials (A first)
        if (x == 1) mbar_wait(&turn[1], it & 1);
        else if (it > 0) mbar_wait(&turn[0], (it - 1) & 1);
        const float nm = -m;
        float lsa[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) lsa[a] = 0.f;
#pragma unroll
        for (int c = 0; c < FBN / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float p0 = fast_exp2(fmaf(__uint_as_float(sv[c * 32 + i]), scale_log2, nm));
            const float p1 = fast_exp2(fmaf(__uint_as_float(sv[c * 32 + i + 1]), scale_log2, nm));
            lsa[(i >> 1) & 7] += p0 + p1;
            pk[i / 2] = pack_bf16(p0, p1);
          }
          tmem_st16u(tS + c * 16, pk);  // packed P keys 32c..32c+31 -> columns 16c..16c+15
        }
        l += ((lsa[0] + lsa[1]) + (lsa[2] + lsa[3])) + ((lsa[4] + lsa[5]) + (lsa[6] + lsa[7]));
        mbar_arrive(&turn[x ^ 1]);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[x]);
      }
      mbar_wait(o_done, nu & 1);
      tc_fence_after();
      if (slot < 0) {  // whole key range: normalize and store
        const float inv = 1.0f / l;
        bf16* orow = out + (size_t)qrow * ldo + (size_t)h * HD;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + c * 16, o);
          if (qrow < S) {
            uint4 a = make_uint4(pack_bf16(o[0] * inv, o[1] * inv), pack_bf16(o[2] * inv, o[3] * inv),
                                 pack_bf16(o[4] * inv, o[5] * inv), pack_bf16(o[6] * inv, o[7] * inv));
            uint4 b = make_uint4(pack_bf16(o[8] * inv, o[9] * inv), pack_bf16(o[10] * inv, o[11] * inv),
                                 pack_bf16(o[12] * inv, o[13] * inv), pack_bf16(o[14] * inv, o[15] * inv));
            reinterpret_cast<uint4*>(orow + c * 16)[0] = a;
            reinterpret_cast<uint4*>(orow + c * 16)[1] = b;
          }
        }
        tc_fence_before();
        mbar_arrive(q_empty);
      } else {  // key chunk: (m, l, O) partial; the last chunk of the unit merges in chunk order
        float* wr = ws + ((size_t)slot * 2 * FBM + x * FBM + row) * PW;
        *reinterpret_cast<float4*>(wr) = make_float4(m, l, 0.f, 0.f);
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + c * 16, o);
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(wr + 4 + c * 16 + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
        }
        tc_fence_before();
        mbar_arrive(q_empty);
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int grp = (u - plan.full) / plan.KC;
        if (threadIdx.x == 128) *s_last = atomicAdd(&tickets[grp], 1) == plan.KC - 1;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (*s_last) {
          __threadfence();
          const float* base = ws + ((size_t)grp * plan.KC * 2 * FBM + x * FBM + row) * PW;
          const size_t cstride = (size_t)2 * FBM * PW;
          float M = -1e30f;
          for (int c2 = 0; c2 < plan.KC; ++c2) M = fmaxf(M, __ldcg(base + c2 * cstride));
          float den = 0.f, acc[HD];
#pragma unroll
          for (int d = 0; d < HD; ++d) acc[d] = 0.f;
          for (int c2 = 0; c2 < plan.KC; ++c2) {  // chunk order; one row = HD/4 independent 16-byte loads
            const float* pr2 = base + c2 * cstride;
            const float4 ml = __ldcg(reinterpret_cast<const float4*>(pr2));
            float4 ov[HD / 4];
#pragma unroll
            for (int q = 0; q < HD / 4; ++q) ov[q] = __ldcg(reinterpret_cast<const float4*>(pr2 + 4) + q);
            const float f = exp2f(ml.x - M);
            den += f * ml.y;
#pragma unroll
            for (int q = 0; q < HD / 4; ++q) {
              acc[4 * q] += f * ov[q].x;
              acc[4 * q + 1] += f * ov[q].y;
              acc[4 * q + 2] += f * ov[q].z;
              acc[4 * q + 3] += f * ov[q].w;
            }
          }
          const float inv = 1.0f / den;
          bf16* orow = out + (size_t)qrow * ldo + (size_t)h * HD;
          if (qrow < S) {
#pragma unroll
            for (int d0 = 0; d0 < HD; d0 += 8)
              *reinterpret_cast<uint4*>(orow + d0) =
                  make_uint4(pack_bf16(acc[d0] * inv, acc[d0 + 1] * inv), pack_bf16(acc[d0 + 2] * inv, acc[d0 + 3] * inv),
                             pack_bf16(acc[d0 + 4] * inv, acc[d0 + 5] * inv), pack_bf16(acc[d0 + 6] * inv, acc[d0 + 7] * inv));
          }
          if (threadIdx.x == 128) tickets[grp] = 0;
        }
      }
      ++nu;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// ------------------------------------------------------------------------------------------------
// v4: v3's two-Q-tile ping-pong with 64-key tiles and DOUBLE-BUFFERED S per Q tile.  In v3 the
// S MMA of tile j+1 could only start after softmax j had produced P_j (P aliases S), so every
// tile paid the chain P_j -> PV_j -> S_{j+1} -> tcgen05.ld before the exps could restart
// (measured: tensor pipe 32%, MUFU 52% busy on the ViT shape).  Here S_x(j+2) is issued right
// after PV_x(j) into the buffer P_x(j) occupied, so when softmax x finishes tile j the scores of
// tile j+1 are already in TMEM and the MUFU alternates A/B without gaps.
//   TMEM (512 cols): S_A[0] S_A[1] S_B[0] S_B[1] (64 each) | O_A (256..) | O_B (384..)
//   smem: Q_A, Q_B (128 rows) + 4-stage K and V rings (64-row tiles)
// O rescaling (rare, lazy) waits for PV_x(j-1) through o_ready[x], since S_x(j) no longer
// orders after it.  Numerics per (row, head): fixed key order, fixed 64-key tiling.
constexpr int KT4 = 64;    // keys per tile
// exp2 of a pair on the FMA pipe (FA4's MUFU offload), for x <= 0: x = n + f with n = rint(x)
// by the 1.5 * 2^23 magic add, f in [-0.5, 0.5]; 2^f by a degree-3 polynomial (max rel err
// 7.5e-5, far below P's bf16 rounding); 2^n added into the exponent field with one IMAD
// ((bits(t) << 23) == n << 23 mod 2^32 because bits(1.5 * 2^23) has nine zero low bits).
NOVA_DEV float2 exp2_fma2(float2 x) {
  x.x = fmaxf(x.x, -126.0f);
  x.y = fmaxf(x.y, -126.0f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 n = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __fadd2_rn(x, make_float2(-n.x, -n.y));
  float2 p = __ffma2_rn(make_float2(0.05517149344f, 0.05517149344f), f, make_float2(0.24261111021f, 0.24261111021f));
  p = __ffma2_rn(p, f, make_float2(0.69326102734f, 0.69326102734f));
  p = __ffma2_rn(p, f, make_float2(0.99992805719f, 0.99992805719f));
  return make_float2(__int_as_float(__float_as_int(t.x) * (1 << 23) + __float_as_int(p.x)),
                     __int_as_float(__float_as_int(t.y) * (1 << 23) + __float_as_int(p.y)));
}
#ifndef NOVA_EXP_POLY
#define NOVA_EXP_POLY 2
#endif
constexpr int EXP_POLY_OF_8 = NOVA_EXP_POLY;  // pairs of P per 8 whose exponentials run on the FMA pipe
constexpr int KST4 = 4;    // K / V ring depth
template <int HD>
struct Ft4Cfg {
  static constexpr int NCH = (HD + CHUNK - 1) / CHUNK;
  static constexpr int Q_BYTES = NCH * FBM * CHUNK * 2;    // one 128-row Q tile
  static constexpr int KV_BYTES = NCH * KT4 * CHUNK * 2;   // one 64-row K or V tile
  static constexpr int QA_OFF = 0, QB_OFF = Q_BYTES;
  static constexpr int K_OFF = 2 * Q_BYTES;
  static constexpr int V_OFF = K_OFF + KST4 * KV_BYTES;
  static constexpr int BAR_OFF = V_OFF + KST4 * KV_BYTES;
  static constexpr int SMEM = 1024 + BAR_OFF + 512;
};

template <int HD, bool CAUSAL>
__global__ void __launch_bounds__(384, 1)
    fmha4_kernel(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, int ldo, int S, int H, int KV,
                 float scale_log2, float* __restrict__ ws, int* __restrict__ tickets, int split, int turns) {
  using C = Ft4Cfg<HD>;
  constexpr int NCH = C::NCH;
  constexpr int PW = HD + 4;
  constexpr uint32_t IDESC_S = umma_idesc_bf16(FBM, KT4);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(FBM, HD) | (1u << 16);  // B (V) MN-major
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;    // 256 arrivals
  uint64_t* k_full = bars + 2;     // [KST4]
  uint64_t* k_empty = bars + 6;    // [KST4]
  uint64_t* v_full = bars + 10;    // [KST4]
  uint64_t* v_empty = bars + 14;   // [KST4]
  uint64_t* s_full = bars + 18;    // [2 groups][2 buffers]
  // P_x(g) ready, per (group, S buffer): a group may finish two tiles before the MMA warp has
  // consumed the first (S_x(g+1) is already issued), so one barrier per group could complete two
  // phases unobserved; per buffer it cannot (S_x(g+2) waits for PV_x(g)).
  uint64_t* p_full = bars + 22;    // [2 groups][2 buffers], 128 arrivals
  uint64_t* o_ready = bars + 26;   // [2]: PV_x(j) complete
  uint64_t* o_done = bars + 28;
  uint64_t* turn = bars + 29;      // [2], 128 arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 31);
  int* s_last = reinterpret_cast<int*>(bars + 32);

  // warp index through a shuffle: provably warp-uniform, so warp-role code keeps its scalars in
  // uniform registers (MMA descriptors without per-lane R2UR waterfalls)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const Fmha3Plan plan(S, H, split & 255, CAUSAL ? 1 : 0, KT4, CAUSAL ? (split >> 8) & 1 : 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < 31; ++i) {
      uint32_t cnt = 1;
      if (i == 1) cnt = 256;
      if ((i >= 22 && i < 26) || i == 29 || i == 30) cnt = 128;
      mbar_init(&bars[i], cnt);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 0) {  // ---------------- TMA producer (lane 0); the branch is warp-uniform
     if (lane == 0) {
      int g = 0, nu = 0;
      for (int k = 0, u; (u = plan.unit_of(k, blockIdx.x, gridDim.x)) != -2; ++k) {
        if (u < 0) continue;
        int h, pr, t0, t1, slot, ch;
        plan.decode(u, h, pr, t0, t1, slot, ch);
        const int kvh = h / (H / KV), q0 = pr * 2 * FBM;
        const int qcol = h * HD, kcol = (H + kvh) * HD, vcol = (H + KV + kvh) * HD;
        mbar_wait(q_empty, (nu & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, 2 * C::Q_BYTES);
        for (int c = 0; c < NCH; ++c)
          for (int r = 0; r < 2 * FBM / KT4; ++r)  // Q_A then Q_B rows, 64-row boxes
            tma_load_2d(smem + (r < FBM / KT4 ? C::QA_OFF : C::QB_OFF) + c * FBM * 128 + (r % (FBM / KT4)) * KT4 * 128,
                        &tm, q_full, qcol + c * CHUNK, q0 + r * KT4);
        for (int j = t0; j < t1; ++j, ++g) {
          const int st = g % KST4;
          const uint32_t ph = ((g / KST4) & 1) ^ 1;
          mbar_wait(&k_empty[st], ph);
          mbar_arrive_expect_tx(&k_full[st], C::KV_BYTES);
          for (int c = 0; c < NCH; ++c)
            tma_load_2d(smem + C::K_OFF + st * C::KV_BYTES + c * KT4 * 128, &tm, &k_full[st], kcol + c * CHUNK,
                        j * KT4);
          mbar_wait(&v_empty[st], ph);
          mbar_arrive_expect_tx(&v_full[st], C::KV_BYTES);
          for (int c = 0; c < NCH; ++c)
            tma_load_2d(smem + C::V_OFF + st * C::KV_BYTES + c * KT4 * 128, &tm, &v_full[st], vcol + c * CHUNK,
                        j * KT4);
        }
        ++nu;
      }
      // producer tail: the MMA warp's releases (asynchronous tcgen05.commit arrives) of the last
      // ring slots have landed before this CTA can exit and hand its shared memory to a successor
      for (int i = 0; i < KST4; ++i, ++g) {
        const int st = g % KST4;
        const uint32_t ph = ((g / KST4) & 1) ^ 1;
        mbar_wait(&k_empty[st], ph);
        mbar_wait(&v_empty[st], ph);
      }
     }
    } else if (warp == 1) {  // ---------------- MMA issuer: the whole warp waits, lane 0 issues
      // Descriptors are built once from warp-uniform values (uniform registers); per MMA only a
      // constant is added to the start-address field (smem < 256 KB: no carry out of it).
      const uint64_t qd[2] = {umma_desc_sw128(smem_u32(smem + C::QA_OFF)), umma_desc_sw128(smem_u32(smem + C::QB_OFF))};
      const uint64_t kd0 = umma_desc_sw128(smem_u32(smem + C::K_OFF));
      const uint64_t vd0 = umma_desc_sw128_mn(smem_u32(smem + C::V_OFF), KT4 * 128);
      auto tS = [&](int x, int g) { return tbase + (uint32_t)(x * 2 * KT4 + (g & 1) * KT4); };
      const uint32_t tO[2] = {tbase + 256, tbase + 384};
      auto issue_s = [&](int x, int g) {  // S_x(g) = Q_x K_g^T -> S buffer g & 1 of group x
        const uint64_t kb = kd0 + (uint64_t)((g % KST4) * (C::KV_BYTES >> 4));
        const uint32_t d = tS(x, g);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t qoff = ((k * 16 / CHUNK) * FBM * 128 + (k * 16 % CHUNK) * 2) >> 4;
          const uint32_t koff = ((k * 16 / CHUNK) * KT4 * 128 + (k * 16 % CHUNK) * 2) >> 4;
          umma_bf16_ss_warp(d, qd[x] + qoff, kb + koff, IDESC_S, k > 0 ? 1u : 0u);
        }
        umma_commit_warp(&s_full[x * 2 + (g & 1)]);
      };
      auto issue_pv = [&](int x, int g, bool first) {
        const uint64_t vb = vd0 + (uint64_t)((g % KST4) * (C::KV_BYTES >> 4));
        const uint32_t a = tS(x, g), d = tO[x];
#pragma unroll
        for (int k = 0; k < KT4 / 16; ++k)  // P: 16 keys = 8 packed TMEM columns per step
          umma_bf16_ts_warp(d, a + k * 8, vb + (uint64_t)((k * 16 * 128) >> 4), IDESC_O, (!first || k > 0) ? 1u : 0u);
        umma_commit_warp(&o_ready[x]);
      };
      auto commit = [&](uint64_t* bar) { umma_commit_warp(bar); };
      auto wait_k = [&](int g) {
        mbar_wait(&k_full[g % KST4], (g / KST4) & 1);
        tc_fence_after();
      };
      int g = 0, nu = 0;
      for (int k = 0, u; (u = plan.unit_of(k, blockIdx.x, gridDim.x)) != -2; ++k) {
        if (u < 0) continue;
        int h, pr, t0, t1, slot, ch;
        plan.decode(u, h, pr, t0, t1, slot, ch);
        const int n = t1 - t0, g0 = g;
        mbar_wait(q_full, nu & 1);
        for (int j = 0; j < 2 && j < n; ++j) {  // prologue: S(0), S(1) of both tiles
          wait_k(g0 + j);
          issue_s(0, g0 + j);
          issue_s(1, g0 + j);
          commit(&k_empty[(g0 + j) % KST4]);
        }
        for (int j = 0; j < n; ++j, ++g) {
          const int st = g % KST4;
          const bool more = j + 2 < n;
          mbar_wait(&v_full[st], (g / KST4) & 1);
          mbar_wait(&p_full[0 + (g & 1)], (g >> 1) & 1);
          tc_fence_after();
          issue_pv(0, g, j == 0);
          if (more) {
            wait_k(g + 2);
            issue_s(0, g + 2);
          }
          mbar_wait(&p_full[2 + (g & 1)], (g >> 1) & 1);
          tc_fence_after();
          issue_pv(1, g, j == 0);
          commit(&v_empty[st]);
          if (more) {
            issue_s(1, g + 2);
            commit(&k_empty[(g + 2) % KST4]);
          }
        }
        commit(o_done);
        ++nu;
      }
      if (g > 0) {  // the last PV releases (o_ready) have landed too (nothing else waits for them)
        mbar_wait(&o_ready[0], (g - 1) & 1);
        mbar_wait(&o_ready[1], (g - 1) & 1);
      }
    }
  } else {  // ---------------- softmax warpgroups: x = 0 (warps 4-7, tile A), 1 (warps 8-11, tile B)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    const int x = (warp - 4) >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tSx = tbase + x * 2 * KT4 + lane_off, tO = tbase + 256 + x * 128 + lane_off;
    int g = 0, nu = 0;
    for (int k = 0, u; (u = plan.unit_of(k, blockIdx.x, gridDim.x)) != -2; ++k) {
      if (u < 0) continue;
      int h, pr, t0, t1, slot, ch, grp, kcn;
      plan.decode(u, h, pr, t0, t1, slot, ch, grp, kcn);
      const int qrow = pr * 2 * FBM + x * FBM + row;
      const int qlo = pr * 2 * FBM + x * FBM;
      float m = -1e30f, l = 0.f;
      for (int j = t0; j < t1; ++j, ++g) {
        const uint32_t tS = tSx + (g & 1) * KT4;
        mbar_wait_sleep(&s_full[x * 2 + (g & 1)], (g >> 1) & 1);
        tc_fence_after();
        uint32_t sv[KT4];
        tmem_ld32_nw<32>(tS, sv);
        tmem_ld32_nw<32>(tS + 32, sv + 32);
        tmem_ld_wait32(sv);
        tmem_ld_wait32(sv + 32);
        const int k0 = j * KT4;
        if (CAUSAL) {
          if (k0 + KT4 - 1 > qlo || k0 + KT4 > S) {
            const int lim = min(S, qrow + 1);
#pragma unroll
            for (int i = 0; i < KT4; ++i)
              if (k0 + i >= lim) sv[i] = __float_as_uint(-1e30f);
          }
        } else if (k0 + KT4 > S) {
#pragma unroll
          for (int i = 0; i < KT4; ++i)
            if (k0 + i >= S) sv[i] = __float_as_uint(-1e30f);
        }
        float mxa[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mxa[a] = __uint_as_float(sv[a]);
#pragma unroll
        for (int i = 8; i < KT4; i += 8)
#pragma unroll
          for (int a = 0; a < 8; ++a) mxa[a] = fmaxf(mxa[a], __uint_as_float(sv[i + a]));
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        const bool none = CAUSAL && mx == -1e30f && m == -1e30f;
        const float mnew = none ? m : fmaxf(m, mx * scale_log2);
        const bool need = (mnew - m) > 8.0f;
        if (__any_sync(0xffffffffu, need) && j > t0) {  // lazy rescale of O: PV_x(g-1) must be complete
          mbar_wait(&o_ready[x], (g - 1) & 1);
          tc_fence_after();
          const float f = need ? fast_exp2(m - mnew) : 1.0f;
#pragma unroll
          for (int c = 0; c < HD / 16; ++c) {
            float o[16];
            tmem_ld16(tO + c * 16, o);
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= f;
            tmem_st16(tO + c * 16, o);
          }
        }
        if (need) {
          l *= fast_exp2(m - mnew);
          m = mnew;
        }
        if (turns) {  // optional MUFU ping-pong (A's exps, then B's, ...)
          if (x == 1) mbar_wait_sleep(&turn[1], g & 1);
          else if (g > 0) mbar_wait_sleep(&turn[0], (g - 1) & 1);
        }
        // exponent arguments and row sums on the packed f32x2 pipe (FFMA2 / FADD2): the MUFU is the
        // bottleneck, so the rest of the phase must issue in as few slots as possible
        const float sl = none ? 0.f : scale_log2, nmv = none ? -200.f : -m;
        const float2 sc2 = make_float2(sl, sl), nm2 = make_float2(nmv, nmv);
        float2 ls2[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) ls2[a] = make_float2(0.f, 0.f);
        uint32_t pk[KT4 / 2];
#pragma unroll
        for (int i = 0; i < KT4; i += 2) {
          const float2 xx = __ffma2_rn(make_float2(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sc2, nm2);
          float p0, p1;
          if (((i >> 1) & 7) < EXP_POLY_OF_8) {
            const float2 pp = exp2_fma2(xx);
            p0 = pp.x;
            p1 = pp.y;
          } else {
            p0 = fast_exp2(xx.x);
            p1 = fast_exp2(xx.y);
          }
          ls2[(i >> 1) & 3] = __fadd2_rn(ls2[(i >> 1) & 3], make_float2(p0, p1));
          pk[i / 2] = pack_bf16(p0, p1);
        }
        // hand the MUFU to the other tile as soon as the last exponential is in (the data
        // dependency on pk keeps the arrive after it); P stores and sums finish in its shadow
        if (turns) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&turn[x ^ 1])), "r"(pk[KT4 / 2 - 1])
                       : "memory");
        }
        tmem_st16u(tS, pk);        // packed P keys 0..31  -> columns 0..15
        tmem_st16u(tS + 16, pk + 16);  // keys 32..63 -> columns 16..31
        const float2 s01 = __fadd2_rn(ls2[0], ls2[1]), s23 = __fadd2_rn(ls2[2], ls2[3]);
        const float2 s4 = __fadd2_rn(s01, s23);
        l += s4.x + s4.y;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[x * 2 + (g & 1)]);
      }
      mbar_wait(o_done, nu & 1);
      tc_fence_after();
      if (slot < 0) {
        const float inv = 1.0f / l;
        bf16* orow = out + (size_t)qrow * ldo + (size_t)h * HD;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + c * 16, o);
          if (qrow < S) {
            uint4 a = make_uint4(pack_bf16(o[0] * inv, o[1] * inv), pack_bf16(o[2] * inv, o[3] * inv),
                                 pack_bf16(o[4] * inv, o[5] * inv), pack_bf16(o[6] * inv, o[7] * inv));
            uint4 b = make_uint4(pack_bf16(o[8] * inv, o[9] * inv), pack_bf16(o[10] * inv, o[11] * inv),
                                 pack_bf16(o[12] * inv, o[13] * inv), pack_bf16(o[14] * inv, o[15] * inv));
            reinterpret_cast<uint4*>(orow + c * 16)[0] = a;
            reinterpret_cast<uint4*>(orow + c * 16)[1] = b;
          }
        }
        tc_fence_before();
        mbar_arrive(q_empty);
      } else {  // key chunk: (m, l, O) partial; the last chunk of the unit merges in chunk order
        // partial slot layout column-major, rows fastest: element (d, r) at d * 2 FBM + r (d 0 = m, 1 = l,
        // 4.. = O), so each warp store / load is one coalesced 128-byte access (a row-major slot made
        // every warp access touch 32 rows: ~33 x 32 L1 wavefronts per thread block, the split's cost)
        constexpr int R2 = 2 * FBM;
        float* wr = ws + (size_t)slot * R2 * PW + x * FBM + row;
        wr[0] = m;
        wr[R2] = l;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + c * 16, o);
#pragma unroll
          for (int i = 0; i < 16; ++i) wr[(size_t)(4 + c * 16 + i) * R2] = o[i];
        }
        tc_fence_before();
        mbar_arrive(q_empty);
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (threadIdx.x == 128) *s_last = atomicAdd(&tickets[grp], 1) == kcn - 1;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (*s_last) {
          __threadfence();
          const float* base = ws + (size_t)(slot - ch) * R2 * PW + x * FBM + row;
          const size_t cstride = (size_t)R2 * PW;
          float M = -1e30f;
          float mc[16];
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            mc[c2] = c2 < kcn ? __ldcg(base + c2 * cstride) : -1e30f;
            if (c2 < kcn) M = fmaxf(M, mc[c2]);
          }
          float fc[16], den = 0.f;
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            fc[c2] = 0.f;
            if (c2 < kcn) {
              fc[c2] = exp2f(mc[c2] - M);
              den += fc[c2] * __ldcg(base + c2 * cstride + R2);
            }
          }
          const float inv = 1.0f / den;
          bf16* orow = out + (size_t)qrow * ldo + (size_t)h * HD;
#pragma unroll 1
          for (int d0 = 0; d0 < HD; d0 += 16) {  // 16 columns x every chunk per round trip
            float acc[16];
#pragma unroll
            for (int d = 0; d < 16; ++d) acc[d] = 0.f;
            for (int c2 = 0; c2 < kcn; ++c2) {
              const float* pc = base + c2 * cstride + (size_t)(4 + d0) * R2;
              float v[16];
#pragma unroll
              for (int d = 0; d < 16; ++d) v[d] = __ldcg(pc + (size_t)d * R2);
#pragma unroll
              for (int d = 0; d < 16; ++d) acc[d] += fc[c2] * v[d];
            }
            if (qrow < S) {
              *reinterpret_cast<uint4*>(orow + d0) =
                  make_uint4(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv),
                             pack_bf16(acc[4] * inv, acc[5] * inv), pack_bf16(acc[6] * inv, acc[7] * inv));
              *reinterpret_cast<uint4*>(orow + d0 + 8) =
                  make_uint4(pack_bf16(acc[8] * inv, acc[9] * inv), pack_bf16(acc[10] * inv, acc[11] * inv),
                             pack_bf16(acc[12] * inv, acc[13] * inv), pack_bf16(acc[14] * inv, acc[15] * inv));
            }
          }
          if (threadIdx.x == 128) tickets[grp] = 0;
        }
      }
      ++nu;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_qkv_map(CUtensorMap* m, const bf16* ptr, int rows, int cols, int box_rows = FBN) {
  static PFN_encodeTiled_t enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)CHUNK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD, bool CAUSAL>
cudaError_t fmha_launch(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, cudaStream_t s) {
  CUtensorMap tm;
  if (!make_qkv_map(&tm, qkv, S, ld)) return cudaErrorInvalidValue;
  auto kern = fmha_tc_kernel<HD, CAUSAL>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FtCfg<HD>::SMEM);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const float sl2 = LOG2E_F / sqrtf((float)HD);
  count_launch();
  kern<<<dim3((S + FBM - 1) / FBM, H), 256, FtCfg<HD>::SMEM, s>>>(tm, out, ldo, S, H, KV, sl2);
  return cudaGetLastError();
}

template <int HD, bool CAUSAL>
cudaError_t fmha2_launch(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, cudaStream_t s) {
  CUtensorMap tm;
  if (!make_qkv_map(&tm, qkv, S, ld)) return cudaErrorInvalidValue;
  auto kern = fmha2_kernel<HD, CAUSAL>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Ft2Cfg<HD>::SMEM);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const float sl2 = LOG2E_F / sqrtf((float)HD);
  return launch_k(kern, dim3((S + FBM - 1) / FBM, H), dim3(256), Ft2Cfg<HD>::SMEM, s, false, tm, out, ldo, S, H, KV,
                  sl2);
}

}  // namespace

float* g_fmha_ws = nullptr;  // split-chunk partials: <= 148 chunks x 256 rows x (hd + 2) f32
int* g_fmha_tickets = nullptr;

template <int HD, bool CAUSAL>
cudaError_t fmha3_launch(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, int max_ctas,
                         cudaStream_t s) {
  CUtensorMap tm;
  if (!make_qkv_map(&tm, qkv, S, ld)) return cudaErrorInvalidValue;
  auto kern = fmha3_kernel<HD, CAUSAL>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Ft3Cfg<HD>::SMEM);
    if (e != cudaSuccess) return e;
    set = true;
  }
  if (!g_fmha_ws) {  // once per process (one device per engine process)
    if (cudaMalloc(&g_fmha_ws, (size_t)FMHA_WS_SLOTS * 2 * FBM * (128 + 4) * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&g_fmha_tickets, FMHA_TICKETS * sizeof(int)) != cudaSuccess ||
        cudaMemset(g_fmha_tickets, 0, FMHA_TICKETS * sizeof(int)) != cudaSuccess)
      return cudaErrorMemoryAllocation;
  }
  static const int split = getenv("NOVA_FMHA_SPLIT") ? atoi(getenv("NOVA_FMHA_SPLIT")) : 1;  // experiments only
  const Fmha3Plan plan(S, H, split, CAUSAL ? 1 : 0);
  int grid = max_ctas > 0 ? max_ctas : 148;
  if (grid > plan.total) grid = plan.total;
  const float sl2 = LOG2E_F / sqrtf((float)HD);
  return launch_k(kern, dim3(grid), dim3(384), Ft3Cfg<HD>::SMEM, s, false, tm, out, ldo, S, H, KV, sl2, g_fmha_ws,
                  g_fmha_tickets, split);
}

template <int HD, bool CAUSAL>
cudaError_t fmha4_launch(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, int max_ctas,
                         cudaStream_t s) {
  CUtensorMap tm;
  if (!make_qkv_map(&tm, qkv, S, ld, KT4)) return cudaErrorInvalidValue;
  auto kern = fmha4_kernel<HD, CAUSAL>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Ft4Cfg<HD>::SMEM);
    if (e != cudaSuccess) return e;
    set = true;
  }
  if (!g_fmha_ws) {
    if (cudaMalloc(&g_fmha_ws, (size_t)FMHA_WS_SLOTS * 2 * FBM * (128 + 4) * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&g_fmha_tickets, FMHA_TICKETS * sizeof(int)) != cudaSuccess ||
        cudaMemset(g_fmha_tickets, 0, FMHA_TICKETS * sizeof(int)) != cudaSuccess)
      return cudaErrorMemoryAllocation;
  }
  static const int split = getenv("NOVA_FMHA_SPLIT") ? atoi(getenv("NOVA_FMHA_SPLIT")) : 1;
  static const int csplit = getenv("NOVA_FMHA_CSPLIT") ? atoi(getenv("NOVA_FMHA_CSPLIT")) : 0;
  const int split_arg = (split & 255) | ((CAUSAL && csplit) ? 256 : 0);
  const Fmha3Plan plan(S, H, split & 255, CAUSAL ? 1 : 0, KT4, (CAUSAL && csplit) ? 1 : 0);
  int grid = max_ctas > 0 ? max_ctas : 148;
  if (grid > plan.total) grid = plan.total;
  const float sl2 = LOG2E_F / sqrtf((float)HD);
  static const int turns = getenv("NOVA_FMHA_TURN") ? atoi(getenv("NOVA_FMHA_TURN")) : 1;  // experiments
  return launch_k(kern, dim3(grid), dim3(384), Ft4Cfg<HD>::SMEM, s, false, tm, out, ldo, S, H, KV, sl2, g_fmha_ws,
                  g_fmha_tickets, split_arg, turns);
}

// ld (the qkv row length in elements) must be a multiple of 8; hd in {80, 128} (64-col SW128 chunks).
cudaError_t flash_attn_tc(const bf16* qkv, int ld, bf16* out, int ldo, int S, int H, int KV, int hd, int causal,
                          int max_ctas, cudaStream_t s) {
  if (S <= 0) return cudaSuccess;
  if (ld % 8 || H % KV || ldo % 8) return cudaErrorInvalidValue;
  if (g_fmha_version == 4) {
    switch (hd) {
      case 80: return causal ? fmha4_launch<80, true>(qkv, ld, out, ldo, S, H, KV, max_ctas, s)
                             : fmha4_launch<80, false>(qkv, ld, out, ldo, S, H, KV, max_ctas, s);
      case 128: return causal ? fmha4_launch<128, true>(qkv, ld, out, ldo, S, H, KV, max_ctas, s)
                              : fmha4_launch<128, false>(qkv, ld, out, ldo, S, H, KV, max_ctas, s);
    }
    return cudaErrorInvalidValue;
  }
  if (g_fmha_version == 3) {
    switch (hd) {
      case 80: return causal ? fmha3_launch<80, true>(qkv, ld, out, ldo, S, H, KV, max_ctas, s)
                             : fmha3_launch<80, false>(qkv, ld, out, ldo, S, H, KV, max_ctas, s);
      case 128: return causal ? fmha3_launch<128, true>(qkv, ld, out, ldo, S, H, KV, max_ctas, s)
                              : fmha3_launch<128, false>(qkv, ld, out, ldo, S, H, KV, max_ctas, s);
    }
    return cudaErrorInvalidValue;
  }
  if (g_fmha_version >= 2) {
    switch (hd) {
      case 80: return causal ? fmha2_launch<80, true>(qkv, ld, out, ldo, S, H, KV, s)
                             : fmha2_launch<80, false>(qkv, ld, out, ldo, S, H, KV, s);
      case 128: return causal ? fmha2_launch<128, true>(qkv, ld, out, ldo, S, H, KV, s)
                              : fmha2_launch<128, false>(qkv, ld, out, ldo, S, H, KV, s);
    }
    return cudaErrorInvalidValue;
  }
  switch (hd) {
    case 80: return causal ? fmha_launch<80, true>(qkv, ld, out, ldo, S, H, KV, s)
                           : fmha_launch<80, false>(qkv, ld, out, ldo, S, H, KV, s);
    case 128: return causal ? fmha_launch<128, true>(qkv, ld, out, ldo, S, H, KV, s)
                            : fmha_launch<128, false>(qkv, ld, out, ldo, S, H, KV, s);
  }
  return cudaErrorInvalidValue;
}

int g_fmha_version = getenv("NOVA_FMHA") ? atoi(getenv("NOVA_FMHA")) : 4;

}  // namespace nova
