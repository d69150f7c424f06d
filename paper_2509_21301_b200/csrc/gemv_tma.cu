// Decode GEMV, TMA-streamed and persistent (§7 hard part 3: "decode
// must saturate HBM from a minority of SMs ... requires deep TMA-bulk smem pipelines").
//
//   Y[b][n] (epilogue) = sum_k X[b][k] W[n][k] + bias[n],   B <= 16 rows (bf16 X)
//
// The paper's decode stage is memory-bound and Nova gives it a SLICE
// of the SMs, so the kernel must stream HBM at full rate from however many SMs the
// partition owns.  Design:
//  * grid = 4 CTAs per SM of the partition's budget (~40 KB of smem each); each CTA walks a
//    static list of work units (row block x K split) and streams every weight tile of its units
//    through ONE continuous mbarrier ring (3 x 8 KB), so the bytes in flight per SM stay constant
//    across unit boundaries;
//  * warp 0 (one lane) is the TMA producer: [RB x 64] weight tiles (SWIZZLE_128B) + the matching
//    [16 x 64] x tile; before griddepcontrol.wait it already requests the weight tiles of the
//    first ring slots (weights never depend on the previous kernel), x after;
//  * RB/16 consumer warps, one m16 tile each: swap-AB mma.sync m16n8k16 (weights on M, batch on
//    N) from ldmatrix on the swizzled tiles;
//  * the work decomposition (RB, split count P, unit order) depends only on (N, K, epilogue):
//    P <= 8 is chosen so units / 592 is close to a whole number of waves on the full GPU; on a
//    smaller grid a CTA first takes whole row blocks (split partials summed in registers).  Split-K
//    partials go to a workspace and the last CTA of a row block (atomic ticket) adds them in
//    split order 0..P-1 -> the result is bitwise independent of the grid and of the batch;
//  * epilogues: bf16 / f32 store / f32 residual add / SiLU(gate)*up (interleaved 16-row gate|up
//    blocks) / qkv bias + RoPE + paged-KV append (RB = 128 = one head: warp w and w + 4 hold the
//    two halves of the rotation pairs).
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"

namespace nova {

bool g_use_tma_gemv = true;
int g_dec_tma_mask = getenv("NOVA_DEC_TMA") ? atoi(getenv("NOVA_DEC_TMA")) : -1;  // -1: per-shape rule (stages.cpp)

namespace {

// Ring geometry (scripts/gpu_ring2.sh, decode iterations on 8..112-SM slices and the full GPU):
// 3 stages x one 8 KB weight tile per CTA, 4 CTAs per SM beat 2 x 16 KB (-8% on 32 SMs, -2% full
// GPU), 4 x 8 KB, 3 x 16 KB at 3 CTAs/SM, and 5-6 CTAs/SM: the ring's handoff latency, not the
// bytes in flight, limits a slice -- finer stages release the consumer sooner.
#ifndef GEMV_STAGES
#define GEMV_STAGES 3  // ring stages per CTA
#endif
#ifndef GEMV_SKB64
#define GEMV_SKB64 1   // 64-k blocks per stage (64-row blocks)
#endif
#ifndef GEMV_CPS
#define GEMV_CPS 4     // CTAs per SM of the budget
#endif
constexpr int KC = 64;        // k per stage (128-byte rows -> SWIZZLE_128B)
constexpr int XR = 16;        // x rows per stage tile (batch padded to 16)
constexpr int X_BYTES = XR * KC * 2;

// Ring geometry: ~40 KB per CTA and FOUR CTAs per SM of the budget.  scripts/probe_bw.cu on
// B200 partitions: bulk-copy streaming scales with the number of independent producer CTAs per
// SM (1 CTA x 24 x 8 KB: 77 GB/s/SM; 4 CTAs x 6 x 8 KB: 215 GB/s/SM on a 24-SM slice), not
// with the bytes in flight.
template <int RB, int XHL>
struct PCfg {
  static constexpr int NW = RB / 16;                 // m16 tiles = epilogue warps
  static constexpr int SKB = RB == 64 ? GEMV_SKB64 : 1;  // 64-k blocks per ring stage
  static constexpr int NWC = SKB >= 2 ? 2 * NW : NW; // consumer warps: (m tile, k half)
  static constexpr int KB_W = RB * KC * 2;           // weight bytes per k block
  static constexpr int W_BYTES = SKB * KB_W;
  static constexpr int XT = XHL ? 2 : 1;             // x tiles per k block (hi, lo)
  static constexpr int XS_BYTES = SKB * X_BYTES;     // x bytes per stage (per part)
  static constexpr int STAGES = GEMV_STAGES;
  static constexpr int RED_FLOATS = NW * 2 * 32 * 4; // epilogue exchange (NT <= 2)
  static constexpr int SMEM = 1024 + STAGES * (W_BYTES + XT * XS_BYTES) + 8 * (2 * STAGES) + 64 + 2 * RED_FLOATS * 4;
};

NOVA_DEV float silu_t(float z) { return __fdividef(z, 1.0f + __expf(-z)); }

// address of the 16-byte chunk `c16` of row `r` in a [rows][64] bf16 SWIZZLE_128B tile
NOVA_DEV uint32_t sw128(uint32_t base, int r, int c16) { return base + r * 128 + ((c16 ^ (r & 7)) << 4); }

struct PGemvArgs {
  void* Y;
  const bf16* wblk;  // weights in the streaming layout (block_weights), or null: row-major via tmW
  const bf16* bias;
  float* ws;       // [P][B][N] partials (P > 1)
  int* tickets;    // [N / RB] (P > 1), zero on entry, restored to zero by the last CTA
  int N, K, B, ldy, ks, P, units;
  GemvAux aux;     // EPI_QKV_ROPE_KV / EPI_F32_ARGMAX
};

template <int RB, int NT, int EPI, int XHL>
__global__ void __launch_bounds__(32 * (1 + PCfg<RB, XHL>::NWC), GEMV_CPS) gemv_tma_kernel(const __grid_constant__ CUtensorMap tmW,
                                                                          const __grid_constant__ CUtensorMap tmX,
                                                                          const __grid_constant__ CUtensorMap tmX2,
                                                                          PGemvArgs a) {
  using C = PCfg<RB, XHL>;
  constexpr int STAGES = C::STAGES, NW = C::NW, NWC = C::NWC, SKB = C::SKB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * C::W_BYTES;
  uint8_t* sX2 = sX + STAGES * C::XS_BYTES;  // lo parts (XHL)
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + C::XT * STAGES * C::XS_BYTES);
  uint64_t* empty = full + STAGES;
  int* s_last = reinterpret_cast<int*>(empty + STAGES);
  float* red = reinterpret_cast<float*>(s_last + 16);
  float* redk = red + C::RED_FLOATS;  // k-half partials

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int kblocks = a.K / KC;
  // k blocks of K split p (the last split may be shorter) and its ring stages
  auto unit_kb = [&](int p) {
    const int k0 = p * a.ks, k1 = min(a.K, k0 + a.ks);
    return (k1 - k0 + KC - 1) / KC;
  };
  // The unit sequence of this CTA (the producer and the consumers walk the same one).  With
  // split-K (P > 1) and at least G row blocks, the first R = blocks / G rounds give each CTA WHOLE
  // row blocks: it streams the P splits of a block back to back and adds their partials in
  // split order in registers (0 + s_0 + s_1 + ... -- the same fp32 operations as the workspace
  // reduction, so the result is bitwise the same for any grid) with no workspace round trip,
  // ticket or stall between units; the remaining blocks go out as split units as before.
  const int blocks = a.units / a.P;
  const int R = a.P > 1 ? blocks / G : 0;
  auto unit_at = [&](int i, int& blk, int& p, bool& local) -> bool {
    if (i < R * a.P) {
      blk = (i / a.P) * G + blockIdx.x;
      p = i % a.P;
      local = true;
      return true;
    }
    const int u = blockIdx.x + (i - R * a.P) * G;
    if (u >= (blocks - R * G) * a.P) return false;
    blk = R * G + u / a.P;
    p = u % a.P;
    local = false;
    return true;
  };
  // one ring stage: n k blocks starting at k (global), row block blk
  auto load_stage = [&](int st, int k, int n, int blk, bool with_w, bool with_x) {
    if (with_w) {
      if (a.wblk) {  // streaming layout: the n k blocks of a 64-row block are one contiguous run
#pragma unroll
        for (int b2 = 0; b2 < RB / 64; ++b2)
          bulk_load(sW + st * C::W_BYTES + b2 * SKB * 8192,
                    a.wblk + ((size_t)(blk * (RB / 64) + b2) * kblocks + k / KC) * (64 * KC), n * 8192, &full[st]);
      } else {
        for (int i = 0; i < n; ++i)
          tma_load_2d(sW + st * C::W_BYTES + i * C::KB_W, &tmW, &full[st], k + i * KC, blk * RB);
      }
    }
    if (with_x) {
      for (int i = 0; i < n; ++i) {
        tma_load_2d(sX + st * C::XS_BYTES + i * X_BYTES, &tmX, &full[st], k + i * KC, 0);
        if constexpr (XHL) tma_load_2d(sX2 + st * C::XS_BYTES + i * X_BYTES, &tmX2, &full[st], k + i * KC, 0);
      }
    }
  };
  // weight sub-tile (k block i, m tile t) inside a stage
  auto w_tile = [&](uint32_t stage_base, int i, int t) -> uint32_t {
    return a.wblk ? stage_base + ((t / 4) * SKB + i) * 8192 + (t % 4) * 16 * 128
                  : stage_base + i * C::KB_W + t * 16 * 128;
  };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    if constexpr (XHL) tma_prefetch_desc(&tmX2);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWC);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer: one continuous ring over all units of this CTA
      // pass 1 (before griddepcontrol.wait): weights of the first STAGES ring slots
      int ui = 0, blk = 0, p = 0, kb = 0, i = 0;
      bool loc;
      bool have = unit_at(ui, blk, p, loc);
      int nkb = have ? unit_kb(p) : 0;
      while (have && i < STAGES) {
        const int n = min(SKB, nkb - kb);
        mbar_arrive_expect_tx(&full[i], n * (C::KB_W + C::XT * X_BYTES));
        load_stage(i, p * a.ks + kb * KC, n, blk, true, false);
        ++i;
        kb += n;
        if (kb == nkb) {
          kb = 0;
          have = unit_at(++ui, blk, p, loc);
          nkb = have ? unit_kb(p) : 0;
        }
      }
      pdl_launch_dependents();
      pdl_wait();  // x is written by the previous kernel
      // pass 2: x of those slots, then the steady-state ring
      ui = 0;
      kb = 0;
      have = unit_at(ui, blk, p, loc);
      nkb = have ? unit_kb(p) : 0;
      for (int j = 0; have; ++j) {
        const int st = j % STAGES;
        const int n = min(SKB, nkb - kb);
        const int k = p * a.ks + kb * KC;
        if (j < STAGES) {
          load_stage(st, k, n, blk, false, true);
        } else {
          mbar_wait(&empty[st], ((j / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], n * (C::KB_W + C::XT * X_BYTES));
          load_stage(st, k, n, blk, true, true);
        }
        kb += n;
        if (kb == nkb) {
          kb = 0;
          have = unit_at(++ui, blk, p, loc);
          nkb = have ? unit_kb(p) : 0;
        }
      }
    }
    return;
  }
  // ---------------- consumers: warp (1..NWC): m16 tile t, k half h (odd / even k blocks of a stage)
  pdl_launch_dependents();
  pdl_wait();  // epilogues read / write activations of the previous kernels
  const int t = (warp - 1) % NW, h = NWC > NW ? (warp - 1) / NW : 0;
  const int g = lane >> 2, c = lane & 3;
  int j = 0;  // ring position
  float sum[NT][4];  // whole-block split sum (local units)
  int blk, p;
  bool local;
  for (int ui = 0; unit_at(ui, blk, p, local); ++ui) {
    const int r0 = blk * RB;
    const int nkb = unit_kb(p);
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
    for (int kb = 0; kb < nkb; kb += SKB, ++j) {
      const int stage = j % STAGES;
      const int n = min(SKB, nkb - kb);
      mbar_wait(&full[stage], (j / STAGES) & 1);
      const uint32_t sb = smem_u32(sW + stage * C::W_BYTES);
      for (int i = h; i < n; i += NWC / NW) {
        const uint32_t wb = w_tile(sb, i, t);
        const uint32_t xb = smem_u32(sX + stage * C::XS_BYTES + i * X_BYTES);
#pragma unroll
        for (int kk = 0; kk < KC / 16; ++kk) {
          uint32_t af[4];
          ldmatrix_x4(af, sw128(wb, lane & 15, kk * 2 + (lane >> 4)));
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            uint32_t bfr[2];
            ldmatrix_x2(bfr, sw128(xb, nt * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)));
            mma_bf16_16816(acc[nt], af, bfr);
            if constexpr (XHL) {  // f32 x = hi + lo: second product on the lo part
              ldmatrix_x2(bfr, sw128(xb + STAGES * C::XS_BYTES, nt * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)));
              mma_bf16_16816(acc[nt], af, bfr);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
    }
    // k halves: acc = half 0 + half 1 (fixed order); the half-0 warps run the epilogue
    if constexpr (NWC > NW) {
    if (h == 1) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) redk[((t * NT + nt) * 32 + lane) * 4 + jj] = acc[nt][jj];
    }
    asm volatile("bar.sync 2, %0;" ::"r"(NWC * 32) : "memory");
    if (h == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[nt][jj] += redk[((t * NT + nt) * 32 + lane) * 4 + jj];
    }
    asm volatile("bar.sync 2, %0;" ::"r"(NWC * 32) : "memory");  // redk is reused by the next unit
    if (h == 1) continue;
    }
    // acc[nt]: c0:(row g, batch 2c) c1:(g, 2c+1) c2:(g+8, 2c) c3:(g+8, 2c+1)
    if (local) {  // split partials summed in split order in registers (== the workspace reduction)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) sum[nt][jj] = (p == 0 ? 0.f : sum[nt][jj]) + acc[nt][jj];
      if (p < a.P - 1) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[nt][jj] = sum[nt][jj];
    } else if (a.P > 1) {  // split-K: partials, then the last CTA of the row block reduces in split order
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int b = nt * 8 + 2 * c + (jj & 1);
          if (b < a.B) a.ws[((size_t)p * a.B + b) * a.N + r0 + t * 16 + g + ((jj >> 1) << 3)] = acc[nt][jj];
        }
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
      if (threadIdx.x == 32) *s_last = (atomicAdd(&a.tickets[blk], 1) == a.P - 1);
      asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
      const bool last = *s_last;
      asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");  // s_last is reused by the next unit
      if (!last) continue;
      __threadfence();
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int b = nt * 8 + 2 * c + (jj & 1);
          float s = 0.f;
          if (b < a.B)
            for (int q = 0; q < a.P; ++q)
              s += __ldcg(&a.ws[((size_t)q * a.B + b) * a.N + r0 + t * 16 + g + ((jj >> 1) << 3)]);
          acc[nt][jj] = s;
        }
      if (threadIdx.x == 32) a.tickets[blk] = 0;
    }
    if constexpr (EPI == EPI_BF16_SILUMUL || EPI == EPI_QKV_ROPE_KV) {
      // pair exchange: SILU pairs warp t (gate) with t + 1 (up); RoPE pairs t with t + NW/2
      constexpr int PART = EPI == EPI_BF16_SILUMUL ? 1 : NW / 2;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) red[((t * NT + nt) * 32 + lane) * 4 + jj] = acc[nt][jj];
      asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
      const bool owner = EPI == EPI_BF16_SILUMUL ? !(t & 1) : t < NW / 2;
      if (owner) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int b = nt * 8 + 2 * c + (jj & 1);
            if (b >= a.B) continue;
            const float v2raw = red[(((t + PART) * NT + nt) * 32 + lane) * 4 + jj];
            const int ro = g + ((jj >> 1) << 3);
            if constexpr (EPI == EPI_BF16_SILUMUL) {
              const int n = r0 / 2 + (t / 2) * 16 + ro;
              reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + n] = __float2bfloat16_rn(silu_t(acc[nt][jj]) * v2raw);
            } else {
              const GemvAux& x = a.aux;
              const int hd = x.hd, half = hd / 2;
              const int n1 = r0 + t * 16 + ro, n2 = n1 + half;
              const int hh = n1 / hd, i = n1 % hd;
              float v1 = acc[nt][jj], v2 = v2raw;
              if (a.bias != nullptr) {
                v1 += __bfloat162float(a.bias[n1]);
                v2 += __bfloat162float(a.bias[n2]);
              }
              const DecodeRow rr = x.rows[b];
              if (hh < x.H + x.KV) {  // t = h = w = pos for generated text: plain RoPE at pos
                const float inv = exp2f(-(2.0f * i / hd) * x.log2_theta);
                float sn, cs;
                sincosf((float)rr.pos * inv, &sn, &cs);
                const float o1 = v1 * cs - v2 * sn, o2 = v2 * cs + v1 * sn;
                v1 = o1;
                v2 = o2;
              }
              if (hh < x.H) {
                bf16* q = reinterpret_cast<bf16*>(a.Y) + (size_t)b * a.ldy;
                q[n1] = __float2bfloat16_rn(v1);
                q[n2] = __float2bfloat16_rn(v2);
              } else {
                const int isv = hh >= x.H + x.KV;
                const int kvh = hh - x.H - (isv ? x.KV : 0);
                const size_t page_stride = (size_t)2 * x.KV * 64 * hd;
                bf16* pg = x.pool + ((size_t)x.layer * x.n_pages + x.bt[(size_t)rr.slot * x.max_pages + (rr.ctx >> 6)]) *
                                        page_stride;
                bf16* dst = pg + (((size_t)isv * x.KV + kvh) * 64 + (rr.ctx & 63)) * hd;
                dst[i] = __float2bfloat16_rn(v1);
                dst[i + half] = __float2bfloat16_rn(v2);
              }
            }
          }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");  // red is reused by the next unit
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int b = nt * 8 + 2 * c + (jj & 1);
          if (b >= a.B) continue;
          const int n = r0 + t * 16 + g + ((jj >> 1) << 3);
          float v = acc[nt][jj];
          if (a.bias != nullptr) v += __bfloat162float(a.bias[n]);
          if constexpr (EPI == EPI_BF16) {
            reinterpret_cast<bf16*>(a.Y)[(size_t)b * a.ldy + n] = __float2bfloat16_rn(v);
          } else if constexpr (EPI == EPI_F32_RESID) {
            float* yp = reinterpret_cast<float*>(a.Y) + (size_t)b * a.ldy + n;
            const float h = *yp + v;
            *yp = h;
            if (a.aux.nxout)
              a.aux.nxout[(size_t)b * a.aux.ldnx + n] = __float2bfloat16_rn(h * __bfloat162float(a.aux.ngamma[n]));
          } else {
            reinterpret_cast<float*>(a.Y)[(size_t)b * a.ldy + n] = v;
          }
        }
      if constexpr (EPI == EPI_F32_ARGMAX) {  // greedy pick: packed (ordered logit, ~index) maximum
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int jb = 0; jb < 2; ++jb) {
            const int b = nt * 8 + 2 * c + jb;
            unsigned long long best = 0ull;
#pragma unroll
            for (int jr = 0; jr < 2; ++jr) {
              const int n = r0 + t * 16 + g + 8 * jr;
              uint32_t uu = __float_as_uint(acc[nt][jr * 2 + jb]);
              uu = (uu & 0x80000000u) ? ~uu : (uu | 0x80000000u);
              const unsigned long long key = ((unsigned long long)uu << 32) | (0xFFFFFFFFu - (uint32_t)n);
              best = key > best ? key : best;
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
              const unsigned long long ot = __shfl_xor_sync(0xffffffffu, best, o);
              best = ot > best ? ot : best;
            }
            if (g == 0 && b < a.B) atomicMax(a.aux.keys + b, best);
          }
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

// weight tensor maps are reused every decode iteration: cache by (pointer, N, K, box rows)
std::mutex g_map_mu;
std::unordered_map<uint64_t, CUtensorMap>* g_maps = nullptr;

bool weight_map(CUtensorMap* m, const bf16* W, int N, int K, int RB) {
  const uint64_t key = reinterpret_cast<uint64_t>(W) ^ ((uint64_t)N << 48) ^ ((uint64_t)K << 28) ^ ((uint64_t)RB << 20);
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

template <int RB, int NT, int EPI, int XHL>
cudaError_t launch(const CUtensorMap& mw, const CUtensorMap& mx, const CUtensorMap& mx2, const PGemvArgs& a, int grid,
                   cudaStream_t s) {
  auto kern = gemv_tma_kernel<RB, NT, EPI, XHL>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PCfg<RB, XHL>::SMEM);
    if (e != cudaSuccess) return e;
    set = true;
  }
  return launch_k(kern, dim3(grid), dim3(32 * (1 + PCfg<RB, XHL>::NWC)), PCfg<RB, XHL>::SMEM, s, true, mw, mx, mx2, a);
}

template <int RB, int EPI, int XHL = 0>
cudaError_t launch_nt(const CUtensorMap& mw, const CUtensorMap& mx, const CUtensorMap& mx2, const PGemvArgs& a,
                      int grid, cudaStream_t s) {
  return a.B > 8 ? launch<RB, 2, EPI, XHL>(mw, mx, mx2, a, grid, s) : launch<RB, 1, EPI, XHL>(mw, mx, mx2, a, grid, s);
}

}  // namespace

// Shape-only work decomposition: row block RB (128 for the RoPE epilogue, else 64) and the K
// split P that makes units / 592 (4 CTAs x 148 SMs) closest to a whole number of waves (chunks
// >= 256 k, P <= 8).
GemvTmaPlan gemv_tma_plan(int N, int K, int epi) {
  GemvTmaPlan pl;
  pl.RB = epi == EPI_QKV_ROPE_KV ? 128 : 64;
  const int blocks = N / pl.RB;
  int bestP = 1;
  double best = 1e30;
  // P <= 8: decode iterations on 8..112-SM slices 6-11% (2B) / 0-4% (7B) faster than P <= 16 at equal
  // full-GPU time (scripts/gpu_maxp.sh); env NOVA_GEMV_MAXP is the sweep knob
  static const int env_maxp = getenv("NOVA_GEMV_MAXP") ? atoi(getenv("NOVA_GEMV_MAXP")) : 8;
  const int maxP = epi == EPI_F32_ARGMAX ? 1 : env_maxp;
  for (int P = 1; P <= maxP; ++P) {
    const int ks = ((K + P - 1) / P + KC - 1) / KC * KC;
    const int Pe = (K + ks - 1) / ks;
    if (Pe != P || (P > 1 && ks < 256)) continue;
    const double w = (double)blocks * P / 592.0;
    const double eff = w / (double)((blocks * P + 591) / 592);   // fraction of the last wave used
    const double cost = (1.0 - eff) + 0.01 * P;                  // prefer balance, then fewer splits
    if (cost < best) {
      best = cost;
      bestP = P;
    }
  }
  pl.P = bestP;
  pl.ks = ((K + bestP - 1) / bestP + KC - 1) / KC * KC;
  pl.units = blocks * bestP;
  return pl;
}

int gemv_tma_splits(int N, int K) { return gemv_tma_plan(N, K, EPI_BF16).P; }

cudaError_t gemv_tma(const bf16* X, int ldx, const bf16* W, int N, int K, void* Y, int ldy, const bf16* bias, int B,
                     int epi, float* ws, int* tickets, cudaStream_t s, int max_ctas, const GemvAux* aux,
                     const bf16* W_blocked, const bf16* X_lo) {
  if (B <= 0) return cudaSuccess;
  const GemvTmaPlan pl = gemv_tma_plan(N, K, epi);
  if (B > 16 || N % pl.RB || K % KC || ldx % 8) return cudaErrorInvalidValue;
  if (epi == EPI_QKV_ROPE_KV && (!aux || aux->hd != 128 || !aux->rows || !aux->pool || !aux->bt))
    return cudaErrorInvalidValue;
  if (epi == EPI_F32_ARGMAX && (!aux || !aux->keys || !X_lo)) return cudaErrorInvalidValue;
  CUtensorMap mw, mx, mx2;
  if (!encode(&mx, X, B, K, ldx, XR)) return cudaErrorInvalidValue;
  if (X_lo && !encode(&mx2, X_lo, B, K, ldx, XR)) return cudaErrorInvalidValue;
  if (!X_lo) mx2 = mx;
  if (W_blocked) {
    mw = mx;  // unused: tiles come from the streaming layout by bulk copy
  } else if (!weight_map(&mw, W, N, K, pl.RB)) {
    return cudaErrorInvalidValue;
  }
  if (pl.P > 1 && (!ws || !tickets)) return cudaErrorInvalidValue;
  PGemvArgs a{Y, W_blocked, bias, ws, tickets, N, K, B, ldy, pl.ks, pl.P, pl.units, aux ? *aux : GemvAux{}};
  // four CTAs per SM of the budget (PCfg)
  int grid = GEMV_CPS * (max_ctas > 0 ? max_ctas : 148);
  if (grid > pl.units) grid = pl.units;
  if (X_lo) {  // f32 x given as bf16 hi + lo (decode lm_head)
    if (epi == EPI_F32_ARGMAX) return launch_nt<64, EPI_F32_ARGMAX, 1>(mw, mx, mx2, a, grid, s);
    if (epi == EPI_F32_STORE) return launch_nt<64, EPI_F32_STORE, 1>(mw, mx, mx2, a, grid, s);
    return cudaErrorInvalidValue;
  }
  switch (epi) {
    case EPI_BF16: return launch_nt<64, EPI_BF16>(mw, mx, mx2, a, grid, s);
    case EPI_BF16_SILUMUL: return launch_nt<64, EPI_BF16_SILUMUL>(mw, mx, mx2, a, grid, s);
    case EPI_F32_RESID: return launch_nt<64, EPI_F32_RESID>(mw, mx, mx2, a, grid, s);
    case EPI_F32_STORE: return launch_nt<64, EPI_F32_STORE>(mw, mx, mx2, a, grid, s);
    case EPI_QKV_ROPE_KV: return launch_nt<128, EPI_QKV_ROPE_KV>(mw, mx, mx2, a, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nova
