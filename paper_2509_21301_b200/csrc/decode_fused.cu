// Fused persistent decode iteration (DESIGN.md §5 "dec_fused").
//
// One launch runs a WHOLE LLM decode iteration for a batch of B <= 16 requests:
//
//   embed -> L x [ qkv | attention | o-proj + residual | gate|up + SiLU.mul | down + residual ]
//         -> lm_head + greedy argmax -> tokens
//
// PAPER.md P:88 / P:141 / P:283: decode is memory-bound (86-92% DRAM active on the A6000) and
// Nova runs it on a SLICE of the SMs (Eq. 5).  On B200 the per-op launches of the
// unfused path (~6 per layer) each pay their own fill / drain and single-CTA RMSNorm kernels sit
// between them (2B decode at 30% of HBM solo, 13% inside the serving replay).  Here
// the grid (4 CTAs per SM of the decode partition) stays resident for the whole iteration:
//
//  * every CTA walks the same phase sequence; a CTA that finishes phase k release-adds 1 to
//    phase k's OWN monotone counter, and a phase's inputs are ready once the previous phase's counter
//    reached base + grid (acquire-polled).  One counter per phase, because a CTA with no work in
//    later phases runs ahead and arrives for them at once (a single shared counter would then pass
//    a barrier before slow CTAs finished the phase it guards);
//  * a CTA's producer lane streams its units of EVERY phase through ONE continuous mbarrier ring
//    (3 x 12 KB: an 8 KB pre-swizzled 64x64 weight tile + 16x64 activation tiles), and it issues the
//    weight tiles of the next phase BEFORE the barrier that guards the activations (weights never
//    depend on the iteration) -- the ring stays full across op boundaries;
//  * RMSNorm is folded into its neighbours (an exact reformulation, DESIGN R25): the residual
//    epilogue that finalises a 64-column block also writes x~ = bf16(h * gamma) for the next linear
//    and that block's sum of squares; the next linear contracts W . x~ and scales row b by
//    rsqrt(sum_blocks ss / D + eps) in its epilogue (ss bulk-loaded with its first stage);
//  * attention: units (request b, KV head, 128-key chunk); K/V 16-key tiles (SWIZZLE_128B boxes of
//    the paged pool) flow through the same ring, stage i computed by consumer warp i mod 4
//    (mma.sync m16n8k16, GQA group on M); warp states merged in warp order in shared memory, chunk
//    partials merged in chunk order by the last CTA of (b, KV head) (atomic ticket).  q and the new
//    token's k are M-RoPE'd in this phase (t = h = w for generated text, P:468 / DESIGN R4) from the
//    f32 qkv rows; the new k, v are patched into the staged tile and appended to the page;
//  * every reduction order is a function of the model shape only (K splits, 64-column ss blocks,
//    128-key chunks, warp order), never of the grid or the batch composition, so a request's tokens
//    and logits are bitwise identical on any decode partition (co-execution == serial, §8(c) c6).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace nova {

int g_dec_fused = getenv("NOVA_DEC_FUSED") ? atoi(getenv("NOVA_DEC_FUSED")) : 0;  // measured slower

namespace {

constexpr int CW = 4;                  // consumer warps (one m16 tile of a 64-row block each)
constexpr int NTHR = 32 * (1 + CW);    // + the producer warp
constexpr int KC = 64;                 // k per weight tile
constexpr int W_BYTES = 8192;          // 64 x 64 bf16 weight tile / 16-key K + V tile
constexpr int X_BYTES = 16 * KC * 2;   // 16 x 64 bf16 activation tile
constexpr int STAGE = W_BYTES + 2 * X_BYTES;
constexpr int CK = 128;                // keys per attention unit
constexpr int MAXCH = 64;              // chunks per (request, KV head): contexts <= 8192
constexpr int UNION = 13 * 1024;       // phase-private scratch (see the layout in the kernel)
constexpr int smem_of(int st) { return 1024 + st * STAGE + UNION + 256; }
// ring geometries (env NOVA_DEC_CFG): stages per CTA x CTAs per SM of the partition
constexpr int CFG_ST[4] = {3, 4, 5, 8};
constexpr int CFG_CPS[4] = {4, 3, 3, 2};

enum { PH_EMBED = 0, PH_QKV, PH_ATTN, PH_O, PH_GU, PH_DOWN, PH_LM, PH_FIN };

NOVA_DEV float silu_f(float z) { return __fdividef(z, 1.0f + __expf(-z)); }
NOVA_DEV uint32_t swz(uint32_t base, int r, int c16) { return base + r * 128 + ((c16 ^ (r & 7)) << 4); }

NOVA_DEV void cbar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }  // the 4 consumer warps
NOVA_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
NOVA_DEV unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
NOVA_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// counter >= target?  relaxed polls (no L1 invalidation per spin); acquire ordering once it holds
NOVA_DEV bool bar_reached(const unsigned long long* c, unsigned long long target) {
  if (ld_relaxed_u64(c) < target) return false;
  fence_acq_rel_gpu();
  return true;
}
NOVA_DEV void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
NOVA_DEV void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
NOVA_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
NOVA_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
NOVA_DEV void mbar_arrive_cnt(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}

// 64-row block units of one linear: whole-block rounds first (split partials summed in registers),
// then split units (partials to the workspace, last CTA of the block reduces in split order).
// Same decomposition as gemv_tma (gemv_tma_plan), so the same shape gives the same sums.
NOVA_DEV bool gunit(int i, int blocks, int P, int G, int bx, int& blk, int& p, bool& local) {
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

}  // namespace

struct FdLayer {
  const bf16 *ln1, *ln2, *qkv_b, *qkv_wb, *o_wb, *gu_wb, *down_wb;
};

struct FdMaps {
  CUtensorMap xg, xlo, attn, act, kv;
};

struct FdParams {
  int L, D, H, KV, F, V, B, ldq, nbp, hd;
  float eps, log2_theta, scale_log2;
  const FdLayer* layers;
  const bf16 *embed, *final_norm, *lm_wb;
  float* hid;          // [Bmax][D] f32 residual stream
  bf16 *xg, *xlo;      // [Bmax][D] normed-input tiles (x~ = bf16(h * gamma); lm_head: hi / lo)
  float* qkvf;         // [Bmax][ldq] f32 raw q|k|v (bias added, norm scale applied)
  bf16 *attn, *act;    // [Bmax][H * hd], [Bmax][F]
  float* ss;           // [Bmax][nbp] per-64-column sums of squares of the residual rows
  float* logits;       // [Bmax][V] (written when store_logits)
  unsigned long long* keys;  // [Bmax] greedy argmax, zero on entry, left zero
  float* ws;           // split-K partials
  int* tickets;        // row-block tickets (zero on entry, left zero)
  float* aws;          // attention chunk partials [B][KV][MAXCH][G][hd + 2]
  int* atk;            // attention tickets [B][KV] (zero on entry, left zero)
  unsigned long long* bar;       // [5 L + 2] per-phase arrival counters (monotone)
  unsigned long long bar_base;   // every counter's value at launch (sum of the earlier grids)
  bf16* pool;
  int n_pages, max_pages;
  const int* bt;
  const DecodeRow* rows;
  int* last_tok;
  int* tok_out;
  GemvTmaPlan pq, po, pgu, pd, plm;
  int store_logits;
  int ph_end;          // phases >= ph_end are skipped (debug bisection; 5L + 3 = all)
  uint32_t pf_bytes;   // L2 prefetch budget per CTA per phase (0 = off)
  int dbg;             // debug flags (env NOVA_DEC_FUSED_DBG): 1 sink probes, 2 no early weights, 4 phase timeline
  unsigned long long* tdbg;  // dbg & 4: [3 * phase] = {barrier seen by CTA 0, last CTA arrival, CTA 0 arrival}
  int mch;             // chunk capacity per (request, KV head) of aws
};

namespace {

struct GDesc {
  const bf16* wb;
  const bf16* bias;
  int N, K, P, ks, blocks, norm, xhl;
  const CUtensorMap* mx;
};

template <int NT, int HD, int ST, int CPS>
__global__ void __launch_bounds__(NTHR, CPS)
    decode_fused_kernel(const FdMaps* __restrict__ gmaps, const __grid_constant__ FdParams p) {
  // the tensor maps live in global memory (built once per engine): descriptor addresses taken from
  // a __grid_constant__ struct and carried in a per-phase descriptor were not reliable TMA operands
  const FdMaps& maps = *gmaps;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                         // ST x [W 8 KB | X 2 KB | X2 2 KB]
  uint8_t* uni = smem + ST * STAGE;             // phase-private scratch:
  float* sSS = reinterpret_cast<float*>(uni);                 //   norm phases: ss rows (<= 4 KB)
  float* sRed = reinterpret_cast<float*>(uni + 4096);         //   gate|up exchange [CW][2][32][4] (4 KB)
  float* sRed2 = reinterpret_cast<float*>(uni + 8192);        //   residual ss partials [CW][16]
  bf16* sQ = reinterpret_cast<bf16*>(uni);                    //   attention: Q [16][HD + 8] bf16
  float* sO = reinterpret_cast<float*>(uni + 16 * (HD + 8) * 2);  // [16][HD] f32
  float* sML = sO + 16 * HD;                                  //   [CW][16][2]
  uint64_t* full = reinterpret_cast<uint64_t*>(uni + UNION);
  uint64_t* empty = full + ST;
  int* sflag = reinterpret_cast<int*>(empty + ST);
  int* sCum = sflag + 4;  // [17] attention unit prefix over requests
  volatile int* sPh = sflag + 24;  // phase the consumers are in (prefetch lane pacing)
  static_assert(16 * (HD + 8) * 2 + 16 * HD * 4 + CW * 16 * 2 * 4 <= UNION, "attention scratch");
  static_assert(16 * (HD + 8) * 2 + (2 * MAXCH * 16 + 16) * 4 <= UNION, "attention merge scratch");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, bx = blockIdx.x;
  const int L = p.L, D = p.D, B = p.B;
  const int GQ = p.H / p.KV;  // query heads per KV head
  constexpr int TK = W_BYTES / (4 * HD);     // keys per attention stage (16 at hd 128)

  if ((p.dbg & 4) && bx == 0 && threadIdx.x == 0) p.tdbg[0] = gtimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
    int c = 0;
    for (int b = 0; b < 16; ++b) {
      sCum[b] = c;
      if (b < B) c += p.KV * ((p.rows[b].ctx + 1 + CK - 1) / CK);
    }
    sCum[16] = c;
    *sPh = 0;
  }
  __syncthreads();

  auto phase_of = [&](int ph, int& layer) -> int {
    if (ph == 0) return PH_EMBED;
    if (ph == 5 * L + 1) return PH_LM;
    if (ph == 5 * L + 2) return PH_FIN;
    layer = (ph - 1) / 5;
    return PH_QKV + (ph - 1) % 5;
  };
  auto gdesc = [&](int kind, int l) -> GDesc {
    GDesc d;
    const FdLayer& ly = p.layers[l < L ? l : 0];
    const GemvTmaPlan* pl;
    d.bias = nullptr;
    d.norm = 0;
    d.xhl = 0;
    if (kind == PH_QKV) {
      d.wb = ly.qkv_wb, d.bias = ly.qkv_b, d.N = p.ldq, d.K = D, pl = &p.pq, d.norm = 1, d.mx = &maps.xg;
    } else if (kind == PH_O) {
      d.wb = ly.o_wb, d.N = D, d.K = p.H * HD, pl = &p.po, d.mx = &maps.attn;
    } else if (kind == PH_GU) {
      d.wb = ly.gu_wb, d.N = 2 * p.F, d.K = D, pl = &p.pgu, d.norm = 1, d.mx = &maps.xg;
    } else if (kind == PH_DOWN) {
      d.wb = ly.down_wb, d.N = D, d.K = p.F, pl = &p.pd, d.mx = &maps.act;
    } else {
      d.wb = p.lm_wb, d.N = p.V, d.K = D, pl = &p.plm, d.norm = 1, d.xhl = 1, d.mx = &maps.xg;
    }
    d.P = pl->P;
    d.ks = pl->ks;
    d.blocks = d.N / 64;
    return d;
  };
  auto unit_kb = [&](const GDesc& d, int pp) {
    const int k0 = pp * d.ks, k1 = min(d.K, k0 + d.ks);
    return (k1 - k0) / KC;
  };
  // attention unit u -> (b, KV head, chunk), its key count and stage count
  auto aunit = [&](int u, int& b, int& kvh, int& c, int& nkeys, int& ns) {
    b = 0;
    while (b + 1 < B && sCum[b + 1] <= u) ++b;
    const int Lb = p.rows[b].ctx + 1;
    const int nch = (Lb + CK - 1) / CK;
    const int r = u - sCum[b];
    kvh = r / nch;
    c = r % nch;
    nkeys = min(CK, Lb - c * CK);
    ns = (nkeys + TK - 1) / TK;
  };
  const size_t page_rows = (size_t)2 * p.KV * 64;  // pool rows of hd elements per page (per layer: x n_pages)

  if (warp == 0) {
    if (lane == 0) {
      // ================================================================= producer
      uint32_t j = 0;
      for (int ph = 1; ph <= 5 * L + 1 && ph < p.ph_end; ++ph) {
        int l = 0;
        const int kind = phase_of(ph, l);
        const unsigned long long target = p.bar_base + (unsigned long long)G;
        const unsigned long long* ctr = p.bar + (ph - 1);  // arrivals of the previous phase
        bool passed = false;
        auto wait_bar = [&]() {
          if (!passed) {
            unsigned long long v;
            while ((v = ld_relaxed_u64(ctr)) < target) {
            }
            fence_acq_rel_gpu();
            fence_proxy_async_global();
            passed = true;
            if ((p.dbg & 4) && bx == 0) p.tdbg[3 * ph] = gtimer();
            if ((p.dbg & 1) && bx == 0 && ph < 12) {
              float* o = p.qkvf + (size_t)14 * p.ldq + ph * 3;
              o[0] = ph, o[1] = (float)(target - p.bar_base), o[2] = (float)(v - p.bar_base);  // per-phase counter
            }
          }
        };
        auto wait_slot = [&](uint32_t jj) {
          if (jj >= (uint32_t)ST) mbar_wait(&empty[jj % ST], ((jj / ST) & 1) ^ 1);
        };
        if (kind == PH_ATTN) {
          const int U = sCum[16];
          for (int u = bx; u < U; u += G) {
            int b, kvh, c, nkeys, ns;
            aunit(u, b, kvh, c, nkeys, ns);
            wait_bar();
            const int* btr = p.bt + (size_t)p.rows[b].slot * p.max_pages;
            for (int i = 0; i < ns; ++i, ++j) {
              wait_slot(j);
              const int st = j % ST;
              uint8_t* dst = ring + st * STAGE;
              const int k0 = c * CK + i * TK;
              const size_t rowK = ((size_t)l * p.n_pages + btr[k0 >> 6]) * page_rows + (size_t)kvh * 64 + (k0 & 63);
              const size_t rowV = rowK + (size_t)p.KV * 64;
              const uint32_t qb = i == 0 ? (uint32_t)(GQ * HD * 4) : 0u;  // raw q rows of the group -> X area
              mbar_arrive_expect_tx(&full[st], W_BYTES + qb);
              if (qb) bulk_load(dst + W_BYTES, p.qkvf + (size_t)b * p.ldq + (size_t)kvh * GQ * HD, qb, &full[st]);
              if constexpr (HD >= 64) {
#pragma unroll
                for (int h2 = 0; h2 < HD / 64; ++h2) {
                  tma_load_2d(dst + h2 * (TK * 128), &maps.kv, &full[st], h2 * 64, (int)rowK);
                  tma_load_2d(dst + W_BYTES / 2 + h2 * (TK * 128), &maps.kv, &full[st], h2 * 64, (int)rowV);
                }
              } else {
                bulk_load(dst, p.pool + rowK * HD, TK * HD * 2, &full[st]);
                bulk_load(dst + W_BYTES / 2, p.pool + rowV * HD, TK * HD * 2, &full[st]);
              }
            }
          }
          continue;
        }
        const GDesc d = gdesc(kind, l);
        const uint32_t ssb = d.norm ? (uint32_t)(B * p.nbp * 4) : 0u;
        if (p.dbg & 2) wait_bar();
        // stages whose activation part waits for the barrier: (slot, k, with ss)
        int pend_st[ST], pend_k[ST], pend_ss[ST];
        int np = 0;
        auto issue_x = [&](int st, int k, int with_ss) {
          uint8_t* dst = ring + st * STAGE + W_BYTES;
          if (p.dbg & 8) {  // timing experiment: no activation tiles (wrong results)
            if (with_ss) bulk_load(sSS, p.ss, ssb, &full[st]);
            return;
          }
          tma_load_2d(dst, d.mx, &full[st], k, 0);
          if (d.xhl) tma_load_2d(dst + X_BYTES, &maps.xlo, &full[st], k, 0);
          if (with_ss) bulk_load(sSS, p.ss, ssb, &full[st]);
        };
        auto flush = [&]() {
          for (int q = 0; q < np; ++q) issue_x(pend_st[q], pend_k[q], pend_ss[q]);
          np = 0;
        };
        bool first = true;
        int blk, pp;
        bool loc;
        for (int ui = 0; gunit(ui, d.blocks, d.P, G, bx, blk, pp, loc); ++ui) {
          const int nkb = unit_kb(d, pp);
          for (int kb = 0; kb < nkb; ++kb, ++j) {
            const int st = j % ST;
            if (j >= (uint32_t)ST) {  // wait for the slot; meanwhile release deferred activations
              const uint32_t a = smem_u32(&empty[st]), par = ((j / ST) & 1) ^ 1;
              while (!mbar_try_wait(a, par)) {
                if (np && bar_reached(ctr, target)) {
                  fence_proxy_async_global();
                  passed = true;
                  if ((p.dbg & 4) && bx == 0) p.tdbg[3 * ph] = gtimer();
                  flush();
                }
              }
            }
            const int k = pp * d.ks + kb * KC;
            mbar_arrive_expect_tx(&full[st], W_BYTES + ((p.dbg & 8) ? 0 : (1 + d.xhl) * X_BYTES) + (first ? ssb : 0u));
            bulk_load(ring + st * STAGE, d.wb + ((size_t)blk * (d.K / KC) + k / KC) * (64 * KC), W_BYTES, &full[st]);
            if (!passed && bar_reached(ctr, target)) {
              fence_proxy_async_global();
              passed = true;
              if ((p.dbg & 4) && bx == 0) p.tdbg[3 * ph] = gtimer();
            }
            if (passed) {
              flush();
              issue_x(st, k, first && ssb);
            } else {
              pend_st[np] = st, pend_k[np] = k, pend_ss[np] = first && ssb, ++np;
            }
            first = false;
          }
        }
        if (np) {
          wait_bar();
          flush();
        }
      }
    } else if (lane == 1 && p.pf_bytes > 0) {
      // ================================================================= L2 prefetch lane
      // While the consumers work on phase ph, pull this CTA's weights (or K/V rows) of phase ph + 1
      // into L2, up to pf_bytes: HBM keeps streaming through barriers and latency-bound phases, and
      // the next phase's ring loads hit L2.  Weights never depend on the iteration; K/V rows only
      // warm L2 (the step's own token is patched in from the qkv rows).
      for (int ph = 1; ph <= 5 * L + 1 && ph < p.ph_end; ++ph) {
        while (*sPh < ph - 1) __nanosleep(200);
        int l = 0;
        const int kind = phase_of(ph, l);
        uint32_t budget = p.pf_bytes;
        if (kind == PH_ATTN) {
          const int U = sCum[16];
          for (int u = bx; u < U && budget > 0; u += G) {
            int b, kvh, c, nkeys, ns;
            aunit(u, b, kvh, c, nkeys, ns);
            const int* btr = p.bt + (size_t)p.rows[b].slot * p.max_pages;
            for (int k0 = c * CK; k0 < c * CK + nkeys; k0 += 64) {
              const size_t rowK = ((size_t)l * p.n_pages + btr[k0 >> 6]) * page_rows + (size_t)kvh * 64;
              l2_prefetch(p.pool + rowK * HD, 64 * HD * 2);
              l2_prefetch(p.pool + (rowK + (size_t)p.KV * 64) * HD, 64 * HD * 2);
            }
            budget = budget > 2u * CK * HD * 2 ? budget - 2u * CK * HD * 2 : 0u;
          }
          continue;
        }
        const GDesc d = gdesc(kind, l);
        int blk, pp;
        bool loc;
        for (int ui = 0; budget > 0 && gunit(ui, d.blocks, d.P, G, bx, blk, pp, loc); ++ui) {
          const uint32_t n = min((uint32_t)unit_kb(d, pp) * W_BYTES, budget);
          l2_prefetch(d.wb + ((size_t)blk * (d.K / KC) + (pp * d.ks) / KC) * (64 * KC), n);
          budget -= n;
        }
      }
    }
    return;
  }

  // =================================================================== consumers (warps 1..4)
  const int t = warp - 1, ct = threadIdx.x - 32;  // warp's m16 tile / consumer thread index
  const int g = lane >> 2, c4 = lane & 3;
  uint32_t j = 0;
  // dbg & 4: latest time (over CTAs, so the last layer's) each milestone m of phase kind k was reached
  auto mark = [&](int k, int m) {
    if ((p.dbg & 4) && ct == 0) atomicMax(p.tdbg + 1024 + k * 8 + m, gtimer());
  };
  for (int ph = 0; ph <= 5 * L + 2 && ph < p.ph_end; ++ph) {
    int l = 0;
    const int kind = phase_of(ph, l);
    if (ct == 0) *sPh = ph;
    if (kind == PH_FIN) {
      if (bx == 0) {
        if (ct == 0) {
          const unsigned long long target = p.bar_base + (unsigned long long)G;
          while (!bar_reached(p.bar + (ph - 1), target)) {
          }
        }
        cbar();
        if (ct < B) {
          const unsigned long long key = atomicExch(p.keys + ct, 0ull);
          const int tok = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
          p.tok_out[ct] = tok;
          p.last_tok[p.rows[ct].slot] = tok;
        }
      }
      break;
    }
    if (kind == PH_EMBED) {
      // hid = Embed[last token]; x~ = bf16(hid * ln1[0]); ss per 64-column block (fixed order)
      const bf16* gam = p.layers[0].ln1;
      for (int cb = bx; cb < D / 64; cb += G) {
        const int b = ct >> 3, col = cb * 64 + (ct & 7) * 8;
        float sq = 0.f;
        if (b < B) {
          const int tok = p.last_tok[p.rows[b].slot];
          const uint4 e = *reinterpret_cast<const uint4*>(p.embed + (size_t)tok * D + col);
          const uint4 gg = *reinterpret_cast<const uint4*>(gam + col);
          const uint32_t* ew = reinterpret_cast<const uint32_t*>(&e);
          const uint32_t* gw = reinterpret_cast<const uint32_t*>(&gg);
          float h[8];
          uint32_t xo[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 ef = unpack_bf16(ew[i]), gf = unpack_bf16(gw[i]);
            h[2 * i] = ef.x;
            h[2 * i + 1] = ef.y;
            xo[i] = pack_bf16(ef.x * gf.x, ef.y * gf.y);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) sq += h[i] * h[i];
          float4* hp = reinterpret_cast<float4*>(p.hid + (size_t)b * D + col);
          hp[0] = make_float4(h[0], h[1], h[2], h[3]);
          hp[1] = make_float4(h[4], h[5], h[6], h[7]);
          *reinterpret_cast<uint4*>(p.xg + (size_t)b * D + col) = make_uint4(xo[0], xo[1], xo[2], xo[3]);
        }
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        sq += __shfl_xor_sync(0xffffffffu, sq, 4);
        if ((ct & 7) == 0 && b < B) p.ss[(size_t)b * p.nbp + cb] = sq;
      }
    } else if (kind == PH_ATTN) {
      // ------------------------------------------------------------- paged GQA attention
      constexpr int HDP = HD + 8, KT = HD / 16, DT = HD / 8, NKT = TK / 8, PKT = TK / 16;
      const int U = sCum[16];
      const int H = p.H, KV = p.KV;
      const int Ghd = 32 + GQ * HD;  // chunk partial: m[16] | l[16] | o[GQ][HD] (o 16-byte aligned)
      for (int u = bx; u < U; u += G) {
        int b, kvh, c, nkeys, ns;
        aunit(u, b, kvh, c, nkeys, ns);
        const DecodeRow rr = p.rows[b];
        const int Lb = rr.ctx + 1;
        const int nch = (Lb + CK - 1) / CK;
        const uint32_t j0 = j;
        // stage 0 landed => the grid barrier passed (the producer issued it after acquiring)
        if (t == 0) mbar_wait(&full[j0 % ST], (j0 / ST) & 1);
        mark(PH_ATTN, 0);
        cbar();
        // Q rows of this KV head's query group, M-RoPE (t = h = w = pos), bf16, rows >= GQ zero
        {
          const float* qr = reinterpret_cast<const float*>(ring + (j0 % ST) * STAGE + W_BYTES);  // bulk-loaded
          for (int i = ct; i < 16 * (HD / 2); i += 128) {
            const int r = i / (HD / 2), d = i % (HD / 2);
            float o1 = 0.f, o2 = 0.f;
            if (r < GQ) {
              const float v1 = qr[r * HD + d], v2 = qr[r * HD + d + HD / 2];
              const float inv = exp2f(-(2.0f * d / HD) * p.log2_theta);
              float sn, cs;
              sincosf((float)rr.pos * inv, &sn, &cs);
              o1 = v1 * cs - v2 * sn;
              o2 = v2 * cs + v1 * sn;
            }
            sQ[r * HDP + d] = __float2bfloat16_rn(o1);
            sQ[r * HDP + d + HD / 2] = __float2bfloat16_rn(o2);
          }
        }
        cbar();
        mark(PH_ATTN, 1);
        float mx[2] = {-1e30f, -1e30f}, ls[2] = {0.f, 0.f};
        float o[DT][4];
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
        // Every warp waits on every stage in ring order and releases it (count CW per stage), and
        // only the stage's owner (i mod CW) computes on it: a warp that skipped ahead to a slot whose
        // previous use had not completed could not tell the two phases apart by parity.
        for (int i = 0; i < ns; ++i) {
          const uint32_t jj = j0 + i;
          const int st = jj % ST;
          mbar_wait(&full[st], (jj / ST) & 1);
          if (i % CW != t) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            continue;
          }
          uint8_t* sK = ring + st * STAGE;
          uint8_t* sV = sK + W_BYTES / 2;
          const uint32_t kb_ = smem_u32(sK), vb_ = smem_u32(sV);
          auto kv_addr = [&](uint32_t base, int r, int c16) -> uint32_t {  // 16-byte chunk c16 of key row r
            if constexpr (HD >= 64) return swz(base + (c16 >> 3) * (TK * 128), r, c16 & 7);
            else return base + r * (HD * 2) + c16 * 16;
          };
          const int k0 = c * CK + i * TK;
          // tail keys past the context: zero V (P = 0 there, but 0 * NaN from stale pages is NaN)
          if (k0 + TK > Lb) {
            for (int e = lane; e < TK * (HD / 8); e += 32) {
              const int r = e / (HD / 8), cc = e % (HD / 8);
              if (k0 + r >= Lb) *reinterpret_cast<uint4*>(sV + (kv_addr(vb_, r, cc) - vb_)) = make_uint4(0, 0, 0, 0);
            }
          }
          // the token of this step (cache index Lb - 1): M-RoPE'd k and v from the qkv rows
          if (k0 <= Lb - 1 && Lb - 1 < k0 + TK) {
            const int r = Lb - 1 - k0;
            const float* kr = p.qkvf + (size_t)b * p.ldq + (size_t)(H + kvh) * HD;
            const float* vr = p.qkvf + (size_t)b * p.ldq + (size_t)(H + KV + kvh) * HD;
            const int* btr = p.bt + (size_t)rr.slot * p.max_pages;
            bf16* pg = p.pool + (((size_t)l * p.n_pages + btr[rr.ctx >> 6]) * page_rows) * HD;
            bf16* gk = pg + ((size_t)kvh * 64 + (rr.ctx & 63)) * HD;
            bf16* gv = gk + (size_t)KV * 64 * HD;
            for (int d = lane; d < HD / 2; d += 32) {
              const float v1 = __ldcg(kr + d), v2 = __ldcg(kr + d + HD / 2);
              const float inv = exp2f(-(2.0f * d / HD) * p.log2_theta);
              float sn, cs;
              sincosf((float)rr.pos * inv, &sn, &cs);
              const bf16 k1 = __float2bfloat16_rn(v1 * cs - v2 * sn), k2 = __float2bfloat16_rn(v2 * cs + v1 * sn);
              const bf16 w1 = __float2bfloat16_rn(__ldcg(vr + d)), w2 = __float2bfloat16_rn(__ldcg(vr + d + HD / 2));
              const int d2 = d + HD / 2;
              *reinterpret_cast<bf16*>(sK + (kv_addr(kb_, r, d >> 3) - kb_) + (d & 7) * 2) = k1;
              *reinterpret_cast<bf16*>(sK + (kv_addr(kb_, r, d2 >> 3) - kb_) + (d2 & 7) * 2) = k2;
              *reinterpret_cast<bf16*>(sV + (kv_addr(vb_, r, d >> 3) - vb_) + (d & 7) * 2) = w1;
              *reinterpret_cast<bf16*>(sV + (kv_addr(vb_, r, d2 >> 3) - vb_) + (d2 & 7) * 2) = w2;
              gk[d] = k1;
              gk[d2] = k2;
              gv[d] = w1;
              gv[d2] = w2;
            }
          }
          __syncwarp();
          // S = Q K^T (16 x TK), rows g / g + 8, keys k0 + nt * 8 + 2 c + (e & 1)
          float sc[NKT][4];
#pragma unroll
          for (int nt = 0; nt < NKT; ++nt) {
            sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
              uint32_t qa[4], bb[2];
              ldmatrix_x4(qa, smem_u32(sQ + (lane & 15) * HDP + kk * 16 + (lane >> 4) * 8));
              ldmatrix_x2(bb, kv_addr(kb_, nt * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)));
              mma_bf16_16816(sc[nt], qa, bb);
            }
          }
          float bm[2] = {-1e30f, -1e30f};
#pragma unroll
          for (int nt = 0; nt < NKT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const bool ok = k0 + nt * 8 + 2 * c4 + (e & 1) < Lb;
              sc[nt][e] = ok ? sc[nt][e] * p.scale_log2 : -1e30f;
              bm[e >> 1] = fmaxf(bm[e >> 1], sc[nt][e]);
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
          uint32_t pa[PKT][4];
#pragma unroll
          for (int nt = 0; nt < NKT; ++nt) {
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
          for (int kk = 0; kk < PKT; ++kk)
#pragma unroll
            for (int dt = 0; dt < DT; ++dt) {
              uint32_t bb[2];
              ldmatrix_x2_trans(bb, kv_addr(vb_, kk * 16 + (lane & 15), dt));
              mma_bf16_16816(o[dt], pa[kk], bb);
            }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
        }
        j = j0 + ns;
        mark(PH_ATTN, 2);
        // CTA state: warp states merged in warp order (m = max, then sum_w f_w o_w sequentially)
        if (c4 == 0) {
          sML[(t * 16 + g) * 2] = mx[0];
          sML[(t * 16 + g) * 2 + 1] = ls[0];
          sML[(t * 16 + g + 8) * 2] = mx[1];
          sML[(t * 16 + g + 8) * 2 + 1] = ls[1];
        }
        cbar();
        float fw[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int row = g + 8 * r;
          float M = -1e30f;
#pragma unroll
          for (int w = 0; w < CW; ++w) M = fmaxf(M, sML[(w * 16 + row) * 2]);
          fw[r] = exp2f((r ? mx[1] : mx[0]) - M);
        }
#pragma unroll
        for (int w = 0; w < CW; ++w) {
          if (t == w) {
#pragma unroll
            for (int dt = 0; dt < DT; ++dt)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int row = g + 8 * (e >> 1), col = dt * 8 + 2 * c4 + (e & 1);
                const float v = fw[e >> 1] * o[dt][e];
                sO[row * HD + col] = w == 0 ? v : sO[row * HD + col] + v;
              }
          }
          cbar();
        }
        // chunk partial -> workspace: m[16] | l[16] | o[GQ][HD]
        float* part = p.aws + (((size_t)b * KV + kvh) * p.mch + c) * Ghd;
        if (ct < GQ) {
          float M = -1e30f;
          for (int w = 0; w < CW; ++w) M = fmaxf(M, sML[(w * 16 + ct) * 2]);
          float lsum = 0.f;
          for (int w = 0; w < CW; ++w) lsum += exp2f(sML[(w * 16 + ct) * 2] - M) * sML[(w * 16 + ct) * 2 + 1];
          part[ct] = M;
          part[16 + ct] = lsum;
        }
        for (int i = ct; i < GQ * HD / 4; i += 128)
          reinterpret_cast<float4*>(part + 32)[i] = reinterpret_cast<const float4*>(sO)[i];  // rows < GQ of [16][HD]
        __threadfence();
        cbar();
        if (ct == 0) sflag[0] = atomicAdd(p.atk + b * KV + kvh, 1) == nch - 1;
        cbar();
        const bool last = sflag[0];
        cbar();  // sflag / sO reused below and by the next unit
        mark(PH_ATTN, 3);
        if (!last) continue;
        __threadfence();
        // merge the chunk partials in chunk order: f[c][row] = 2^(m_c - M), den = sum_c f l_c.
        // (m, l) of every chunk fetched in parallel into smem first; the o sums keep 8 loads in flight.
        float* sF = sO;                   // [MAXCH][16]: m_c, then f_c
        float* sLc = sO + MAXCH * 16;     // [MAXCH][16]: l_c
        float* sDen = sLc + MAXCH * 16;   // [16]
        const float* base = p.aws + ((size_t)b * KV + kvh) * p.mch * Ghd;
        for (int i = ct; i < nch * GQ; i += 128) {
          const int cc = i / GQ, row = i % GQ;
          sF[cc * 16 + row] = __ldcg(base + (size_t)cc * Ghd + row);
          sLc[cc * 16 + row] = __ldcg(base + (size_t)cc * Ghd + 16 + row);
        }
        cbar();
        if (ct < GQ) {
          float M = -1e30f;
          for (int cc = 0; cc < nch; ++cc) M = fmaxf(M, sF[cc * 16 + ct]);
          float den = 0.f;
          for (int cc = 0; cc < nch; ++cc) {
            const float f = exp2f(sF[cc * 16 + ct] - M);
            sF[cc * 16 + ct] = f;
            den += f * sLc[cc * 16 + ct];
          }
          sDen[ct] = den;
        }
        cbar();
        // 4 consecutive dims per thread; the chunk loads of a batch of 16 chunks all in flight
        for (int i = ct; i < GQ * HD / 4; i += 128) {
          const int row = (i * 4) / HD, d = (i * 4) % HD;
          const float4* src = reinterpret_cast<const float4*>(base + 32) + i;
          float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int c0 = 0; c0 < nch; c0 += 16) {
            float4 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              v[q] = c0 + q < nch ? __ldcg(src + (size_t)(c0 + q) * (Ghd / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c0 + q < nch) {
                const float f = sF[(c0 + q) * 16 + row];
                num.x += f * v[q].x, num.y += f * v[q].y, num.z += f * v[q].z, num.w += f * v[q].w;
              }
          }
          const float inv = 1.0f / sDen[row];
          bf16* dst = p.attn + (size_t)b * H * HD + (size_t)(kvh * GQ + row) * HD + d;
          *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(num.x * inv, num.y * inv), pack_bf16(num.z * inv, num.w * inv));
        }
        if (ct == 0) p.atk[b * KV + kvh] = 0;
        cbar();  // sF reused by the next unit
        mark(PH_ATTN, 4);
      }
    } else {
      // ------------------------------------------------------------- linear (64-row blocks)
      const GDesc d = gdesc(kind, l);
      float invb[NT][2];
      bool have_inv = false;
      float sum[NT][4];
      int blk, pp;
      bool local;
      if ((p.dbg & 1) && bx == 0 && ct == 0 && ph < 10) {  // debug sink: qkvf row 15
        const bool has = gunit(0, d.blocks, d.P, G, bx, blk, pp, local);
        float* o = p.qkvf + (size_t)15 * p.ldq + ph * 12;
        o[0] = ph, o[1] = kind, o[2] = d.N, o[3] = d.K, o[4] = d.P, o[5] = d.ks, o[6] = d.blocks, o[7] = G;
        o[8] = has, o[9] = blk, o[10] = pp, o[11] = has ? unit_kb(d, pp) : -1;
      }
      for (int ui = 0; gunit(ui, d.blocks, d.P, G, bx, blk, pp, local); ++ui) {
        const int r0 = blk * 64;
        const int nkb = unit_kb(d, pp);
        // residual phases: this block's rows of the residual stream, requested before the mainloop
        // (last written >= 2 barriers ago; only this block's epilogue writes them in this phase)
        float hpre[NT][4];
        if (kind == PH_O || kind == PH_DOWN) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int b = nt * 8 + 2 * c4 + (e & 1);
              hpre[nt][e] = b < B ? __ldcg(p.hid + (size_t)b * D + r0 + t * 16 + g + ((e >> 1) << 3)) : 0.f;
            }
        }
        float acc[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
        for (int kb = 0; kb < nkb; ++kb, ++j) {
          const int st = j % ST;
          mbar_wait(&full[st], (j / ST) & 1);
          if (kb == 0 && ui == 0) mark(kind, 0);
          if (d.norm && !have_inv) {  // rsqrt(mean of squares + eps) of each row, block sums in order
            float iv = 0.f;
            if (lane < B) {
              float s = 0.f;
              for (int q = 0; q < D / 64; ++q) s += sSS[lane * p.nbp + q];
              iv = rsqrtf(s / (float)D + p.eps);
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              invb[nt][0] = __shfl_sync(0xffffffffu, iv, nt * 8 + 2 * c4);
              invb[nt][1] = __shfl_sync(0xffffffffu, iv, nt * 8 + 2 * c4 + 1);
            }
            have_inv = true;
          }
          const uint32_t wb = smem_u32(ring + st * STAGE) + t * 16 * 128;
          const uint32_t xb = smem_u32(ring + st * STAGE + W_BYTES);
#pragma unroll
          for (int kk = 0; kk < KC / 16; ++kk) {
            if (p.dbg & 16) break;  // timing experiment: no math (wrong results)
            uint32_t af[4];
            ldmatrix_x4(af, swz(wb, lane & 15, kk * 2 + (lane >> 4)));
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              uint32_t bfr[2];
              ldmatrix_x2(bfr, swz(xb, nt * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)));
              mma_bf16_16816(acc[nt], af, bfr);
              if (d.xhl) {  // f32 x = hi + lo: second product on the lo tile
                ldmatrix_x2(bfr, swz(xb + X_BYTES, nt * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)));
                mma_bf16_16816(acc[nt], af, bfr);
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
        }
        mark(kind, 1);
        // acc[nt]: e0 (row g, batch 2c) e1 (g, 2c+1) e2 (g+8, 2c) e3 (g+8, 2c+1)
        if (local) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) sum[nt][e] = (pp == 0 ? 0.f : sum[nt][e]) + acc[nt][e];
          if (pp < d.P - 1) continue;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[nt][e] = sum[nt][e];
        } else if (d.P > 1) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int b = nt * 8 + 2 * c4 + (e & 1);
              if (b < B) p.ws[((size_t)pp * B + b) * d.N + r0 + t * 16 + g + ((e >> 1) << 3)] = acc[nt][e];
            }
          __threadfence();
          cbar();
          if (ct == 0) sflag[0] = (atomicAdd(&p.tickets[blk], 1) == d.P - 1);
          cbar();
          const bool last = sflag[0];
          cbar();
          if (!last) continue;
          __threadfence();
          // all split partials requested at once (one L2 round trip), then summed in split order
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int b = nt * 8 + 2 * c4 + (e & 1);
              const float* src = p.ws + (size_t)b * d.N + r0 + t * 16 + g + ((e >> 1) << 3);
              float v[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) v[q] = (b < B && q < d.P) ? __ldcg(src + (size_t)q * B * d.N) : 0.f;
              float s = 0.f;
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (q < d.P) s += v[q];
              acc[nt][e] = s;
            }
          if (ct == 0) p.tickets[blk] = 0;
        }
        mark(kind, 2);
        // ---- epilogues
        if (kind == PH_QKV) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int b = nt * 8 + 2 * c4 + (e & 1);
              if (b >= B) continue;
              const int n = r0 + t * 16 + g + ((e >> 1) << 3);
              p.qkvf[(size_t)b * p.ldq + n] = acc[nt][e] * invb[nt][e & 1] + __bfloat162float(d.bias[n]);
            }
        } else if (kind == PH_GU) {
          // rows interleave 16 gate | 16 up: warp t (gate, even) pairs with warp t + 1 (up)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) sRed[((t * 2 + nt) * 32 + lane) * 4 + e] = acc[nt][e];
          cbar();
          if (!(t & 1)) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int b = nt * 8 + 2 * c4 + (e & 1);
                if (b >= B) continue;
                const float up = sRed[(((t + 1) * 2 + nt) * 32 + lane) * 4 + e] * invb[nt][e & 1];
                const int n = r0 / 2 + (t / 2) * 16 + g + ((e >> 1) << 3);
                p.act[(size_t)b * p.F + n] = __float2bfloat16_rn(silu_f(acc[nt][e] * invb[nt][e & 1]) * up);
              }
          }
          cbar();
        } else if (kind == PH_LM) {
          const bool stl = p.store_logits;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int jb = 0; jb < 2; ++jb) {
              const int b = nt * 8 + 2 * c4 + jb;
              unsigned long long best = 0ull;
#pragma unroll
              for (int jr = 0; jr < 2; ++jr) {
                const int n = r0 + t * 16 + g + 8 * jr;
                const float v = acc[nt][jr * 2 + jb] * invb[nt][jb];
                if (stl && b < B) p.logits[(size_t)b * p.V + n] = v;
                uint32_t uu = __float_as_uint(v);
                uu = (uu & 0x80000000u) ? ~uu : (uu | 0x80000000u);
                const unsigned long long key = ((unsigned long long)uu << 32) | (0xFFFFFFFFu - (uint32_t)n);
                best = key > best ? key : best;
              }
#pragma unroll
              for (int o = 4; o < 32; o <<= 1) {
                const unsigned long long ot = __shfl_xor_sync(0xffffffffu, best, o);
                best = ot > best ? ot : best;
              }
              if (g == 0 && b < B) atomicMax(p.keys + b, best);
            }
        } else {
          // residual add (o-proj, down) + the next norm's input tile and block sum of squares:
          // o-proj -> ln2 of this layer; down -> ln1 of the next layer, or the final norm as f32
          // hi / lo tiles for the lm_head.
          const bool fin = kind == PH_DOWN && l == L - 1;
          const bf16* gam = kind == PH_O ? p.layers[l].ln2 : (fin ? p.final_norm : p.layers[l + 1 < L ? l + 1 : 0].ln1);
          float sq[NT][2];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            sq[nt][0] = sq[nt][1] = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int b = nt * 8 + 2 * c4 + (e & 1);
              if (b >= B) continue;
              const int n = r0 + t * 16 + g + ((e >> 1) << 3);
              const float h = hpre[nt][e] + acc[nt][e];
              p.hid[(size_t)b * D + n] = h;
              const float xf = h * __bfloat162float(gam[n]);
              const bf16 hi = __float2bfloat16_rn(xf);
              p.xg[(size_t)b * D + n] = hi;
              if (fin) p.xlo[(size_t)b * D + n] = __float2bfloat16_rn(xf - __bfloat162float(hi));
              sq[nt][e & 1] += h * h;
            }
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int jb = 0; jb < 2; ++jb) {
              float v = sq[nt][jb];
              v += __shfl_xor_sync(0xffffffffu, v, 4);
              v += __shfl_xor_sync(0xffffffffu, v, 8);
              v += __shfl_xor_sync(0xffffffffu, v, 16);
              if (g == 0) sRed2[t * 16 + nt * 8 + 2 * c4 + jb] = v;
            }
          cbar();
          if (ct < B) p.ss[(size_t)ct * p.nbp + blk] = (sRed2[ct] + sRed2[16 + ct]) + (sRed2[32 + ct] + sRed2[48 + ct]);
          cbar();
        }
      }
    }
    // ---- phase end: publish this CTA's writes (generic and, for TMA readers, async proxy)
    fence_proxy_async_global();
    __threadfence();
    cbar();
    if (ct == 0) {
      red_release_add(p.bar + ph, 1ull);
      if (p.dbg & 4) {
        const unsigned long long now = gtimer();
        atomicMax(p.tdbg + 3 * ph + 1, now);
        if (bx == 0) p.tdbg[3 * ph + 2] = now;
      }
    }
  }
  // debug bisection: arrive for the skipped phases so every counter advances by the grid per launch
  if (ct == 0)
    for (int ph = p.ph_end; ph <= 5 * L + 1; ++ph) red_release_add(p.bar + ph, 1ull);
}

std::mutex g_fd_mu;

template <int NT, int HD, int ST, int CPS>
cudaError_t fd_launch(const FdMaps* m, const FdParams& p, int grid, cudaStream_t s) {
  auto kern = decode_fused_kernel<NT, HD, ST, CPS>;
  static bool set = false;
  {
    std::lock_guard<std::mutex> g(g_fd_mu);
    if (!set) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_of(ST));
      if (e != cudaSuccess) return e;
      set = true;
    }
  }
  return launch_k(kern, dim3(grid), dim3(NTHR), smem_of(ST), s, false, m, p);
}
template <int NT, int HD>
cudaError_t fd_launch_cfg(int cfg, const FdMaps* m, const FdParams& p, int sms, cudaStream_t s) {
  switch (cfg) {
    case 1: return fd_launch<NT, HD, CFG_ST[1], CFG_CPS[1]>(m, p, CFG_CPS[1] * sms, s);
    case 2: return fd_launch<NT, HD, CFG_ST[2], CFG_CPS[2]>(m, p, CFG_CPS[2] * sms, s);
    case 3: return fd_launch<NT, HD, CFG_ST[3], CFG_CPS[3]>(m, p, CFG_CPS[3] * sms, s);
  }
  return fd_launch<NT, HD, CFG_ST[0], CFG_CPS[0]>(m, p, CFG_CPS[0] * sms, s);
}
int fd_cfg() {
  static const int c = getenv("NOVA_DEC_CFG") ? std::max(0, std::min(3, atoi(getenv("NOVA_DEC_CFG")))) : 0;
  return c;
}

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool enc2d(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_elems, uint32_t box_rows) {
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
  cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)KC, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool decode_fused_supported(int D, int H, int KV, int hd, int F, int V) {
  if (hd != 128 && hd != 32) return false;
  if (D % 64 || F % 64 || V % 64 || (H * hd) % 64 || ((H + 2 * KV) * hd) % 64 || H % KV) return false;
  if (H / KV > 16 || D > 4096) return false;
  return true;
}

int decode_fused_smem() { return smem_of(CFG_ST[fd_cfg()]); }
int decode_fused_grid(int sms) { return CFG_CPS[fd_cfg()] * (sms > 0 ? sms : 148); }
int decode_fused_phase_chunk() { return CK; }

// Host side: the tensor maps of the activation tiles and of the paged pool, built once per engine.
struct DecFusedState {
  FdMaps maps;
  FdMaps* d_maps = nullptr;  // device copy (64-byte aligned: cudaMalloc)
  FdLayer* d_layers = nullptr;
};

DecFusedState* decode_fused_create(const DecFusedSetup& su) {
  if (!decode_fused_supported(su.D, su.H, su.KV, su.hd, su.F, su.V)) return nullptr;
  DecFusedState* st = new DecFusedState();
  bool ok = enc2d(&st->maps.xg, su.xg, su.bmax, su.D, su.D, 16) && enc2d(&st->maps.xlo, su.xlo, su.bmax, su.D, su.D, 16) &&
            enc2d(&st->maps.attn, su.attn, su.bmax, su.H * su.hd, su.H * su.hd, 16) &&
            enc2d(&st->maps.act, su.act, su.bmax, su.F, su.F, 16);
  if (ok && su.hd >= 64) {
    const int TKh = W_BYTES / (4 * su.hd);
    const uint64_t rows = (uint64_t)su.L * su.n_pages * 2 * su.KV * 64;
    ok = enc2d(&st->maps.kv, su.pool, rows, su.hd, su.hd, TKh);
  } else {
    st->maps.kv = st->maps.xg;  // unused (hd 32: bulk copies)
  }
  std::vector<FdLayer> ly(su.L);
  for (int l = 0; l < su.L && ok; ++l)
    ly[l] = FdLayer{su.ln1[l], su.ln2[l], su.qkv_b[l], su.qkv_wb[l], su.o_wb[l], su.gu_wb[l], su.down_wb[l]};
  if (ok) ok = cudaMalloc(&st->d_maps, sizeof(FdMaps)) == cudaSuccess;
  if (ok) ok = cudaMemcpy(st->d_maps, &st->maps, sizeof(FdMaps), cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok) ok = cudaMalloc(&st->d_layers, sizeof(FdLayer) * su.L) == cudaSuccess;
  if (ok) ok = cudaMemcpy(st->d_layers, ly.data(), sizeof(FdLayer) * su.L, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    decode_fused_destroy(st);
    return nullptr;
  }
  return st;
}

void decode_fused_destroy(DecFusedState* st) {
  if (!st) return;
  if (st->d_layers) cudaFree(st->d_layers);
  if (st->d_maps) cudaFree(st->d_maps);
  delete st;
}

int decode_fused_barriers(int L) { return 5 * L + 2; }  // per-phase counters (dw.bar capacity)

cudaError_t decode_fused(DecFusedState* st, const DecFusedRun& r, int sms, cudaStream_t s) {
  if (!st || r.B <= 0 || r.B > 16) return cudaErrorInvalidValue;
  FdParams p{};
  p.L = r.L, p.D = r.D, p.H = r.H, p.KV = r.KV, p.F = r.F, p.V = r.V, p.B = r.B, p.hd = r.hd;
  p.ldq = (r.H + 2 * r.KV) * r.hd;
  p.nbp = (r.D / 64 + 3) / 4 * 4;
  p.eps = r.eps;
  p.log2_theta = log2f(r.theta);
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)r.hd);
  p.layers = st->d_layers;
  p.embed = r.embed, p.final_norm = r.final_norm, p.lm_wb = r.lm_wb;
  p.hid = r.hid, p.xg = r.xg, p.xlo = r.xlo, p.qkvf = r.qkvf, p.attn = r.attn, p.act = r.act, p.ss = r.ss;
  p.logits = r.logits, p.keys = r.keys, p.ws = r.ws, p.tickets = r.tickets, p.aws = r.aws, p.atk = r.atk;
  p.bar = r.bar, p.bar_base = r.bar_base;
  p.pool = r.pool, p.n_pages = r.n_pages, p.max_pages = r.max_pages, p.bt = r.bt, p.rows = r.rows;
  p.last_tok = r.last_tok, p.tok_out = r.tok_out, p.store_logits = r.store_logits;
  p.pq = gemv_tma_plan(p.ldq, r.D, EPI_BF16);
  p.po = gemv_tma_plan(r.D, r.H * r.hd, EPI_BF16);
  p.pgu = gemv_tma_plan(2 * r.F, r.D, EPI_BF16);
  p.pd = gemv_tma_plan(r.D, r.F, EPI_BF16);
  p.plm = gemv_tma_plan(r.V, r.D, EPI_F32_ARGMAX);
  p.ph_end = r.ph_end > 0 ? r.ph_end : 5 * r.L + 3;
  // L2 prefetch budget: ~48 MB of the next phase across the grid (env NOVA_DEC_PF_MB overrides; 0 = off)
  static const double pf_mb = getenv("NOVA_DEC_PF_MB") ? atof(getenv("NOVA_DEC_PF_MB")) : 48.0;
  const int grid_ = decode_fused_grid(sms);
  p.pf_bytes = pf_mb > 0 ? (uint32_t)std::min(4.0e6, pf_mb * 1e6 / grid_) / 16 * 16 : 0u;
  p.mch = r.mch;
  static const int dbg = getenv("NOVA_DEC_FUSED_DBG") ? atoi(getenv("NOVA_DEC_FUSED_DBG")) : 0;
  p.dbg = dbg;
  p.tdbg = (dbg & 4) ? reinterpret_cast<unsigned long long*>(r.logits + (size_t)15 * r.V) : nullptr;
  if (r.max_ctx + 1 > MAXCH * CK || r.max_ctx + 1 > r.mch * CK || 5 * r.L + 2 > 512) return cudaErrorInvalidValue;
  const int c = fd_cfg(), S = sms > 0 ? sms : 148;
  if (r.hd == 128) return r.B > 8 ? fd_launch_cfg<2, 128>(c, st->d_maps, p, S, s) : fd_launch_cfg<1, 128>(c, st->d_maps, p, S, s);
  if (r.hd == 32) return r.B > 8 ? fd_launch_cfg<2, 32>(c, st->d_maps, p, S, s) : fd_launch_cfg<1, 32>(c, st->d_maps, p, S, s);
  return cudaErrorInvalidValue;
}

}  // namespace nova
