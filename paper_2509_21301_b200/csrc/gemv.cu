// Decode GEMV (the decode linears
// are memory-bound, ~75% of decode time, >40% long-scoreboard stalls on A6000).
//
//   Y[b][n] (epilogue) = sum_k Xin[b][k] W[n][k] + bias[n],   B <= 16 rows
//
// Swap-AB on the legacy tensor core (mma.sync m16n8k16): the weight rows are the
// M side, the batch the N side, so one instruction covers 16 weight rows x 8
// batch rows x 16 k.  Each thread loads 16 contiguous bytes of a weight row
// (128-bit, L1::no_allocate streaming) and of the matching x row; the k order
// inside the 32-wide chunk is permuted identically for both operands, which
// leaves the dot product unchanged.  A CTA owns MT x 16 weight rows and splits K over
// WARPS warps; partials are reduced through shared memory in fixed warp order.
//
// Input modes (XM): bf16 x; f32 x split hi/lo on the tensor core; or the f32 residual
// stream with the RMSNorm applied on load (x * rstd * gamma, "kernel fusion
// ... RMSNorm"): every CTA recomputes the B row statistics exactly as rmsnorm_kernel does
// (same order -> same bits) while its first weight batch is in flight, so the norm costs no
// launch and no HBM pass.
// Epilogues: bf16 / f32 store / f32 residual add / SiLU(gate)*up (interleaved 16-row
// gate|up blocks) / M-RoPE + paged-KV append (RMAP_ROPE: the CTA's second m-tile holds the
// rows half a head further, so each thread owns both halves of its rotation pairs) /
// logits + greedy argmax (packed (ordered value, ~index) 64-bit atomicMax: exact, and
// independent of arrival order).
// The configuration depends only on (N, K), never on the grid or the batch size,
// so results are bitwise invariant to the SM budget and to the batch composition.
// PDL prologue: the first weight batch is requested before griddepcontrol.wait, so
// weight streaming of this linear overlaps the drain of the previous kernel.
#include "common.cuh"
#include "kernels.h"

namespace nova {

bool g_use_pdl = true;

namespace {

constexpr int UNROLL = 4;
enum XMode { XM_BF16 = 0, XM_F32 = 1, XM_NORM_BF16 = 2, XM_NORM_F32 = 3 };
enum RMap { RMAP_LINEAR = 0, RMAP_ROPE = 1 };

NOVA_DEV float silu_f(float z) { return z / (1.0f + __expf(-z)); }

template <int NT, int XM>
struct XFrag {
  uint4 v[NT];                                       // bf16 x (or hi part)
  uint4 lo[(XM == XM_F32 || XM == XM_NORM_F32) ? NT : 1];
};

NOVA_DEV void split_hi_lo(const float* xs, uint4& hiv, uint4& lov) {
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bf16 h0 = __float2bfloat16_rn(xs[2 * j]), h1 = __float2bfloat16_rn(xs[2 * j + 1]);
    float r0 = xs[2 * j] - __bfloat162float(h0), r1 = xs[2 * j + 1] - __bfloat162float(h1);
    __nv_bfloat162 hh = __halves2bfloat162(h0, h1);
    hi[j] = *reinterpret_cast<uint32_t*>(&hh);
    lo[j] = pack_bf16(r0, r1);
  }
  hiv = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  lov = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

template <int NT, int XM>
NOVA_DEV void load_x(XFrag<NT, XM>& f, const void* X, int ldx, int B, int g, int k, const bf16* gamma,
                     const float* s_rs) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int b = nt * 8 + g;
    if constexpr (XM == XM_BF16) {
      f.v[nt] = b < B ? *reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(X) + (size_t)b * ldx + k)
                      : make_uint4(0, 0, 0, 0);
    } else {
      if (b < B) {
        const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(X) + (size_t)b * ldx + k);
        float4 x0 = p[0], x1 = p[1];
        float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        if constexpr (XM == XM_NORM_BF16 || XM == XM_NORM_F32) {
          const float rs = s_rs[b];
          const uint4 gu = *reinterpret_cast<const uint4*>(gamma + k);
          const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 gg = unpack_bf16(gw[q]);
            xs[2 * q] = xs[2 * q] * rs * gg.x;  // same expression order as rmsnorm_kernel
            xs[2 * q + 1] = xs[2 * q + 1] * rs * gg.y;
          }
        }
        if constexpr (XM == XM_NORM_BF16) {
          f.v[nt] = make_uint4(pack_bf16(xs[0], xs[1]), pack_bf16(xs[2], xs[3]), pack_bf16(xs[4], xs[5]),
                               pack_bf16(xs[6], xs[7]));
        } else {
          split_hi_lo(xs, f.v[nt], f.lo[nt]);
        }
      } else {
        f.v[nt] = make_uint4(0, 0, 0, 0);
        if constexpr (XM == XM_F32 || XM == XM_NORM_F32) f.lo[nt] = make_uint4(0, 0, 0, 0);
      }
    }
  }
}

// acc[mt][nt][4] += W rows (wg: row g, wg8: row g+8 of each m tile) . x
template <int MT, int NT, int XM>
NOVA_DEV void mma_chunk(float (*acc)[NT][4], const uint4* wg, const uint4* wg8, const XFrag<NT, XM>& f) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const uint32_t a1[4] = {wg[mt].x, wg8[mt].x, wg[mt].y, wg8[mt].y};
    const uint32_t a2[4] = {wg[mt].z, wg8[mt].z, wg[mt].w, wg8[mt].w};
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const uint32_t b1[2] = {f.v[nt].x, f.v[nt].y};
      const uint32_t b2[2] = {f.v[nt].z, f.v[nt].w};
      mma_bf16_16816(acc[mt][nt], a1, b1);
      mma_bf16_16816(acc[mt][nt], a2, b2);
      if constexpr (XM == XM_F32 || XM == XM_NORM_F32) {
        const uint32_t c1[2] = {f.lo[nt].x, f.lo[nt].y};
        const uint32_t c2[2] = {f.lo[nt].z, f.lo[nt].w};
        mma_bf16_16816(acc[mt][nt], a1, c1);
        mma_bf16_16816(acc[mt][nt], a2, c2);
      }
    }
  }
}

template <int MT>
NOVA_DEV void load_w(uint4 (&wg)[MT], uint4 (&wg8)[MT], const bf16* const* wrow, int kk) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    wg[mt] = ld_nc_v4(wrow[2 * mt] + kk);
    wg8[mt] = ld_nc_v4(wrow[2 * mt + 1] + kk);
  }
}

NOVA_DEV unsigned long long argmax_key(float v, int n) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // order-preserving float -> uint
  return ((unsigned long long)u << 32) | (0xFFFFFFFFu - (uint32_t)n);
}

template <int NT, int XM, int EPI, int MT, int WARPS, int RMAP>
__global__ void __launch_bounds__(WARPS * 32) gemv_kernel(const void* __restrict__ X, int ldx,
                                                          const bf16* __restrict__ W, int N, int K,
                                                          void* __restrict__ Y, int ldy,
                                                          const bf16* __restrict__ bias, int B, int kslice,
                                                          GemvAux aux) {
  __shared__ float red[WARPS][MT][NT][32][4];
  __shared__ float s_rs[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  int rbase[MT];  // first weight row of each m tile
  if constexpr (RMAP == RMAP_ROPE) {
    const int half = aux.hd / 2, per_head = half / 16;
    const int r0 = (blockIdx.x / per_head) * aux.hd + (blockIdx.x % per_head) * 16;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) rbase[mt] = r0 + mt * half;
  } else {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) rbase[mt] = blockIdx.x * (16 * MT) + 16 * mt;
  }
  float acc[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[mt][nt][j] = 0.f;

  const int kbeg = warp * kslice;
  const int kend = min(K, kbeg + kslice);
  const bf16* wrow[2 * MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    wrow[2 * mt] = W + (size_t)(rbase[mt] + g) * K;
    wrow[2 * mt + 1] = W + (size_t)(rbase[mt] + g + 8) * K;
  }
  // PDL prologue: weights do not depend on the previous kernel -- request the first batch now
  uint4 wg[UNROLL][MT], wg8[UNROLL][MT];
  int k = kbeg;
  const bool full0 = k + UNROLL * 32 <= kend;
  if (full0) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) load_w<MT>(wg[u], wg8[u], wrow, k + u * 32 + 8 * c);
  }
  pdl_launch_dependents();
  pdl_wait();
  if constexpr (XM == XM_NORM_BF16 || XM == XM_NORM_F32) {
    // RMSNorm statistics of the B input rows in the canonical order (common.cuh), one row per
    // 128-thread group, all groups in parallel -- identical bits to rmsnorm_kernel
    static_assert(WARPS % 4 == 0, "norm-on-load needs whole 128-thread groups");
    __shared__ float red4[WARPS / 4][4];
    const int grp = warp >> 2, v = threadIdx.x & 127;
    for (int b0 = 0; b0 < B; b0 += WARPS / 4) {
      const int b = b0 + grp;
      if (b < B) {
        const float ss = row_sumsq_canonical(reinterpret_cast<const float*>(X) + (size_t)b * ldx, K, v, red4[grp],
                                             grp + 1);
        if (v == 0) s_rs[b] = rsqrtf(ss / K + aux.eps);
      }
    }
    __syncthreads();
  }
  if (full0) {
    for (;;) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        XFrag<NT, XM> f;
        load_x<NT, XM>(f, X, ldx, B, g, k + u * 32 + 8 * c, aux.gamma, s_rs);
        mma_chunk<MT, NT, XM>(acc, wg[u], wg8[u], f);
      }
      k += UNROLL * 32;
      if (k + UNROLL * 32 > kend) break;
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) load_w<MT>(wg[u], wg8[u], wrow, k + u * 32 + 8 * c);
    }
  }
  for (; k < kend; k += 32) {
    uint4 a[MT], b[MT];
    load_w<MT>(a, b, wrow, k + 8 * c);
    XFrag<NT, XM> f;
    load_x<NT, XM>(f, X, ldx, B, g, k + 8 * c, aux.gamma, s_rs);
    mma_chunk<MT, NT, XM>(acc, a, b, f);
  }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[warp][mt][nt][lane][j] = acc[mt][nt][j];
  __syncthreads();
  if (warp != 0) return;
  // fixed-order reduction over the K slices
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float s = red[0][mt][nt][lane][j];
#pragma unroll
        for (int w = 1; w < WARPS; ++w) s += red[w][mt][nt][lane][j];
        acc[mt][nt][j] = s;
      }
  // c0:(row g, col 2c) c1:(g, 2c+1) c2:(g+8, 2c) c3:(g+8, 2c+1); rows = n, cols = batch
  if constexpr (EPI == EPI_F32_ARGMAX) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {  // batch column 2c + jb of tile nt
        const int b = nt * 8 + 2 * c + jb;
        unsigned long long best = 0ull;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int jr = 0; jr < 2; ++jr) {
            const int n = rbase[mt] + g + 8 * jr;
            const float v = acc[mt][nt][jr * 2 + jb];
            if (b < B) reinterpret_cast<float*>(Y)[(size_t)b * ldy + n] = v;
            const unsigned long long key = argmax_key(v, n);
            best = key > best ? key : best;
          }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const unsigned long long ot = __shfl_xor_sync(0xffffffffu, best, o);
          best = ot > best ? ot : best;
        }
        if (g == 0 && b < B) atomicMax(aux.keys + b, best);
      }
    return;
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = nt * 8 + 2 * c + (j & 1);
      const int ro = g + ((j >> 1) << 3);
      if (b >= B) continue;
      if constexpr (EPI == EPI_BF16_SILUMUL) {
        const float gt = acc[0][nt][j], up = acc[MT - 1][nt][j];
        reinterpret_cast<bf16*>(Y)[(size_t)b * ldy + rbase[0] / 2 + ro] = __float2bfloat16_rn(silu_f(gt) * up);
      } else if constexpr (EPI == EPI_QKV_ROPE_KV) {
        // rows n1 (first half of head hh) and n2 = n1 + hd/2 -> rotate (q, k), append (k, v) to the cache
        const int hd = aux.hd, half = hd / 2;
        const int n1 = rbase[0] + ro, n2 = rbase[1] + ro;
        const int hh = n1 / hd, i = n1 % hd;
        float v1 = acc[0][nt][j], v2 = acc[1][nt][j];
        if (bias != nullptr) {
          v1 += __bfloat162float(bias[n1]);
          v2 += __bfloat162float(bias[n2]);
        }
        const DecodeRow rr = aux.rows[b];
        if (hh < aux.H + aux.KV) {  // t = h = w = pos for generated text: plain RoPE at pos
          const float inv = exp2f(-(2.0f * i / hd) * aux.log2_theta);
          float sn, cs;
          sincosf((float)rr.pos * inv, &sn, &cs);
          const float o1 = v1 * cs - v2 * sn, o2 = v2 * cs + v1 * sn;
          v1 = o1;
          v2 = o2;
        }
        if (hh < aux.H) {
          bf16* q = reinterpret_cast<bf16*>(Y) + (size_t)b * ldy;
          q[n1] = __float2bfloat16_rn(v1);
          q[n2] = __float2bfloat16_rn(v2);
        } else {
          const int isv = hh >= aux.H + aux.KV;
          const int kvh = hh - aux.H - (isv ? aux.KV : 0);
          const size_t page_stride = (size_t)2 * aux.KV * 64 * hd;
          bf16* pg = aux.pool + ((size_t)aux.layer * aux.n_pages +
                                 aux.bt[(size_t)rr.slot * aux.max_pages + (rr.ctx >> 6)]) * page_stride;
          bf16* dst = pg + (((size_t)isv * aux.KV + kvh) * 64 + (rr.ctx & 63)) * hd;
          dst[i] = __float2bfloat16_rn(v1);
          dst[i + half] = __float2bfloat16_rn(v2);
        }
      } else {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int n = rbase[mt] + ro;
          float v = acc[mt][nt][j];
          if (bias != nullptr) v += __bfloat162float(bias[n]);
          if constexpr (EPI == EPI_BF16) {
            reinterpret_cast<bf16*>(Y)[(size_t)b * ldy + n] = __float2bfloat16_rn(v);
          } else if constexpr (EPI == EPI_F32_RESID) {
            float* yp = reinterpret_cast<float*>(Y) + (size_t)b * ldy + n;
            const float h = *yp + v;
            *yp = h;
            if (aux.nxout) aux.nxout[(size_t)b * aux.ldnx + n] = __float2bfloat16_rn(h * __bfloat162float(aux.ngamma[n]));
          } else {
            reinterpret_cast<float*>(Y)[(size_t)b * ldy + n] = v;
          }
        }
      }
    }
  }
}

template <int NT, int XM, int EPI, int MT, int WARPS, int RMAP>
cudaError_t launch_cfg(const void* X, int ldx, const bf16* W, int N, int K, void* Y, int ldy, const bf16* bias, int B,
                       const GemvAux& aux, cudaStream_t s) {
  const int kslice = ((K + WARPS * 32 - 1) / (WARPS * 32)) * 32;
  return launch_k(gemv_kernel<NT, XM, EPI, MT, WARPS, RMAP>, dim3(N / (16 * MT)), dim3(WARPS * 32), 0, s, true, X,
                  ldx, W, N, K, Y, ldy, bias, B, kslice, aux);
}

// Shape-only configuration: many rows -> 32 rows x 8 warps; few rows -> 16 rows x 32 warps
// (32 rows x 16 warps where the epilogue pairs two m-tiles).
template <int NT, int XM, int EPI>
cudaError_t launch_epi(const void* X, int ldx, const bf16* W, int N, int K, void* Y, int ldy, const bf16* bias, int B,
                       const GemvAux& aux, cudaStream_t s) {
  const bool big = N / 32 >= 4 * 148;
  if constexpr (EPI == EPI_QKV_ROPE_KV) {
    return launch_cfg<NT, XM, EPI, 2, 16, RMAP_ROPE>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
  } else if constexpr (EPI == EPI_BF16_SILUMUL) {
    if (big) return launch_cfg<NT, XM, EPI, 2, 8, RMAP_LINEAR>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    return launch_cfg<NT, XM, EPI, 2, 16, RMAP_LINEAR>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
  } else {
    if (big) return launch_cfg<NT, XM, EPI, 2, 8, RMAP_LINEAR>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    return launch_cfg<NT, XM, EPI, 1, 32, RMAP_LINEAR>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
  }
}

template <int NT, int XM>
cudaError_t launch_nt(const void* X, int ldx, const bf16* W, int N, int K, void* Y, int ldy, const bf16* bias, int B,
                      int epi, const GemvAux& aux, cudaStream_t s) {
  switch (epi) {
    case EPI_BF16: return launch_epi<NT, XM, EPI_BF16>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    case EPI_BF16_SILUMUL: return launch_epi<NT, XM, EPI_BF16_SILUMUL>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    case EPI_F32_RESID: return launch_epi<NT, XM, EPI_F32_RESID>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    case EPI_F32_STORE: return launch_epi<NT, XM, EPI_F32_STORE>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    case EPI_QKV_ROPE_KV: return launch_epi<NT, XM, EPI_QKV_ROPE_KV>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    case EPI_F32_ARGMAX: return launch_epi<NT, XM, EPI_F32_ARGMAX>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
  }
  return cudaErrorInvalidValue;
}

// Only the combinations the stage programs and the op ABI use are instantiated.
template <int NT>
cudaError_t launch_xm(const void* X, int xmode, int ldx, const bf16* W, int N, int K, void* Y, int ldy,
                      const bf16* bias, int B, int epi, const GemvAux& aux, cudaStream_t s) {
  switch (xmode) {
    case XM_BF16:
      if (epi == EPI_QKV_ROPE_KV || epi == EPI_F32_ARGMAX) return cudaErrorInvalidValue;
      return launch_nt<NT, XM_BF16>(X, ldx, W, N, K, Y, ldy, bias, B, epi, aux, s);
    case XM_F32:
      if (epi == EPI_F32_ARGMAX) return launch_epi<NT, XM_F32, EPI_F32_ARGMAX>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
      if (epi != EPI_F32_STORE) return cudaErrorInvalidValue;
      return launch_epi<NT, XM_F32, EPI_F32_STORE>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
    case XM_NORM_BF16:
      if (epi == EPI_QKV_ROPE_KV)
        return launch_epi<NT, XM_NORM_BF16, EPI_QKV_ROPE_KV>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
      if (epi == EPI_BF16_SILUMUL)
        return launch_epi<NT, XM_NORM_BF16, EPI_BF16_SILUMUL>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
      if (epi == EPI_BF16) return launch_epi<NT, XM_NORM_BF16, EPI_BF16>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
      return cudaErrorInvalidValue;
    case XM_NORM_F32:
      if (epi == EPI_F32_ARGMAX)
        return launch_epi<NT, XM_NORM_F32, EPI_F32_ARGMAX>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
      if (epi == EPI_F32_STORE)
        return launch_epi<NT, XM_NORM_F32, EPI_F32_STORE>(X, ldx, W, N, K, Y, ldy, bias, B, aux, s);
      return cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t gemv_ex(const void* X, int xmode, int ldx, const bf16* W, int N, int K, void* Y, int ldy,
                    const bf16* bias, int B, int epi, const GemvAux& aux, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (B > 16 || N % 32 || K % 32 || ldx % 8 || xmode < 0 || xmode > 3) return cudaErrorInvalidValue;
  if (epi == EPI_QKV_ROPE_KV && (aux.hd % 32 || N % aux.hd || !aux.rows || !aux.pool || !aux.bt))
    return cudaErrorInvalidValue;
  if (epi == EPI_F32_ARGMAX && !aux.keys) return cudaErrorInvalidValue;
  if (xmode >= XM_NORM_BF16 && (!aux.gamma || K % 4)) return cudaErrorInvalidValue;
  return B <= 8 ? launch_xm<1>(X, xmode, ldx, W, N, K, Y, ldy, bias, B, epi, aux, s)
                : launch_xm<2>(X, xmode, ldx, W, N, K, Y, ldy, bias, B, epi, aux, s);
}

cudaError_t gemv(const void* X, int x_f32, int ldx, const bf16* W, int N, int K, void* Y, int ldy, const bf16* bias,
                 int B, int epi, cudaStream_t s) {
  GemvAux aux{};
  return gemv_ex(X, x_f32 ? XM_F32 : XM_BF16, ldx, W, N, K, Y, ldy, bias, B, epi, aux, s);
}

}  // namespace nova
