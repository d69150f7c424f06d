// Row-wise and elementwise kernels of the stage programs (SURVEY.md §8(a) rows a1,
// a5-a7): patchify, LayerNorm / RMSNorm ("kernel fusion ... RoPE and
// RMSNorm"), ViT 2D RoPE, LLM M-RoPE fused with the paged KV-cache write,
// embedding gather, deterministic argmax.  All are HBM/latency-bound row kernels.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace nova {
namespace {

// ---------------------------------------------------------------- norms (one warp per row)
// LayerNorm (ViT): the row is loaded once into registers (all loads in flight together), then
// mean, biased variance and the output are computed from registers; the summation order
// (lane-strided float4 chunks, then the xor butterfly) is fixed by d.
constexpr int LN_MAXCH = 12;  // d <= 1536 register-resident; longer rows take the streaming loop
__global__ void layernorm_kernel(const float* __restrict__ x, int ldx, const bf16* __restrict__ gm,
                                 const bf16* __restrict__ bt, bf16* __restrict__ y, int ldy, int M, int d, float eps) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* xr = x + (size_t)row * ldx;
  bf16* yr = y + (size_t)row * ldy;
  const int nch = d >> 2;
  if (nch <= 32 * LN_MAXCH) {
    float4 v[LN_MAXCH];
#pragma unroll
    for (int t = 0; t < LN_MAXCH; ++t) {
      const int f = lane + 32 * t;
      v[t] = f < nch ? reinterpret_cast<const float4*>(xr)[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < LN_MAXCH; ++t)
      if (lane + 32 * t < nch) s += (v[t].x + v[t].y) + (v[t].z + v[t].w);
    const float mu = warp_sum(s) / d;
    float q = 0.f;
#pragma unroll
    for (int t = 0; t < LN_MAXCH; ++t)
      if (lane + 32 * t < nch) {
        const float a = v[t].x - mu, b = v[t].y - mu, c = v[t].z - mu, e = v[t].w - mu;
        q += (a * a + b * b) + (c * c + e * e);
      }
    const float rs = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
    for (int t = 0; t < LN_MAXCH; ++t) {
      const int f = lane + 32 * t;
      if (f >= nch) continue;
      const int i = f * 4;
      const float2 g01 = unpack_bf16(*reinterpret_cast<const uint32_t*>(gm + i));
      const float2 g23 = unpack_bf16(*reinterpret_cast<const uint32_t*>(gm + i + 2));
      const float2 b01 = unpack_bf16(*reinterpret_cast<const uint32_t*>(bt + i));
      const float2 b23 = unpack_bf16(*reinterpret_cast<const uint32_t*>(bt + i + 2));
      uint2 o;
      o.x = pack_bf16((v[t].x - mu) * rs * g01.x + b01.x, (v[t].y - mu) * rs * g01.y + b01.y);
      o.y = pack_bf16((v[t].z - mu) * rs * g23.x + b23.x, (v[t].w - mu) * rs * g23.y + b23.y);
      *reinterpret_cast<uint2*>(yr + i) = o;
    }
    return;
  }
  float s = 0.f;
  for (int i = lane * 4; i < d; i += 128) {
    float4 v = *reinterpret_cast<const float4*>(xr + i);
    s += (v.x + v.y) + (v.z + v.w);
  }
  const float mu = warp_sum(s) / d;
  float q = 0.f;
  for (int i = lane * 4; i < d; i += 128) {
    float4 v = *reinterpret_cast<const float4*>(xr + i);
    const float a = v.x - mu, b = v.y - mu, c = v.z - mu, e = v.w - mu;
    q += (a * a + b * b) + (c * c + e * e);
  }
  const float rs = rsqrtf(warp_sum(q) / d + eps);
  for (int i = lane * 4; i < d; i += 128) {
    float4 v = *reinterpret_cast<const float4*>(xr + i);
    const float2 g01 = unpack_bf16(*reinterpret_cast<const uint32_t*>(gm + i));
    const float2 g23 = unpack_bf16(*reinterpret_cast<const uint32_t*>(gm + i + 2));
    const float2 b01 = unpack_bf16(*reinterpret_cast<const uint32_t*>(bt + i));
    const float2 b23 = unpack_bf16(*reinterpret_cast<const uint32_t*>(bt + i + 2));
    uint2 o;
    o.x = pack_bf16((v.x - mu) * rs * g01.x + b01.x, (v.y - mu) * rs * g01.y + b01.y);
    o.y = pack_bf16((v.z - mu) * rs * g23.x + b23.x, (v.w - mu) * rs * g23.y + b23.y);
    *reinterpret_cast<uint2*>(yr + i) = o;
  }
}

// RMSNorm: one 128-thread group per row (4 rows per 512-thread CTA), canonical statistics
// order (common.cuh row_sumsq_canonical); y = (x * rstd) * gamma.
__global__ void __launch_bounds__(512) rmsnorm_kernel(const float* __restrict__ x, int ldx, const bf16* __restrict__ gm,
                                                      void* __restrict__ y, int y_f32, int ldy, int M, int d, float eps) {
  __shared__ float red[4][4];
  pdl_launch_dependents();
  const int grp = threadIdx.x >> 7, v = threadIdx.x & 127;
  const int row = blockIdx.x * 4 + grp;
  const int nch = d >> 2;
  if (nch <= 8 * NORM_LANES && y_f32 == 0) {
    // d <= 4096, bf16 out (the decode norms before the TMA GEMVs): gamma is requested before
    // griddepcontrol.wait and the row stays in registers between the statistics and the output --
    // the same operations in the same order as row_sumsq_canonical + the loop below (same bits)
    uint2 gv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int f = v + i * NORM_LANES;
      gv[i] = f < nch ? *reinterpret_cast<const uint2*>(gm + 4 * f) : make_uint2(0u, 0u);
    }
    pdl_wait();
    if (row >= M) return;
    const float* xr = x + (size_t)row * ldx;
    float4 xv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int f = v + i * NORM_LANES;
      xv[i] = f < nch ? reinterpret_cast<const float4*>(xr)[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float sq = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int f = v + i * NORM_LANES;
      if (f < nch) sq += (xv[i].x * xv[i].x + xv[i].y * xv[i].y) + (xv[i].z * xv[i].z + xv[i].w * xv[i].w);
    }
    sq = warp_sum(sq);
    if ((v & 31) == 0) red[grp][v >> 5] = sq;
    asm volatile("bar.sync %0, 128;" ::"r"(grp + 1) : "memory");
    const float t = ((red[grp][0] + red[grp][1]) + red[grp][2]) + red[grp][3];
    const float rs = rsqrtf(t / d + eps);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int f = v + i * NORM_LANES;
      if (f >= nch) continue;
      const float2 g01 = unpack_bf16(gv[i].x), g23 = unpack_bf16(gv[i].y);
      uint2 o;
      o.x = pack_bf16(xv[i].x * rs * g01.x, xv[i].y * rs * g01.y);
      o.y = pack_bf16(xv[i].z * rs * g23.x, xv[i].w * rs * g23.y);
      *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(y) + (size_t)row * ldy + 4 * f) = o;
    }
    return;
  }
  pdl_wait();
  if (row >= M) return;  // whole 128-thread group: named barrier grp + 1 stays consistent
  const float* xr = x + (size_t)row * ldx;
  const float rs = rsqrtf(row_sumsq_canonical(xr, d, v, red[grp], grp + 1) / d + eps);
  for (int f = v; f < (d >> 2); f += NORM_LANES) {
    const int i = f * 4;
    float4 xv = *reinterpret_cast<const float4*>(xr + i);
    const float2 g01 = unpack_bf16(*reinterpret_cast<const uint32_t*>(gm + i));
    const float2 g23 = unpack_bf16(*reinterpret_cast<const uint32_t*>(gm + i + 2));
    const float o0 = xv.x * rs * g01.x, o1 = xv.y * rs * g01.y, o2 = xv.z * rs * g23.x, o3 = xv.w * rs * g23.y;
    if (y_f32 == 2) {  // bf16 hi / lo pair (f32 operand of the decode lm_head on the tensor core)
      bf16* yh = reinterpret_cast<bf16*>(y) + (size_t)row * ldy + i;
      bf16* yl = reinterpret_cast<bf16*>(y) + (size_t)M * ldy + (size_t)row * ldy + i;
      const float o[4] = {o0, o1, o2, o3};
      bf16 h[4], lo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        h[q] = __float2bfloat16_rn(o[q]);
        lo[q] = __float2bfloat16_rn(o[q] - __bfloat162float(h[q]));
      }
      *reinterpret_cast<uint2*>(yh) = make_uint2(
          (uint32_t)__bfloat16_as_ushort(h[0]) | ((uint32_t)__bfloat16_as_ushort(h[1]) << 16),
          (uint32_t)__bfloat16_as_ushort(h[2]) | ((uint32_t)__bfloat16_as_ushort(h[3]) << 16));
      *reinterpret_cast<uint2*>(yl) = make_uint2(
          (uint32_t)__bfloat16_as_ushort(lo[0]) | ((uint32_t)__bfloat16_as_ushort(lo[1]) << 16),
          (uint32_t)__bfloat16_as_ushort(lo[2]) | ((uint32_t)__bfloat16_as_ushort(lo[3]) << 16));
    } else if (y_f32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + (size_t)row * ldy + i) = make_float4(o0, o1, o2, o3);
    } else {
      uint2 o;
      o.x = pack_bf16(o0, o1);
      o.y = pack_bf16(o2, o3);
      *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(y) + (size_t)row * ldy + i) = o;
    }
  }
}

// ---------------------------------------------------------------- patchify
// Row r (merge-group-major): group = r / m^2 over the (gh/m) x (gw/m) group grid, row-major;
// inside the group (di, dj) row-major.  Column = ((c*T + t)*P + py)*P + px, frame duplicated over t.
__global__ void patchify_kernel(const bf16* __restrict__ pix, int C, int H, int W, int P, int T, int m,
                                bf16* __restrict__ X0) {
  const int r = blockIdx.x;
  const int gw = W / P;
  const int grp = r / (m * m), in = r % (m * m);
  const int gi = grp / (gw / m), gj = grp % (gw / m);
  const int pi = gi * m + in / m, pj = gj * m + in % m;
  const int K = C * T * P * P;
  for (int col = threadIdx.x; col < K; col += blockDim.x) {
    const int px = col % P, py = (col / P) % P, ch = col / (T * P * P);
    X0[(size_t)r * K + col] = pix[((size_t)ch * H + pi * P + py) * W + pj * P + px];
  }
}

// ---------------------------------------------------------------- RoPE
// ViT: angle for pair i (< hd/2): i < hd/4 -> h * inv[i], else w * inv[i - hd/4]; inv[j] = theta^(-4j/hd).
// CTA = VR rows: the hd/2 (cos, sin) pairs of each row are computed once into smem, then every
// (row, q|k head, 8-pair group) is one thread: two 16-byte loads (x[i..i+7], x[i+half..]) and
// two 16-byte stores, in place.  Same per-element arithmetic as the scalar form.
constexpr int VR = 8;
__global__ void __launch_bounds__(256) vit_rope_kernel(bf16* __restrict__ qkv, int N, int heads, int hd, int gw, int m,
                                                       float log2_theta) {
  extern __shared__ float cs_tab[];  // [VR][half] cos, then [VR][half] sin
  const int half = hd / 2, quarter = hd / 4, r0 = blockIdx.x * VR;
  float* ctab = cs_tab;
  float* stab = cs_tab + VR * half;
  for (int idx = threadIdx.x; idx < VR * half; idx += blockDim.x) {
    const int rr = idx / half, i = idx % half, r = r0 + rr;
    if (r >= N) continue;
    const int grp = r / (m * m), in = r % (m * m);
    const int gi = grp / (gw / m), gj = grp % (gw / m);
    const float ph = (float)(gi * m + in / m), pw = (float)(gj * m + in % m);
    const int j = i < quarter ? i : i - quarter;
    const float inv = exp2f(-(4.0f * j / hd) * log2_theta);
    const float ang = (i < quarter ? ph : pw) * inv;
    float sn, cs;
    sincosf(ang, &sn, &cs);
    ctab[idx] = cs;
    stab[idx] = sn;
  }
  __syncthreads();
  const int groups = half / 8, per_row = 2 * heads * groups;
  for (int u = threadIdx.x; u < VR * per_row; u += blockDim.x) {
    const int rr = u / per_row, rem = u % per_row, r = r0 + rr;
    if (r >= N) continue;
    const int hh = rem / groups, i0 = (rem % groups) * 8;  // hh < heads: q, else k (contiguous)
    bf16* v = qkv + (size_t)r * 3 * heads * hd + (size_t)hh * hd;
    const uint4 a = *reinterpret_cast<const uint4*>(v + i0);
    const uint4 b = *reinterpret_cast<const uint4*>(v + i0 + half);
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
    uint32_t oa[4], ob[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 x1 = unpack_bf16(aw[q]), x2 = unpack_bf16(bw[q]);
      const int i = i0 + 2 * q;
      const float c0 = ctab[rr * half + i], s0 = stab[rr * half + i];
      const float c1 = ctab[rr * half + i + 1], s1 = stab[rr * half + i + 1];
      oa[q] = pack_bf16(x1.x * c0 - x2.x * s0, x1.y * c1 - x2.y * s1);
      ob[q] = pack_bf16(x2.x * c0 + x1.x * s0, x2.y * c1 + x1.y * s1);
    }
    *reinterpret_cast<uint4*>(v + i0) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
    *reinterpret_cast<uint4*>(v + i0 + half) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
  }
}

// LLM M-RoPE (sections sec0 | sec1 | rest over the hd/2 frequencies) + paged KV write.
// One CTA per row; a thread owns 8 consecutive frequencies i0..i0+7 of one q / k head (16-byte loads of
// both halves) and writes a rotated k head straight into its page as well; v heads are 16-byte copies.
// Same per-element arithmetic as the one-element-per-thread version (bitwise the same results).
__global__ void __launch_bounds__(256) llm_rope_kv_kernel(bf16* __restrict__ qkv, int ld, int H, int KV, int hd,
                                                          float log2_theta, int sec0, int sec1,
                                                          const int* __restrict__ pos3, int ld_pos,
                                                          const DecodeRow* __restrict__ rows, int slot, int ctx0,
                                                          bf16* __restrict__ pool, int layer, int n_pages,
                                                          const int* __restrict__ bt, int max_pages) {
  pdl_launch_dependents();
  pdl_wait();
  const int r = blockIdx.x;
  int p[3], cidx, sl;
  if (rows) {
    const DecodeRow rr = rows[r];
    p[0] = p[1] = p[2] = rr.pos;
    cidx = rr.ctx;
    sl = rr.slot;
  } else {
    p[0] = pos3[r];
    p[1] = pos3[ld_pos + r];
    p[2] = pos3[2 * ld_pos + r];
    cidx = ctx0 + r;
    sl = slot;
  }
  const int half = hd / 2, g8 = half / 8;
  bf16* row = qkv + (size_t)r * ld;
  const size_t page_stride = (size_t)2 * KV * 64 * hd;
  bf16* pg = pool + ((size_t)layer * n_pages + bt[(size_t)sl * max_pages + (cidx >> 6)]) * page_stride;
  const int off = cidx & 63;
  const int nrot = (H + KV) * g8, nv = KV * hd / 8;
  for (int u = threadIdx.x; u < nrot + nv; u += blockDim.x) {
    if (u < nrot) {
      const int hh = u / g8, i0 = (u % g8) * 8;
      bf16* v = row + (size_t)hh * hd;
      const uint4 a = *reinterpret_cast<const uint4*>(v + i0);
      const uint4 b = *reinterpret_cast<const uint4*>(v + i0 + half);
      const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
      uint32_t oa[4], ob[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 x1 = unpack_bf16(aw[q]), x2 = unpack_bf16(bw[q]);
        float c[2], sn[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = i0 + 2 * q + e;
          const int comp = i < sec0 ? 0 : (i < sec0 + sec1 ? 1 : 2);
          const float inv = exp2f(-(2.0f * i / hd) * log2_theta);
          sincosf((float)p[comp] * inv, &sn[e], &c[e]);
        }
        oa[q] = pack_bf16(x1.x * c[0] - x2.x * sn[0], x1.y * c[1] - x2.y * sn[1]);
        ob[q] = pack_bf16(x2.x * c[0] + x1.x * sn[0], x2.y * c[1] + x1.y * sn[1]);
      }
      const uint4 A = make_uint4(oa[0], oa[1], oa[2], oa[3]), Bv = make_uint4(ob[0], ob[1], ob[2], ob[3]);
      *reinterpret_cast<uint4*>(v + i0) = A;
      *reinterpret_cast<uint4*>(v + i0 + half) = Bv;
      if (hh >= H) {  // rotated K head -> its page (K half of the page)
        bf16* dst = pg + ((size_t)(hh - H) * 64 + off) * hd;
        *reinterpret_cast<uint4*>(dst + i0) = A;
        *reinterpret_cast<uint4*>(dst + i0 + half) = Bv;
      }
    } else {  // V head chunk -> its page (V half)
      const int w = u - nrot, hh = w / (hd / 8), d0 = (w % (hd / 8)) * 8;
      *reinterpret_cast<uint4*>(pg + (((size_t)KV + hh) * 64 + off) * hd + d0) =
          *reinterpret_cast<const uint4*>(row + (size_t)(H + KV + hh) * hd + d0);
    }
  }
}

// ---------------------------------------------------------------- embedding, argmax
__global__ void embed_kernel(const bf16* __restrict__ table, int d, const int* __restrict__ ids,
                             const DecodeRow* __restrict__ rows, const int* __restrict__ last_tok, float* __restrict__ out,
                             int ldo) {
  pdl_launch_dependents();
  pdl_wait();
  const int r = blockIdx.x;
  const int id = ids ? ids[r] : last_tok[rows[r].slot];
  const bf16* src = table + (size_t)id * d;
  float* dst = out + (size_t)r * ldo;
  for (int i = threadIdx.x * 2; i < d; i += blockDim.x * 2) {
    const float2 f = unpack_bf16(*reinterpret_cast<const uint32_t*>(src + i));
    dst[i] = f.x;
    dst[i + 1] = f.y;
  }
}

__global__ void argmax_kernel(const float* __restrict__ logits, int ldl, int V, int* __restrict__ out_tok,
                              const DecodeRow* __restrict__ rows, int* __restrict__ last_tok, int single_slot) {
  pdl_launch_dependents();
  pdl_wait();
  const int r = blockIdx.x;
  const float* l = logits + (size_t)r * ldl;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = l[i];
    if (v > best) {  // strictly greater keeps the lowest index within a thread
      best = v;
      bi = i;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      out_tok[r] = bi;
      if (rows) last_tok[rows[r].slot] = bi;
      else if (single_slot >= 0 && last_tok) last_tok[single_slot] = bi;
    }
  }
}

__global__ void argmax_finalize_kernel(unsigned long long* __restrict__ keys, int n, int* __restrict__ out_tok,
                                       const DecodeRow* __restrict__ rows, int* __restrict__ last_tok,
                                       int single_slot) {
  pdl_launch_dependents();
  pdl_wait();
  const int r = threadIdx.x;
  if (r >= n) return;
  const int tok = (int)(0xFFFFFFFFu - (uint32_t)(keys[r] & 0xFFFFFFFFull));
  keys[r] = 0ull;
  out_tok[r] = tok;
  if (rows) last_tok[rows[r].slot] = tok;
  else if (single_slot >= 0 && last_tok) last_tok[single_slot] = tok;
}

// [N][K] row-major -> [N/64][K/64] blocks of [64 rows][64 k], each block's rows 128 B with
// the 16-byte chunks XOR-swizzled by (row & 7): the byte image TMA SWIZZLE_128B would leave in
// shared memory, so one 8 KB bulk copy per tile lands ready for ldmatrix.
__global__ void block_weights_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst, int N, int K) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 16-byte chunk of dst
  const size_t nchunks = (size_t)N * K / 8;
  if (i >= nchunks) return;
  const size_t blk = i / 512;               // 64 x 64 bf16 = 512 chunks per block
  const int within = (int)(i % 512), r = within / 8, cpos = within % 8;
  const int c = cpos ^ (r & 7);             // logical 16-byte chunk stored at position cpos
  const int kb = K / 64;
  const size_t n = (blk / kb) * 64 + r, k = (blk % kb) * 64 + c * 8;
  reinterpret_cast<uint4*>(dst)[i] = *reinterpret_cast<const uint4*>(src + n * K + k);
}

}  // namespace

std::atomic<unsigned long long> g_kernel_launches{0};

cudaError_t block_weights(const bf16* src, bf16* dst, int N, int K, cudaStream_t s) {
  if (N % 64 || K % 64) return cudaErrorInvalidValue;
  const size_t n = (size_t)N * K / 8;
  count_launch();
  block_weights_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, dst, N, K);
  return cudaGetLastError();
}

cudaError_t argmax_finalize(unsigned long long* keys, int n, int* out_tok, const DecodeRow* rows, int* last_tok,
                            int single_slot, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > 1024) return cudaErrorInvalidValue;
  return launch_k(argmax_finalize_kernel, dim3(1), dim3(32 * ((n + 31) / 32)), 0, s, true, keys, n, out_tok, rows,
                  last_tok, single_slot);
}

cudaError_t layernorm(const float* x, int ldx, const bf16* g, const bf16* b, bf16* y, int ldy, int M, int d, float eps,
                      cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (d % 4) return cudaErrorInvalidValue;
  return launch_k(layernorm_kernel, dim3((M + 7) / 8), dim3(256), 0, s, true, x, ldx, g, b, y, ldy, M, d, eps);
}
__global__ void rope2d_table_kernel(float2* __restrict__ tab, int npos, float log2_theta) {
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npos * 20) return;
  const int pos = i / 20, j = i % 20;
  const float inv = exp2f(-(4.0f * j / 80.0f) * log2_theta);
  float sn, cs;
  sincosf((float)pos * inv, &sn, &cs);
  tab[i] = make_float2(cs, sn);
}
cudaError_t rope2d_table(float2* tab, int npos, float log2_theta, cudaStream_t s) {
  if (npos <= 0) return cudaSuccess;
  return launch_k(rope2d_table_kernel, dim3((npos * 20 + 127) / 128), dim3(128), 0, s, true, tab, npos, log2_theta);
}
// x~ = bf16(x * g) rows (DESIGN R25: the input of a GEMV whose RMSNorm row scale is folded after it)
__global__ void scale_rows_bf16_kernel(const float* __restrict__ x, int ldx, const bf16* __restrict__ g,
                                       bf16* __restrict__ y, int ldy, int M, int d) {
  pdl_launch_dependents();
  pdl_wait();
  const int n = M * d;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = i / d, c = i - r * d;
    y[(size_t)r * ldy + c] = __float2bfloat16_rn(x[(size_t)r * ldx + c] * __bfloat162float(g[c]));
  }
}
cudaError_t scale_rows_bf16(const float* x, int ldx, const bf16* g, bf16* y, int ldy, int M, int d, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const int blocks = std::min(64, (M * d + 255) / 256);
  return launch_k(scale_rows_bf16_kernel, dim3(blocks), dim3(256), 0, s, true, x, ldx, g, y, ldy, M, d);
}
// one thread per (row, 32-column chunk): x~ = bf16(x * g), ss = sum of x^2 over the chunk in column order
__global__ void rms_prep_kernel(const float* __restrict__ x, int ldx, const bf16* __restrict__ g, bf16* __restrict__ y,
                                int ldy, float* __restrict__ ss, int ss_ld, int M, int d) {
  pdl_launch_dependents();
  pdl_wait();
  const int nt = d / 32;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * nt) return;
  const int r = i / nt, t = i % nt;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)r * ldx + t * 32);
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 v = xr[q];
    s = (((s + v.x * v.x) + v.y * v.y) + v.z * v.z) + v.w * v.w;
    const uint2 gg = *reinterpret_cast<const uint2*>(g + t * 32 + 4 * q);
    const float2 g01 = unpack_bf16(gg.x), g23 = unpack_bf16(gg.y);
    *reinterpret_cast<uint2*>(y + (size_t)r * ldy + t * 32 + 4 * q) =
        make_uint2(pack_bf16(v.x * g01.x, v.y * g01.y), pack_bf16(v.z * g23.x, v.w * g23.y));
  }
  ss[(size_t)r * ss_ld + t] = s;
}
// one thread per row: the folded RMSNorm's row scale from the 32-column sums of squares
__global__ void fold_rows_kernel(const float* __restrict__ ss, int ss_ld, int d, float eps, float* __restrict__ rscale,
                                 int M) {
  pdl_launch_dependents();
  pdl_wait();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const float4* p = reinterpret_cast<const float4*>(ss + (size_t)m * ss_ld);
  const int n4 = d / 128;
  float s = 0.f;
  for (int t = 0; t < n4; t += 8) {
    float4 q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = t + u < n4 ? p[t + u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (t + u < n4) s = (((s + q[u].x) + q[u].y) + q[u].z) + q[u].w;
  }
  rscale[m] = rsqrtf(s / (float)d + eps);
}
cudaError_t fold_rows(const float* ss, int ss_ld, int d, float eps, float* rscale, int M, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (d % 128 || ss_ld % 4) return cudaErrorInvalidValue;
  return launch_k(fold_rows_kernel, dim3((M + 127) / 128), dim3(128), 0, s, true, ss, ss_ld, d, eps, rscale, M);
}
cudaError_t rms_prep(const float* x, int ldx, const bf16* g, bf16* y, int ldy, float* ss, int ss_ld, int M, int d,
                     cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (d % 32 || ldx % 4 || ldy % 4) return cudaErrorInvalidValue;
  const int n = M * (d / 32);
  return launch_k(rms_prep_kernel, dim3((n + 127) / 128), dim3(128), 0, s, true, x, ldx, g, y, ldy, ss, ss_ld, M, d);
}
cudaError_t rmsnorm(const float* x, int ldx, const bf16* g, void* y, int y_f32, int ldy, int M, int d, float eps,
                    cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (d % 4) return cudaErrorInvalidValue;
  return launch_k(rmsnorm_kernel, dim3((M + 3) / 4), dim3(512), 0, s, true, x, ldx, g, y, y_f32, ldy, M, d, eps);
}
cudaError_t patchify(const bf16* pix, int C, int H, int W, int P, int T, int merge, bf16* X0, cudaStream_t s) {
  const int N = (H / P) * (W / P);
  if (N <= 0) return cudaSuccess;
  count_launch();
  patchify_kernel<<<N, 256, 0, s>>>(pix, C, H, W, P, T, merge, X0);
  return cudaGetLastError();
}
cudaError_t vit_rope(bf16* qkv, int N, int heads, int hd, int gw, int merge, float theta, cudaStream_t s) {
  if (N <= 0) return cudaSuccess;
  if (hd % 16) return cudaErrorInvalidValue;
  return launch_k(vit_rope_kernel, dim3((N + VR - 1) / VR), dim3(256), (size_t)2 * VR * (hd / 2) * sizeof(float), s,
                  false, qkv, N, heads, hd, gw, merge, log2f(theta));
}
cudaError_t llm_rope_kv(bf16* qkv, int ld, int nrows, int H, int KV, int hd, float theta, int sec0, int sec1,
                        const int* pos3, int ld_pos, const DecodeRow* rows, int slot, int ctx0, bf16* pool, int layer,
                        int n_pages, const int* bt, int max_pages, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  if (hd % 16 || ld % 8) return cudaErrorInvalidValue;
  const int work = (H + KV) * hd / 16 + KV * hd / 8;
  const int thr = std::min(256, (work + 31) / 32 * 32);
  return launch_k(llm_rope_kv_kernel, dim3(nrows), dim3(thr), 0, s, true, qkv, ld, H, KV, hd, log2f(theta), sec0,
                  sec1, pos3, ld_pos, rows, slot, ctx0, pool, layer, n_pages, bt, max_pages);
}
cudaError_t embed(const bf16* table, int d, const int* ids, const DecodeRow* rows, const int* last_tok, float* out,
                  int ldo, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_k(embed_kernel, dim3(n), dim3(256), 0, s, true, table, d, ids, rows, last_tok, out, ldo);
}
cudaError_t argmax_rows(const float* logits, int ldl, int V, int n, int* out_tok, const DecodeRow* rows, int* last_tok,
                        int single_slot, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_k(argmax_kernel, dim3(n), dim3(1024), 0, s, true, logits, ldl, V, out_tok, rows, last_tok, single_slot);
}

}  // namespace nova
