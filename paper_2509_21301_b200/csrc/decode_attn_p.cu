// Persistent paged decode attention sized to the decode partition.
//
//   out[b][h] = softmax_j(q_b,h . k_j / sqrt(hd)) v_j over the cache keys j <= ctx_b of request b,
//   query head h reading KV head h / (H / KV) (GQA)
//
// Nova runs decode on a slice of the SMs.  The cluster kernel (decode_attn_tc, 8 or 4
// CTAs of ~210 KB per (request, KV head), DSMEM merge) fits one CTA per SM, so on a 32-SM slice a
// batch of 16 takes ~8 waves (39 us per layer in the configs[1] replay, 4% of HBM).  Here:
//  * work units (request b, KV head, 128-key chunk) -- chunking by context length only;
//  * a persistent grid of 3 CTAs per SM of the partition walks the units; in a unit each of the 4
//    warps stages 32 keys of K and V (cp.async, 16-byte chunks, zero-filled past the context) and
//    computes the 16-row (GQA group on M) scores, online softmax and P.V on mma.sync m16n8k16;
//  * the 4 warp states are merged in warp order into a chunk partial (m, l, o) in the workspace;
//    the CTA that completes a (request, KV head) (atomic ticket) merges its chunk partials in chunk
//    order, 16 chunk loads in flight per output quad;
//  * every reduction order depends on the context lengths only, never on the grid -> bitwise
//    identical on any partition (co-execution == serial).
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace nova {

int g_dec_attn_p = getenv("NOVA_DEC_ATTN_P") ? atoi(getenv("NOVA_DEC_ATTN_P")) : 0;  // measured: no gain

namespace {

constexpr float LOG2E_P = 1.4426950408889634f;
constexpr int PW = 4;     // warps per CTA
constexpr int PK = 32;    // keys per warp block
constexpr int CKP = PW * PK;  // keys per unit (128)
constexpr int PCPS = 3;   // CTAs per SM of the partition

template <int HD>
struct PCfg2 {
  static constexpr int HDP = HD + 8;                    // padded rows (conflict-free ldmatrix)
  static constexpr int Q_BYTES = 16 * HDP * 2;
  static constexpr int SLOT = 2 * PK * HDP * 2;          // one warp's K + V block; later its f32 state
  static constexpr int SMEM = Q_BYTES + PW * SLOT + 64;
  static_assert(16 * (HD + 2) * 4 <= SLOT, "warp state fits its slot");
};

template <int HD>
__global__ void __launch_bounds__(32 * PW, PCPS)
    decode_attn_p_kernel(const bf16* __restrict__ qkv, int ld, bf16* __restrict__ out, int ldo,
                         const bf16* __restrict__ pool, int layer, int n_pages, int H, int KV,
                         const int* __restrict__ bt, int max_pages, const DecodeRow* __restrict__ rows, int B,
                         float* __restrict__ ws, int* __restrict__ tickets, int mch, float scale_log2) {
  using C = PCfg2<HD>;
  constexpr int HDP = C::HDP, KT = HD / 16, DT = HD / 8, CH = HD / 8;
  extern __shared__ __align__(16) uint8_t psm[];
  bf16* sQ = reinterpret_cast<bf16*>(psm);
  uint8_t* slots = psm + C::Q_BYTES;
  int* sInt = reinterpret_cast<int*>(psm + C::Q_BYTES + PW * C::SLOT);  // [0] ticket flag, [1..17] unit prefix
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, c4 = lane & 3;
  const int GQ = H / KV;
  const int Ghd = 32 + GQ * HD;  // chunk partial: m[16] | l[16] | o[GQ][HD]
  const size_t page_stride = (size_t)2 * KV * 64 * HD;
  const bf16* lbase = pool + (size_t)layer * n_pages * page_stride;

  pdl_launch_dependents();
  pdl_wait();  // rows, q and this step's K/V are written by the previous kernels
  if (tid == 0) {
    int cum = 0;
    for (int b = 0; b < B; ++b) {
      sInt[1 + b] = cum;
      cum += KV * ((rows[b].ctx + 1 + CKP - 1) / CKP);
    }
    sInt[1 + B] = cum;
  }
  __syncthreads();
  const int U = sInt[1 + B];
  bf16* wK = reinterpret_cast<bf16*>(slots + warp * C::SLOT);
  bf16* wV = wK + PK * HDP;
  float* wS = reinterpret_cast<float*>(slots + warp * C::SLOT);  // the warp's state after its compute

  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    int b = 0;
    while (b + 1 < B && sInt[2 + b] <= u) ++b;
    const DecodeRow rr = rows[b];
    const int L = rr.ctx + 1, nch = (L + CKP - 1) / CKP;
    const int r = u - sInt[1 + b];
    const int kvh = r / nch, ch = r % nch;
    const int k0 = ch * CKP + warp * PK;  // this warp's first key
    // stage this warp's K / V block (zero-filled past the context) and the group's Q rows
    const int* btr = bt + (size_t)rr.slot * max_pages;
    for (int i = lane; i < PK * CH; i += 32) {
      const int rrow = i / CH, cc = i % CH;
      const int j = k0 + rrow;
      const bool ok = j < L;
      const int jj = ok ? j : 0;
      const bf16* kp = lbase + (size_t)btr[jj >> 6] * page_stride + ((size_t)kvh * 64 + (jj & 63)) * HD + cc * 8;
      cp_async16(wK + rrow * HDP + cc * 8, kp, ok);
      cp_async16(wV + rrow * HDP + cc * 8, kp + (size_t)KV * 64 * HD, ok);
    }
    cp_async_commit();
    for (int i = tid; i < 16 * CH; i += 32 * PW) {
      const int rrow = i / CH, cc = i % CH;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (rrow < GQ) v = *reinterpret_cast<const uint4*>(qkv + (size_t)b * ld + (size_t)(kvh * GQ + rrow) * HD + cc * 8);
      *reinterpret_cast<uint4*>(sQ + rrow * HDP + cc * 8) = v;
    }
    cp_async_wait<0>();
    __syncthreads();
    float mx[2] = {-1e30f, -1e30f}, ls[2] = {0.f, 0.f};
    float o[DT][4];
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
    if (k0 < L) {
      float sc[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
          uint32_t qa[4], bb[2];
          ldmatrix_x4(qa, smem_u32(sQ + (lane & 15) * HDP + kk * 16 + (lane >> 4) * 8));
          ldmatrix_x2(bb, smem_u32(wK + (nt * 8 + (lane & 7)) * HDP + kk * 16 + ((lane >> 3) & 1) * 8));
          mma_bf16_16816(sc[nt], qa, bb);
        }
      }
      float bm[2] = {-1e30f, -1e30f};
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool ok = k0 + nt * 8 + 2 * c4 + (e & 1) < L;
          sc[nt][e] = ok ? sc[nt][e] * scale_log2 : -1e30f;
          bm[e >> 1] = fmaxf(bm[e >> 1], sc[nt][e]);
        }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        bm[q] = fmaxf(bm[q], __shfl_xor_sync(0xffffffffu, bm[q], 1));
        bm[q] = fmaxf(bm[q], __shfl_xor_sync(0xffffffffu, bm[q], 2));
        mx[q] = bm[q];
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
      for (int q = 0; q < 2; ++q) {
        ps[q] += __shfl_xor_sync(0xffffffffu, ps[q], 1);
        ps[q] += __shfl_xor_sync(0xffffffffu, ps[q], 2);
        ls[q] = ps[q];
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          uint32_t bb[2];
          ldmatrix_x2_trans(bb, smem_u32(wV + (kk * 16 + (lane & 15)) * HDP + dt * 8));
          mma_bf16_16816(o[dt], pa[kk], bb);
        }
    }
    __syncwarp();  // the slot's K / V are consumed: it now holds the warp state [16][HD + 2]
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int row = g + 8 * q;
      float* w = wS + row * (HD + 2);
      if (c4 == 0) {
        w[0] = mx[q];
        w[1] = ls[q];
      }
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        w[2 + dt * 8 + 2 * c4] = o[dt][2 * q];
        w[2 + dt * 8 + 2 * c4 + 1] = o[dt][2 * q + 1];
      }
    }
    __syncthreads();
    // chunk partial = the 4 warp states merged in warp order
    float* part = ws + (((size_t)b * KV + kvh) * mch + ch) * Ghd;
    auto wst = [&](int w) { return reinterpret_cast<const float*>(slots + w * C::SLOT); };
    if (tid < GQ) {
      float M = -1e30f;
#pragma unroll
      for (int w = 0; w < PW; ++w) M = fmaxf(M, wst(w)[tid * (HD + 2)]);
      float l = 0.f;
#pragma unroll
      for (int w = 0; w < PW; ++w) l += exp2f(wst(w)[tid * (HD + 2)] - M) * wst(w)[tid * (HD + 2) + 1];
      part[tid] = M;
      part[16 + tid] = l;
    }
    for (int i = tid; i < GQ * HD; i += 32 * PW) {
      const int row = i / HD, d = i % HD;
      float M = -1e30f;
#pragma unroll
      for (int w = 0; w < PW; ++w) M = fmaxf(M, wst(w)[row * (HD + 2)]);
      float num = 0.f;
#pragma unroll
      for (int w = 0; w < PW; ++w) num += exp2f(wst(w)[row * (HD + 2)] - M) * wst(w)[row * (HD + 2) + 2 + d];
      part[32 + i] = num;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) sInt[0] = atomicAdd(tickets + b * KV + kvh, 1) == nch - 1;
    __syncthreads();
    const bool last = sInt[0];
    if (last) {
      __threadfence();
      // merge the chunk partials in chunk order (f_c = 2^(m_c - M)); slots reused as [MAXCH][16] f, den
      float* sF = reinterpret_cast<float*>(slots);
      float* sL = sF + 64 * 16;
      float* sDen = sL + 64 * 16;
      const float* base = ws + ((size_t)b * KV + kvh) * mch * Ghd;
      for (int i = tid; i < nch * GQ; i += 32 * PW) {
        const int cc = i / GQ, row = i % GQ;
        sF[cc * 16 + row] = __ldcg(base + (size_t)cc * Ghd + row);
        sL[cc * 16 + row] = __ldcg(base + (size_t)cc * Ghd + 16 + row);
      }
      __syncthreads();
      if (tid < GQ) {
        float M = -1e30f;
        for (int cc = 0; cc < nch; ++cc) M = fmaxf(M, sF[cc * 16 + tid]);
        float den = 0.f;
        for (int cc = 0; cc < nch; ++cc) {
          const float f = exp2f(sF[cc * 16 + tid] - M);
          sF[cc * 16 + tid] = f;
          den += f * sL[cc * 16 + tid];
        }
        sDen[tid] = den;
      }
      __syncthreads();
      for (int i = tid; i < GQ * HD / 4; i += 32 * PW) {
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
        bf16* dst = out + (size_t)b * ldo + (size_t)(kvh * GQ + row) * HD + d;
        *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(num.x * inv, num.y * inv), pack_bf16(num.z * inv, num.w * inv));
      }
      if (tid == 0) tickets[b * KV + kvh] = 0;
    }
    __syncthreads();  // slots / sQ / sInt[0] reused by the next unit
  }
}

std::mutex g_p_mu;

template <int HD>
cudaError_t dap_launch(const bf16* qkv, int ld, bf16* out, int ldo, const bf16* pool, int layer, int n_pages, int H,
                       int KV, const int* bt, int max_pages, const DecodeRow* rows, int B, int max_ctx, float* ws,
                       int* tickets, int mch, int sms, cudaStream_t s) {
  using C = PCfg2<HD>;
  static bool set = false;
  {
    std::lock_guard<std::mutex> g(g_p_mu);
    if (!set) {
      cudaError_t e = cudaFuncSetAttribute(decode_attn_p_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      if (e != cudaSuccess) return e;
      set = true;
    }
  }
  // units of the largest request bound the useful grid
  const int nmax = B * KV * ((max_ctx + 1 + CKP - 1) / CKP);
  int grid = PCPS * (sms > 0 ? sms : 148);
  if (grid > nmax) grid = nmax;
  if (grid < 1) grid = 1;
  return launch_k(decode_attn_p_kernel<HD>, dim3(grid), dim3(32 * PW), C::SMEM, s, true, qkv, ld, out, ldo, pool,
                  layer, n_pages, H, KV, bt, max_pages, rows, B, ws, tickets, mch, LOG2E_P / sqrtf((float)HD));
}

}  // namespace

int decode_attn_p_chunk() { return CKP; }

cudaError_t decode_attn_p(const bf16* qkv, int ld, bf16* out, int ldo, const bf16* pool, int layer, int n_pages, int H,
                          int KV, int hd, const int* bt, int max_pages, const DecodeRow* rows, int B, int max_ctx,
                          float* ws, int* tickets, int mch, int sms, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (B > 16 || H % KV || H / KV > 16 || ld % 8 || (max_ctx + 1 + CKP - 1) / CKP > std::min(mch, 64))
    return cudaErrorInvalidValue;
  switch (hd) {
    case 32: return dap_launch<32>(qkv, ld, out, ldo, pool, layer, n_pages, H, KV, bt, max_pages, rows, B, max_ctx, ws, tickets, mch, sms, s);
    case 64: return dap_launch<64>(qkv, ld, out, ldo, pool, layer, n_pages, H, KV, bt, max_pages, rows, B, max_ctx, ws, tickets, mch, sms, s);
    case 128:
      return dap_launch<128>(qkv, ld, out, ldo, pool, layer, n_pages, H, KV, bt, max_pages, rows, B, max_ctx, ws, tickets, mch, sms, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nova
