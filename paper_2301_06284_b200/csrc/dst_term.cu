// dst_term.cu -- the RGAT destination term of dW and dA (DESIGN.md Sec. 6 "a5").
//
// The score's destination half is A[r,1].(x_dst W_r), so the backward carries
//   dW_r += c_r (x) A[r,1],  dA[r,1] = c_r W_r,  c_r = sum_{e in r} dpre_e x_dst(e).
// Positions are in (etype, dst) order: inside a relation, equal destinations
// are contiguous.  c_r is linear in the pieces, so any split of the positions
// that does not cut through a destination run may sum dpre per piece first:
//   c_r = sum_pieces (sum_{p in piece} dpre[p]) x_{v(piece)}.
// A warp takes 32 positions at a time, forms the pieces with a segmented
// shuffle scan keyed by dst, and gathers one X row per piece (not per edge),
// four pieces' rows in flight at a time (one vector load per lane and row).
// Blocks follow the dW chunk table (never straddling relations), warps stride
// over the chunk, warps are combined in a fixed order: deterministic.
#include "kernels.cuh"

namespace rgnn {

template <typename T, int K>
#ifndef RGNN_DST_MINB
#define RGNN_DST_MINB 3  // minimum resident 512-thread blocks per SM (measured r02 on ogbn-mag: 1 -> 0.27 ms, 3 -> 0.20,
                         // 4 -> 0.21)
#endif
__global__ void __launch_bounds__(512, RGNN_DST_MINB) k_dst_term(const Tile* __restrict__ chunks, const int32_t* __restrict__ dst_s,
                                                  const float* __restrict__ dpre, const T* __restrict__ X, int64_t v0,
                                                  float* __restrict__ cpart) {
  // lane l holds features l*FPL .. l*FPL+FPL-1 (one 4- or 8-byte load per X row); K = 32: one each
  constexpr int FPL = K / 32 >= 1 ? K / 32 : 1, NW = 16, GRP = 4;
  __shared__ float s_acc[NW][K];
  const Tile ch = chunks[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[FPL];
#pragma unroll
  for (int i = 0; i < FPL; ++i) acc[i] = 0.f;
  for (int base = ch.row0 + warp * 32; base < ch.row1; base += NW * 32) {
    const int p = base + lane;
    const bool valid = p < ch.row1;
    const int key = valid ? __ldg(dst_s + p) : -1;
    float d = valid ? __ldg(dpre + p) : 0.f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // segmented inclusive scan (segments = equal, contiguous keys)
      const float y = __shfl_up_sync(0xffffffffu, d, o);
      const int ky = __shfl_up_sync(0xffffffffu, key, o);
      if (lane >= o && ky == key) d += y;
    }
    const int knext = __shfl_down_sync(0xffffffffu, key, 1);
    const bool last = valid && (lane == 31 || knext != key);
    uint32_t mask = __ballot_sync(0xffffffffu, last);
    // GRP pieces at a time: their X rows are loaded together (independent loads in flight), then
    // accumulated in piece order
    while (mask) {
      float D[GRP], xf[GRP][FPL];
#pragma unroll
      for (int g = 0; g < GRP; ++g) {
        D[g] = 0.f;
#pragma unroll
        for (int i = 0; i < FPL; ++i) xf[g][i] = 0.f;
        if (mask) {
          const int l = __ffs(mask) - 1;
          mask &= mask - 1;
          D[g] = __shfl_sync(0xffffffffu, d, l);
          const int v = __shfl_sync(0xffffffffu, key, l);
          const T* xv = X + (v0 + v) * (int64_t)K + lane * FPL;
          if (lane * FPL < K) {
            if constexpr (sizeof(T) == 2 && FPL == 4) {
              const uint2 u = __ldg(reinterpret_cast<const uint2*>(xv));
              const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
              const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
              xf[g][0] = a.x; xf[g][1] = a.y; xf[g][2] = b.x; xf[g][3] = b.y;
            } else if constexpr (sizeof(T) == 2 && FPL == 2) {
              const uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(xv));
              const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
              xf[g][0] = a.x; xf[g][1] = a.y;
            } else {
#pragma unroll
              for (int i = 0; i < FPL; ++i) xf[g][i] = to_f(xv[i]);
            }
          }
        }
      }
#pragma unroll
      for (int g = 0; g < GRP; ++g)
#pragma unroll
        for (int i = 0; i < FPL; ++i) acc[i] = fmaf(D[g], xf[g][i], acc[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < FPL; ++i) {
    const int k = lane * FPL + i;
    if (k < K) s_acc[warp][k] = acc[i];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += s_acc[w][k];
    cpart[(size_t)blockIdx.x * K + k] = s;
  }
}

rgnn_status launch_dst_term(int prec, int K, const rgnn_graph* g, const float* dpre, const void* X, float* cpart,
                            cudaStream_t s) {
  if (g->num_chunks == 0) return RGNN_OK;
  const unsigned grid = (unsigned)g->num_chunks;
#define RGNN_DST(KK)                                                                                               \
  case KK:                                                                                                         \
    if (prec == RGNN_BF16)                                                                                         \
      RGNN_LAUNCH((k_dst_term<__nv_bfloat16, KK>), grid, 512, 0, s, g->chunks, g->dst_s, dpre,                     \
                  static_cast<const __nv_bfloat16*>(X), g->v0, cpart);                                             \
    else                                                                                                           \
      RGNN_LAUNCH((k_dst_term<float, KK>), grid, 512, 0, s, g->chunks, g->dst_s, dpre, static_cast<const float*>(X), \
                  g->v0, cpart);                                                                                   \
    return RGNN_OK;
  switch (K) {
    RGNN_DST(32)
    RGNN_DST(64)
    RGNN_DST(128)
    default:
      return set_error(RGNN_E_UNSUPPORTED, "d_in=%d", K);
  }
#undef RGNN_DST
}

}  // namespace rgnn
