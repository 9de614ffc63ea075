// dst_term.cu -- the RGAT destination term of dW and dA (DESIGN.md Sec. 6 "a5").
//
// The score's destination half is A[r,1].(x_dst W_r), so the backward carries
//   dW_r += c_r (x) A[r,1],  dA[r,1] = c_r W_r,  c_r = sum_{e in r} dpre_e x_dst(e).
// Positions are in (etype, dst) order: inside a relation, equal destinations
// are contiguous.  c_r is linear in the pieces, so any split of the positions
// that does not cut through a destination run may sum dpre per piece first:
//   c_r = sum_pieces (sum_{p in piece} dpre[p]) x_{v(piece)}.
// A warp takes 32 positions at a time, forms the pieces with a segmented
// shuffle scan keyed by dst, and gathers one X row per piece (not per edge).
// Blocks follow the dW chunk table (never straddling relations), warps stride
// over the chunk, warps are combined in a fixed order: deterministic.
#include "kernels.cuh"

namespace rgnn {

template <typename T, int K>
__global__ void __launch_bounds__(512) k_dst_term(const Tile* __restrict__ chunks, const int32_t* __restrict__ dst_s,
                                                  const float* __restrict__ dpre, const T* __restrict__ X, int64_t v0,
                                                  float* __restrict__ cpart) {
  constexpr int PER = (K + 31) / 32, NW = 16;
  __shared__ float s_acc[NW][K];
  const Tile ch = chunks[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
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
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      const float D = __shfl_sync(0xffffffffu, d, l);
      const int v = __shfl_sync(0xffffffffu, key, l);
      const T* xv = X + (v0 + v) * (int64_t)K;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int k = lane + 32 * i;
        if (k < K) acc[i] = fmaf(D, to_f(xv[k]), acc[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int k = lane + 32 * i;
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
