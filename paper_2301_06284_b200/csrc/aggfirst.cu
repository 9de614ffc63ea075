// aggfirst.cu -- aggregate-first RGCN forward (the
// memory-bandwidth relief the paper lists as future work).
//
// RGCN is linear in the messages, so
//     Y_v = sum_r (1/c_{v,r}) sum_{e in run(r,v)} x_src(e) W_r = sum_runs (A_run) W_r,
// with A_run = (1/c) sum_{e in run} x_src(e): the per-edge products Z = x_src W_r of the
// GEMM-first formulation are never formed.  Runs are cut into pieces of <= kPieceRows positions
// (graph tables, RGNN_GRAPH_AGGFIRST) so no piece is long:
//   k_piece_agg : A_i = sum_{p in piece i} inv_c[p] X[src_s[p]]        (this file; inv_c is the
//                 position's RGCN factor, so per-edge norms (RGNN_NORM_EDGE) work too)
//   typed GEMM  : P_i = A_i W_r over the piece segments of each relation (tf32 tensor cores on the
//                 bf16 layer -- W bf16-valued, exact in tf32 --, SIMT fp32 on the fp32 layer)
//   dst walk    : Y_v = sum of the piece products of row v (each piece once: slot weights 1 / 0)
// A and P stay fp32 on both layers: a piece sum is a partial result of up to 64 edges, and rounding
// it (and its product) to bf16 puts two bf16 roundings at the scale of the sum where the GEMM-first
// path has one at the scale of an edge -- measured: up to 1.7x the bf16 bound at single elements.
#include "kernels.cuh"

namespace rgnn {

template <typename T, int K>
__global__ void __launch_bounds__(256) k_piece_agg(int64_t np, const int32_t* __restrict__ piece_ptr,
                                                   const float* __restrict__ inv_c,
                                                   const int32_t* __restrict__ src_s, const T* __restrict__ X,
                                                   float* __restrict__ A) {
  constexpr int EPL = 16 / sizeof(T), L = K / EPL, G = 32 / L;
  constexpr int UNR = L >= 4 ? 4 : L;  // positions in flight per lane group
  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L;
  const unsigned gmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (g * L));
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp0 * G + g; i - g < np; i += nwarps * G) {
    if (i >= np) continue;  // the whole group leaves together
    const int s0 = piece_ptr[i], s1 = piece_ptr[i + 1];
    float acc[EPL];
#pragma unroll
    for (int k = 0; k < EPL; ++k) acc[k] = 0.f;
    for (int base = s0; base < s1; base += UNR) {
      const bool ok = l < UNR && base + l < s1;
      const int mys = ok ? src_s[base + l] : 0;
      const float myw = ok ? inv_c[base + l] : 0.f;
      uint4 xr[UNR];
      float wv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int sidx = __shfl_sync(gmask, mys, u, L);
        wv[u] = __shfl_sync(gmask, myw, u, L);
        xr[u] = base + u < s1 ? ldg16(X + (size_t)sidx * K + l * EPL) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        float xf[EPL];
        Vec16<T>{xr[u]}.to_float(xf);
#pragma unroll
        for (int k = 0; k < EPL; ++k) acc[k] = fmaf(wv[u], xf[k], acc[k]);
      }
    }
    float* out = A + (size_t)i * K + l * EPL;
#pragma unroll
    for (int k = 0; k < EPL; k += 4)
      stg16(out + k, make_uint4(__float_as_uint(acc[k]), __float_as_uint(acc[k + 1]), __float_as_uint(acc[k + 2]),
                                __float_as_uint(acc[k + 3])));
  }
}

rgnn_status launch_piece_agg(int prec, int K, int64_t np, const int32_t* piece_ptr, const float* inv_c,
                             const int32_t* src_s, const void* X, void* A, cudaStream_t s) {
  if (np == 0) return RGNN_OK;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((np + 31) / 32, 148 * 16));
#define RGNN_PIECE_AGG(KK)                                                                                       \
  if (K == KK) {                                                                                                 \
    if (prec == RGNN_BF16)                                                                                       \
      RGNN_LAUNCH((k_piece_agg<__nv_bfloat16, KK>), grid, 256, 0, s, np, piece_ptr, inv_c, src_s,           \
                  static_cast<const __nv_bfloat16*>(X), static_cast<float*>(A));                         \
    else                                                                                                         \
      RGNN_LAUNCH((k_piece_agg<float, KK>), grid, 256, 0, s, np, piece_ptr, inv_c, src_s,                   \
                  static_cast<const float*>(X), static_cast<float*>(A));                                         \
    return RGNN_OK;                                                                                              \
  }
  RGNN_PIECE_AGG(32)
  RGNN_PIECE_AGG(64)
  RGNN_PIECE_AGG(128)
#undef RGNN_PIECE_AGG
  return set_error(RGNN_E_UNSUPPORTED, "d_in=%d", K);
}

}  // namespace rgnn
