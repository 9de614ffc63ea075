// hgt.cu -- HGT layer forward (PAPER.md P:280, P:355,
// P:520-521; reading O23):
//   k = x_s WK[tau(s)], q = x_t WQ[tau(t)], v = x_s WV[tau(s)]   node-typed linears (segment MM over
//                                                                 node-type segments)
//   kw = k W_{a,r},  m = v W_{m,r}        once per (etype, src) pair with compact rows (P:520-521:
//                                          "determined by source node features and edge types")
//   a_e = kw . q_t,  alpha = softmax over the incoming edges of t,  Y_t = sum alpha_e m_e
// The typed linears run on the same typed GEMM as RGCN/RGAT (tcgen05 on the bf16 path); this
// file holds the destination walk: a_e = kw . q_t is the paper's "edge-wise vector inner
// product" after the typed linear, fused with the online softmax and the aggregation.
#include <math_constants.h>

#include "kernels.cuh"

namespace rgnn {

// out[i] = ninv[idx[i]] : GEMM gather rows of the node-typed features (type-sorted rows)
__global__ void k_map_gather(int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ ninv,
                             int32_t* __restrict__ out, int64_t ofs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ninv[idx[i] + ofs];
}

// fp32 copies for the score path of the bf16 layer: X values (exact) and RNE-rounded weights
__global__ void k_bf16_to_f32(int64_t n, const __nv_bfloat16* __restrict__ a, float* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __bfloat162float(a[i]);
}
__global__ void k_round_bf16(int64_t n, const float* __restrict__ a, float* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __bfloat162float(__float2bfloat16_rn(a[i]));
}
rgnn_status launch_bf16_to_f32(int64_t n, const void* a, float* b, cudaStream_t s) {
  if (n == 0) return RGNN_OK;
  RGNN_LAUNCH(k_bf16_to_f32, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s, n,
              static_cast<const __nv_bfloat16*>(a), b);
  return RGNN_OK;
}
rgnn_status launch_round_bf16(int64_t n, const float* a, float* b, cudaStream_t s) {
  if (n == 0) return RGNN_OK;
  RGNN_LAUNCH(k_round_bf16, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s, n, a, b);
  return RGNN_OK;
}

__global__ void k_f32_to_bf16(int64_t n, const float* __restrict__ a, __nv_bfloat16* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __float2bfloat16_rn(a[i]);
}
rgnn_status launch_f32_to_bf16(int64_t n, const float* a, void* b, cudaStream_t s) {
  if (n == 0) return RGNN_OK;
  RGNN_LAUNCH(k_f32_to_bf16, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s, n, a,
              static_cast<__nv_bfloat16*>(b));
  return RGNN_OK;
}

// Zero the gradient rows the walks do not write (instead of clearing whole [V, N] buffers):
// dk / dv rows of nodes without out-edges (srow[u] == srow[u+1]), dq rows of the owned
// destinations without in-edges (empty_rows) and of the rows outside the owned range [v0, v1).
// Also used for dX (NEXT-2): dK = dV = dX, [v0, v1) = [0, V), no empty list.
__global__ void k_hgt_zero_rows(int64_t V, int N, const int32_t* __restrict__ srow, float* __restrict__ dK,
                                float* __restrict__ dV, int64_t v0, int64_t v1, const int32_t* __restrict__ empty_rows,
                                int64_t num_empty, float* __restrict__ dQ) {
  const int nch = N / 4;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < V; u += (int64_t)gridDim.x * blockDim.x) {
    if (srow[u] == srow[u + 1]) {  // one thread per node: only the rows to clear are written
      for (int c = 0; c < nch; ++c) {
        reinterpret_cast<float4*>(dK + (size_t)u * N)[c] = z;
        reinterpret_cast<float4*>(dV + (size_t)u * N)[c] = z;
      }
    }
    if (u < v0 || u >= v1)
      for (int c = 0; c < nch; ++c) reinterpret_cast<float4*>(dQ + (size_t)u * N)[c] = z;
    if (u < num_empty)
      for (int c = 0; c < nch; ++c) reinterpret_cast<float4*>(dQ + (size_t)(v0 + empty_rows[u]) * N)[c] = z;
  }
}
rgnn_status launch_hgt_zero_rows(int64_t V, int N, const int32_t* srow, float* dK, float* dV, int64_t v0, int64_t v1,
                                 const int32_t* empty_rows, int64_t num_empty, float* dQ, cudaStream_t s) {
  if (V == 0) return RGNN_OK;
  RGNN_LAUNCH(k_hgt_zero_rows, (unsigned)std::min<int64_t>((V + 255) / 256, 148 * 32), 256, 0, s, V, N, srow, dK, dV,
              v0, v1, empty_rows, num_empty, dQ);
  return RGNN_OK;
}

__global__ void k_hgt_zero_rows_b(int64_t V, int N, const int32_t* __restrict__ srow, const int32_t* __restrict__ ninv,
                                  uint4* __restrict__ dK, uint4* __restrict__ dV, int64_t v0, int64_t v1,
                                  const int32_t* __restrict__ empty_rows, int64_t num_empty, uint4* __restrict__ dQ) {
  const int nch = N / 8;  // 16-byte chunks of a bf16 row
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < V; u += (int64_t)gridDim.x * blockDim.x) {
    const size_t ro = (size_t)ninv[u] * nch;
    if (srow[u] == srow[u + 1])
      for (int c = 0; c < nch; ++c) { dK[ro + c] = z; dV[ro + c] = z; }
    if (u < v0 || u >= v1)
      for (int c = 0; c < nch; ++c) dQ[ro + c] = z;
    if (u < num_empty) {
      const size_t re = (size_t)ninv[v0 + empty_rows[u]] * nch;
      for (int c = 0; c < nch; ++c) dQ[re + c] = z;
    }
  }
}
rgnn_status launch_hgt_zero_rows_b(int64_t V, int N, const int32_t* srow, const int32_t* ninv, void* dK, void* dV,
                                   int64_t v0, int64_t v1, const int32_t* empty_rows, int64_t num_empty, void* dQ,
                                   cudaStream_t s) {
  if (V == 0) return RGNN_OK;
  RGNN_LAUNCH(k_hgt_zero_rows_b, (unsigned)std::min<int64_t>((V + 255) / 256, 148 * 32), 256, 0, s, V, N, srow, ninv,
              static_cast<uint4*>(dK), static_cast<uint4*>(dV), v0, v1, empty_rows, num_empty, static_cast<uint4*>(dQ));
  return RGNN_OK;
}

rgnn_status launch_map_gather(int64_t n, const int32_t* idx, const int32_t* ninv, int32_t* out, cudaStream_t s,
                              int64_t ofs) {
  if (n == 0) return RGNN_OK;
  RGNN_LAUNCH(k_map_gather, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s, n, idx, ninv, out,
              ofs);
  return RGNN_OK;
}

// One warp per work item (a destination row or a chunk of a hub row), as k_aggregate:
// L = N*sizeof(T)/16 lanes read a 16-byte slice of the kw row and of the m row of an
// edge; the warp's 32/L lane groups take interleaved edges with their own online
// (max, sum, acc) state, merged in a fixed xor tree.  Deterministic, no atomics.
// TS: type of the score factors kw and q (fp32 on both paths: bf16 logits lose ~2-4% of rms(Y)
// at single elements through exp, measured against the oracle; O23); TM: message type.
#ifndef RGNN_HGTF_MINB
#define RGNN_HGTF_MINB 1
#endif
template <typename TS, typename TM, int N>
__global__ void __launch_bounds__(256, RGNN_HGTF_MINB) k_aggregate_hgt(HgtAggArgs a) {
  constexpr int EPL = 16 / sizeof(TM);
  constexpr int SV = EPL * sizeof(TS) / 16;  // 16-byte vectors of a lane's kw / q slice
  constexpr int L = N / EPL;
  constexpr int G = 32 / L;
  constexpr int UNR = G >= 4 ? 2 : 4;
  constexpr int B = G * UNR;
  static_assert(L >= 1 && L <= 32 && B <= 32, "hgt walk shape");
  const TS* KW = static_cast<const TS*>(a.KW);
  const TM* M = static_cast<const TM*>(a.M);
  const TS* Q = static_cast<const TS*>(a.Q);
  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp0; w < a.num_items; w += nwarps) {
    const Item it = a.items[w];
    float qf[EPL];
    {
      const TS* qp = Q + (size_t)a.ninv[a.v0 + it.row] * N + l * EPL;
#pragma unroll
      for (int v = 0; v < SV; ++v) Vec16<TS>{ldg16(qp + v * (16 / sizeof(TS)))}.to_float(qf + v * (16 / sizeof(TS)));
    }
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    float m = -CUDART_INF_F, lsum = 0.f;
    int nq = it.q0 + lane;
    int np = (lane < B && nq < it.q1) ? a.pos[nq] : 0;
    for (int base = it.q0; base < it.q1; base += B) {
      const int myp = np;
      nq = base + B + lane;
      np = (lane < B && nq < it.q1) ? a.pos[nq] : 0;
      uint4 kr[UNR][SV], mr[UNR];
      bool val[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int j = u * G + g;
        const int p = __shfl_sync(0xffffffffu, myp, j);
        val[u] = base + j < it.q1;
#pragma unroll
        for (int v = 0; v < SV; ++v)
          kr[u][v] = val[u] ? ldg16(KW + (size_t)p * N + l * EPL + v * (16 / sizeof(TS))) : make_uint4(0, 0, 0, 0);
        mr[u] = val[u] ? ldg16(M + (size_t)p * N + l * EPL) : make_uint4(0, 0, 0, 0);
      }
      float sc[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        float kf[EPL];
#pragma unroll
        for (int v = 0; v < SV; ++v) Vec16<TS>{kr[u][v]}.to_float(kf + v * (16 / sizeof(TS)));
        float d = 0.f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) d = fmaf(kf[i], qf[i], d);
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        sc[u] = val[u] ? d : -CUDART_INF_F;
      }
      float mnew = m;
#pragma unroll
      for (int u = 0; u < UNR; ++u) mnew = fmaxf(mnew, sc[u]);
      if (mnew != -CUDART_INF_F) {
        const float corr = __expf(m - mnew);
        lsum *= corr;
#pragma unroll
        for (int i = 0; i < EPL; ++i) acc[i] *= corr;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const float e = val[u] ? __expf(sc[u] - mnew) : 0.f;
          lsum += e;
          float mf[EPL];
          Vec16<TM>{mr[u]}.to_float(mf);
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] = fmaf(e, mf[i], acc[i]);
        }
        m = mnew;
      }
    }
#pragma unroll
    for (int o = L; o < 32; o <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float l2 = __shfl_xor_sync(0xffffffffu, lsum, o);
      const float mn = fmaxf(m, m2);
      const float c1 = mn == -CUDART_INF_F ? 0.f : __expf(m - mn);
      const float c2 = mn == -CUDART_INF_F ? 0.f : __expf(m2 - mn);
      lsum = lsum * c1 + l2 * c2;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const float a2 = __shfl_xor_sync(0xffffffffu, acc[i], o);
        acc[i] = acc[i] * c1 + a2 * c2;
      }
      m = mn;
    }
    if (g == 0) {
      if (it.part < 0) {
        const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
        float* y = a.Y + (size_t)it.row * N + l * EPL;
#pragma unroll
        for (int i = 0; i < EPL; i += 4)
          stg16(y + i, make_uint4(__float_as_uint(acc[i] * inv), __float_as_uint(acc[i + 1] * inv),
                                  __float_as_uint(acc[i + 2] * inv), __float_as_uint(acc[i + 3] * inv)));
        if (l == 0) a.lse[it.row] = lsum > 0.f ? m + __logf(lsum) : -CUDART_INF_F;
      } else {
        float* pp = a.part + (size_t)it.part * (N + 4);
#pragma unroll
        for (int i = 0; i < EPL; i += 4)
          stg16(pp + l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]),
                                             __float_as_uint(acc[i + 2]), __float_as_uint(acc[i + 3])));
        if (l == 0) { pp[N] = m; pp[N + 1] = lsum; }
      }
    }
  }
}

template <typename TM, int N>
static rgnn_status hgt_walk(const HgtAggArgs& a, cudaStream_t s) {
  if (a.num_items == 0) return RGNN_OK;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((a.num_items + 7) / 8, 148 * 16));
  RGNN_LAUNCH((k_aggregate_hgt<float, TM, N>), grid, 256, 0, s, a);
  return RGNN_OK;
}

// kw and q are fp32 on both paths; the message rows are bf16 on the bf16 path
rgnn_status launch_aggregate_hgt(int prec, int N, const HgtAggArgs& a, cudaStream_t s) {
  const bool bf = prec == RGNN_BF16;
  switch (N) {
    case 32: return bf ? hgt_walk<__nv_bfloat16, 32>(a, s) : hgt_walk<float, 32>(a, s);
    case 64: return bf ? hgt_walk<__nv_bfloat16, 64>(a, s) : hgt_walk<float, 64>(a, s);
    case 128: return bf ? hgt_walk<__nv_bfloat16, 128>(a, s) : hgt_walk<float, 128>(a, s);
    default: return set_error(RGNN_E_UNSUPPORTED, "d_out=%d not in {32,64,128}", N);
  }
}

// ---------------------------------------------------------------- backward
// Destination walk of the HGT backward (chain rule of the forward above; the oracle's
// oracle_hgt_backward states the same formulas):
//   S_t = G_t . Y_t = sum_e alpha_e (G_t . m_e),  alpha_e = exp(a_e - lse_t),  a_e = kw_e . q_t
//   da_e = alpha_e (G_t . m_e - S_t)       (d a_e, the score gradient)
//   dq_t = sum_e da_e kw_e                 (the query gradient, summed along the row: no atomics)
// alpha_e and da_e are stored by position: the source sums (dk, dv) and the relation dW GEMMs
// read them.  One warp per work item as the forward walk; a lane group of L = N*sizeof(TM)/16
// lanes handles one edge, its lanes each holding EPL features of kw, m, q, G and dq.
#ifndef RGNN_HGTB_UNR
#define RGNN_HGTB_UNR 4
#endif
#ifndef RGNN_HGTB_MINB
#define RGNN_HGTB_MINB 4
#endif
template <typename TM, int N>
__global__ void __launch_bounds__(256, RGNN_HGTB_MINB) k_hgt_bwd_walk(HgtBwdArgs a) {
  constexpr int EPL = 16 / sizeof(TM);
  constexpr int SV = EPL * 4 / 16;  // fp32 16-byte vectors per lane slice (kw, q, G, Y)
  constexpr int L = N / EPL;
  constexpr int G = 32 / L;
  constexpr int UNR = G >= 4 ? 1 : RGNN_HGTB_UNR;  // edges per lane group per step (rows in flight)
  constexpr int B = G * UNR;
  static_assert(L >= 1 && L <= 32 && B <= 32, "hgt bwd walk shape");
  const float* KW = static_cast<const float*>(a.KW);
  const TM* M = static_cast<const TM*>(a.M);
  const float* Q = static_cast<const float*>(a.Q);
  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp0; w < a.num_items; w += nwarps) {
    const Item it = a.items[w];
    float qf[EPL], gf[EPL];
    float S = 0.f;
    {
      const float* qp = Q + (size_t)a.ninv[a.v0 + it.row] * N + l * EPL;
      const float* gp = a.dY + (size_t)it.row * N + l * EPL;
      const float* yp = a.Y + (size_t)it.row * N + l * EPL;
#pragma unroll
      for (int v = 0; v < SV; ++v) {
        float yf[4];
        Vec16<float>{ldg16(qp + 4 * v)}.to_float(qf + 4 * v);
        Vec16<float>{ldg16(gp + 4 * v)}.to_float(gf + 4 * v);
        Vec16<float>{ldg16(yp + 4 * v)}.to_float(yf);
#pragma unroll
        for (int i = 0; i < 4; ++i) S = fmaf(gf[4 * v + i], yf[i], S);
      }
    }
    S = group_sum<L>(S);
    const float lse = a.lse[it.row];
    float dq[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) dq[i] = 0.f;
    for (int32_t base = it.q0; base < it.q1; base += B) {
      uint4 kr[UNR][SV], mr[UNR];
      int32_t pp[UNR];
      bool ok[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int32_t q = base + u * G + g;
        ok[u] = q < it.q1;
        pp[u] = ok[u] ? a.pos[q] : 0;
        const int32_t z = ok[u] ? (a.zrow ? a.zrow[q] : pp[u]) : 0;
#pragma unroll
        for (int v = 0; v < SV; ++v)
          kr[u][v] = ok[u] ? ldg16(KW + (size_t)z * N + l * EPL + 4 * v) : make_uint4(0, 0, 0, 0);
        mr[u] = ok[u] ? ldg16(M + (size_t)z * N + l * EPL) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        float kf[EPL], mf[EPL];
#pragma unroll
        for (int v = 0; v < SV; ++v) Vec16<float>{kr[u][v]}.to_float(kf + 4 * v);
        Vec16<TM>{mr[u]}.to_float(mf);
        float sa = 0.f, sd = 0.f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          sa = fmaf(kf[i], qf[i], sa);
          sd = fmaf(gf[i], mf[i], sd);
        }
        sa = group_sum<L>(sa);
        sd = group_sum<L>(sd);
        const float al = ok[u] ? __expf(sa - lse) : 0.f;
        const float dae = al * (sd - S);
        if (ok[u] && l == 0) {
          a.alpha[pp[u]] = al;
          a.da[pp[u]] = dae;
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) dq[i] = fmaf(dae, kf[i], dq[i]);
      }
    }
#pragma unroll
    for (int o = L; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < EPL; ++i) dq[i] += __shfl_xor_sync(0xffffffffu, dq[i], o);
    if (g == 0) {
      if (a.dQb && it.part < 0) {  // bf16 row in node-type order
        __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(a.dQb) + (size_t)a.ninv[a.v0 + it.row] * N + l * EPL;
#pragma unroll
        for (int i = 0; i < EPL; i += 2)
          *reinterpret_cast<__nv_bfloat162*>(ob + i) = __floats2bfloat162_rn(dq[i], dq[i + 1]);
      } else {
        float* out = it.part < 0 ? a.dQ + (size_t)(a.v0 + it.row) * N : a.part + (size_t)it.part * N;
#pragma unroll
        for (int i = 0; i < EPL; i += 4)
          stg16(out + l * EPL + i, make_uint4(__float_as_uint(dq[i]), __float_as_uint(dq[i + 1]),
                                              __float_as_uint(dq[i + 2]), __float_as_uint(dq[i + 3])));
      }
    }
  }
}

template <int N>
__global__ void __launch_bounds__(256) k_hgt_dq_merge(HgtBwdArgs a) {
  for (int64_t w = blockIdx.x; w < a.num_split_rows; w += gridDim.x) {
    const SplitRow sr = a.split_rows[w];
    if (a.dQb)
      merge_parts<N>(a.part, sr.part0, sr.nparts,
                     static_cast<__nv_bfloat16*>(a.dQb) + (size_t)a.ninv[a.v0 + sr.row] * N, false);
    else
      merge_parts<N>(a.part, sr.part0, sr.nparts, a.dQ + (size_t)(a.v0 + sr.row) * N, false);
  }
}

template <typename TM, int N>
static rgnn_status hgt_bwd_walk(const HgtBwdArgs& a, cudaStream_t s) {
  if (a.num_items > 0) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((a.num_items + 7) / 8, 148 * 16));
    RGNN_LAUNCH((k_hgt_bwd_walk<TM, N>), grid, 256, 0, s, a);
  }
  if (a.num_split_rows > 0)
    RGNN_LAUNCH((k_hgt_dq_merge<N>), (unsigned)std::min<int64_t>(a.num_split_rows, 148 * 8), 256, 0, s, a);
  return RGNN_OK;
}

// One warp per run piece (<= kPieceRows consecutive positions of one (etype, dst) run): lane
// groups of L = N*sizeof(T)/16 lanes gather the v and k rows of interleaved positions, fp32 sums
// merged in a fixed xor tree.  Positions are read in order (alpha, da, vrow contiguous).
template <typename TO, typename T, int N>
__global__ void __launch_bounds__(256) k_hgt_piece_agg(HgtPieceArgs a) {
  constexpr int EPL = 16 / sizeof(T);  // v and k rows: fp32, or their bf16 copies
  constexpr int L = N / EPL;
  constexpr int G = 32 / L;
  static_assert(L >= 1 && L <= 32, "piece agg shape");
  const T* Vn = static_cast<const T*>(a.Vn);
  const T* Kn = static_cast<const T*>(a.Kn);
  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp0; w < a.num_pieces; w += nwarps) {
    const int32_t p0 = a.piece_ptr[w], p1 = a.piece_ptr[w + 1];
    float va[EPL], ka[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) va[i] = ka[i] = 0.f;
    int32_t p = p0 + g;
    for (; p + G < p1; p += 2 * G) {  // two positions per group in flight
      const int32_t r0 = a.vrow[p], r1 = a.vrow[p + G];
      const float al0 = a.alpha[p], al1 = a.alpha[p + G], d0 = a.da[p], d1 = a.da[p + G];
      const uint4 v0 = ldg16(Vn + (size_t)r0 * N + l * EPL), v1 = ldg16(Vn + (size_t)r1 * N + l * EPL);
      const uint4 k0 = ldg16(Kn + (size_t)r0 * N + l * EPL), k1 = ldg16(Kn + (size_t)r1 * N + l * EPL);
      float f[EPL];
      Vec16<T>{v0}.to_float(f);
#pragma unroll
      for (int i = 0; i < EPL; ++i) va[i] = fmaf(al0, f[i], va[i]);
      Vec16<T>{v1}.to_float(f);
#pragma unroll
      for (int i = 0; i < EPL; ++i) va[i] = fmaf(al1, f[i], va[i]);
      Vec16<T>{k0}.to_float(f);
#pragma unroll
      for (int i = 0; i < EPL; ++i) ka[i] = fmaf(d0, f[i], ka[i]);
      Vec16<T>{k1}.to_float(f);
#pragma unroll
      for (int i = 0; i < EPL; ++i) ka[i] = fmaf(d1, f[i], ka[i]);
    }
    if (p < p1) {
      const int32_t r0 = a.vrow[p];
      const float al0 = a.alpha[p], d0 = a.da[p];
      float f[EPL];
      Vec16<T>{ldg16(Vn + (size_t)r0 * N + l * EPL)}.to_float(f);
#pragma unroll
      for (int i = 0; i < EPL; ++i) va[i] = fmaf(al0, f[i], va[i]);
      Vec16<T>{ldg16(Kn + (size_t)r0 * N + l * EPL)}.to_float(f);
#pragma unroll
      for (int i = 0; i < EPL; ++i) ka[i] = fmaf(d0, f[i], ka[i]);
    }
#pragma unroll
    for (int o = L; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        va[i] += __shfl_xor_sync(0xffffffffu, va[i], o);
        ka[i] += __shfl_xor_sync(0xffffffffu, ka[i], o);
      }
    if (g == 0) {
      TO* vo = static_cast<TO*>(a.vagg) + (size_t)w * N + l * EPL;
      TO* ko = static_cast<TO*>(a.kagg) + (size_t)w * N + l * EPL;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        vo[i] = from_f<TO>(va[i]);
        ko[i] = from_f<TO>(ka[i]);
      }
      if (l == 0) {
        const int32_t d = a.dst_s[p0];
        a.pdst[w] = d;
        a.pq[w] = a.ninv[a.v0 + d];
      }
    }
  }
}

rgnn_status launch_hgt_piece_agg(int prec, int N, const HgtPieceArgs& a, cudaStream_t s) {
  if (a.num_pieces == 0) return RGNN_OK;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((a.num_pieces + 7) / 8, 148 * 16));
  const bool bf = prec == RGNN_BF16;
#define RGNN_PIECE(TO, TI, n) \
  if (N == n) { RGNN_LAUNCH((k_hgt_piece_agg<TO, TI, n>), grid, 256, 0, s, a); return RGNN_OK; }
  if (bf && a.in_bf16) {
    RGNN_PIECE(__nv_bfloat16, __nv_bfloat16, 32) RGNN_PIECE(__nv_bfloat16, __nv_bfloat16, 64)
    RGNN_PIECE(__nv_bfloat16, __nv_bfloat16, 128)
  } else if (bf) {
    RGNN_PIECE(__nv_bfloat16, float, 32) RGNN_PIECE(__nv_bfloat16, float, 64) RGNN_PIECE(__nv_bfloat16, float, 128)
  } else { RGNN_PIECE(float, float, 32) RGNN_PIECE(float, float, 64) RGNN_PIECE(float, float, 128) }
#undef RGNN_PIECE
  return set_error(RGNN_E_UNSUPPORTED, "d_out=%d not in {32,64,128}", N);
}

rgnn_status launch_hgt_bwd_walk(int prec, int N, const HgtBwdArgs& a, cudaStream_t s) {
  const bool bf = prec == RGNN_BF16;
  switch (N) {
    case 32: return bf ? hgt_bwd_walk<__nv_bfloat16, 32>(a, s) : hgt_bwd_walk<float, 32>(a, s);
    case 64: return bf ? hgt_bwd_walk<__nv_bfloat16, 64>(a, s) : hgt_bwd_walk<float, 64>(a, s);
    case 128: return bf ? hgt_bwd_walk<__nv_bfloat16, 128>(a, s) : hgt_bwd_walk<float, 128>(a, s);
    default: return set_error(RGNN_E_UNSUPPORTED, "d_out=%d not in {32,64,128}", N);
  }
}

}  // namespace rgnn
