// dx.cu -- input-feature gradient dX of one layer (
// the paper keeps the "required gradients").
//
// Chain rule of the forward (Listing 1; RGCN P:269-275), per edge e
// = (u -> v, r) with owned destination v:
//   RGAT  dX_u += dzs_e W_r^T,  dzs_e = alpha_e G_v + dpre_e A[r,0]
//         dX_v += dpre_e A[r,1] W_r^T = dpre_e U1_r         (U1_r = W_r A[r,1])
//   RGCN  dX_u += (1/c_e) G_v W_r^T ;  dX_v += G_v W0^T (self loop)
// Reordered by linearity (the paper's linear-operator reordering):
// G_v W_r^T depends only on the (etype, dst) run j of e, so
//   H_j = G_{v_j} W_{r_j}^T          one typed GEMM over the J runs (J << E), fp32
//   dX_u = sum_{e: src=u} (alpha_e H_{j(e)} + dpre_e U0_{r(e)})   [RGAT]
//        = sum_{e: src=u} (1/c_e) H_{j(e)}                        [RGCN]
//   dX_v += sum_{e: dst=v} dpre_e U1_{r(e)}   [RGAT]  /  + H0_v [RGCN, H0 = G W0^T]
// The source sums walk a source-major CSR over the positions (built by
// rgnn_graph_create with RGNN_GRAPH_DX): no atomics, fixed order, deterministic.
#include "kernels.cuh"

namespace rgnn {

__device__ __forceinline__ uint32_t tc_pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Wt[r] = W[r]^T : [R, K, N] -> [R, N, K]; on the bf16 path the RNE-rounded
// weight (the values the forward multiplied, reading O16), kept in fp32
__global__ void k_transpose_w(int R, int K, int N, const float* __restrict__ W, float* __restrict__ Wt,
                              int round_bf16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)R * K * N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ((int64_t)K * N), rem = i - r * K * N, k = rem / N, n = rem - k * N;
    const float w = W[i];
    Wt[(r * N + n) * K + k] = round_bf16 ? __bfloat162float(__float2bfloat16_rn(w)) : w;
  }
}

// Source sums.  One warp per source work item (a source node, or a <= cap-slot
// chunk of a hub source); an H row (K fp32) is read by L = K/4 lanes with
// 16-byte loads, the warp's 32/L lane groups take interleaved slots, group
// states merge in a fixed xor tree.  Chunks of split sources write partial
// rows, summed in order by k_dx_merge.
template <int K, bool RGAT, typename TH>
__global__ void __launch_bounds__(256) k_dx_walk(DxArgs a) {
  constexpr int EPL = 16 / sizeof(TH);
  constexpr int L = K / EPL;
  constexpr int G = 32 / L;
  static_assert(L >= 1 && L <= 32, "dx walk shape");
  const TH* H = static_cast<const TH*>(a.H);
  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp0; w < a.num_items; w += nwarps) {
    const Item it = a.items[w];
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    for (int32_t q = it.q0 + g; q < it.q1; q += G) {
      const int32_t j = a.srun[q];
      float c, d = 0.f;
      int32_t r = 0;
      if constexpr (RGAT) {
        const float2 ad = a.ad[a.spos[q]];
        c = ad.x;
        d = ad.y;
        r = a.srel[q];
      } else {
        c = a.wpos ? a.wpos[a.spos[q]] : a.sinvc[q];
      }
      float hf[EPL];
      Vec16<TH>{ldg16(H + (size_t)j * K + l * EPL)}.to_float(hf);
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] = fmaf(c, hf[i], acc[i]);
      if constexpr (RGAT) {
#pragma unroll
        for (int i = 0; i < EPL; i += 4) {
          const float4 u0 = __ldg(reinterpret_cast<const float4*>(a.U0 + (size_t)r * K + l * EPL + i));
          acc[i] = fmaf(d, u0.x, acc[i]); acc[i + 1] = fmaf(d, u0.y, acc[i + 1]);
          acc[i + 2] = fmaf(d, u0.z, acc[i + 2]); acc[i + 3] = fmaf(d, u0.w, acc[i + 3]);
        }
      }
    }
#pragma unroll
    for (int o = L; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    if (g == 0) {
      if (!RGAT && a.outb && it.part < 0) {  // bf16 row in node-type order (HGT dk / dv)
        uint32_t* ob = reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(a.outb) + (size_t)a.orow[it.row] * K +
                                                   l * EPL);
#pragma unroll
        for (int i = 0; i < EPL; i += 2) ob[i / 2] = tc_pack_bf16(acc[i], acc[i + 1]);
      } else {
        float* out = it.part < 0 ? a.dX + (size_t)it.row * K : a.part + (size_t)it.part * K;
#pragma unroll
        for (int i = 0; i < EPL; i += 4)
          stg16(out + l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]),
                                              __float_as_uint(acc[i + 2]), __float_as_uint(acc[i + 3])));
      }
    }
  }
}

template <int K>
__global__ void __launch_bounds__(256) k_dx_merge(DxArgs a) {
  for (int64_t w = blockIdx.x; w < a.num_split; w += gridDim.x) {
    const SplitRow sr = a.split[w];
    if (a.outb)
      merge_parts<K>(a.part, sr.part0, sr.nparts,
                     static_cast<__nv_bfloat16*>(a.outb) + (size_t)a.orow[sr.row] * K, false);
    else
      merge_parts<K>(a.part, sr.part0, sr.nparts, a.dX + (size_t)sr.row * K, false);
  }
}

// Destination terms of the owned rows, added after the source sums:
//   RGAT dX_v += sum_{slots q of v} dpre_q U1_{r_q}   over the destination work items
//   (CSR-by-dst slots, hub rows split into <= cap chunks whose partial rows are
//   summed in order by k_dx_dst_merge);  RGCN dX_v += H0_v (self loop).
template <int K>
__global__ void __launch_bounds__(256) k_dx_dst_rgat(DxArgs a) {
  constexpr int KL = K / 32;  // features per lane
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = w0; w < a.num_ditems; w += nw) {
    const Item it = a.ditems[w];
    float acc[KL];
#pragma unroll
    for (int i = 0; i < KL; ++i) acc[i] = 0.f;
    // slots of a row come grouped by relation: sum dpre along each (etype, dst) run and do
    // the K-wide update once per run
    int32_t cr = -1;
    float ds = 0.f;
    for (int32_t base = it.q0; base < it.q1; base += 32) {
      const int32_t q = base + lane;
      const bool ok = q < it.q1;
      const float dp = ok ? a.ad[a.pos[q]].y : 0.f;
      const int32_t r = ok ? a.et_slot[q] : 0;
      const int cnt = min(32, it.q1 - base);
      for (int t = 0; t < cnt; ++t) {
        const float d = __shfl_sync(0xffffffffu, dp, t);
        const int32_t rt = __shfl_sync(0xffffffffu, r, t);
        if (rt != cr) {  // warp-uniform
          if (cr >= 0) {
            const float* u1 = a.U1 + (size_t)cr * K + lane;
#pragma unroll
            for (int i = 0; i < KL; ++i) acc[i] = fmaf(ds, __ldg(u1 + 32 * i), acc[i]);
          }
          cr = rt;
          ds = 0.f;
        }
        ds += d;
      }
    }
    if (cr >= 0) {
      const float* u1 = a.U1 + (size_t)cr * K + lane;
#pragma unroll
      for (int i = 0; i < KL; ++i) acc[i] = fmaf(ds, __ldg(u1 + 32 * i), acc[i]);
    }
    if (it.part < 0) {
      float* out = a.dX + (size_t)(a.v0 + it.row) * K + lane;
#pragma unroll
      for (int i = 0; i < KL; ++i) out[32 * i] += acc[i];
    } else {
      float* out = a.dpart + (size_t)it.part * K + lane;
#pragma unroll
      for (int i = 0; i < KL; ++i) out[32 * i] = acc[i];
    }
  }
}

template <int K>
__global__ void __launch_bounds__(256) k_dx_dst_merge(DxArgs a) {
  for (int64_t w = blockIdx.x; w < a.num_dsplit; w += gridDim.x) {
    const SplitRow sr = a.dsplit[w];
    merge_parts<K>(a.dpart, sr.part0, sr.nparts, a.dX + (size_t)(a.v0 + sr.row) * K, true);
  }
}

template <int K>
__global__ void __launch_bounds__(256) k_dx_self(DxArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.V_own * K;
       i += (int64_t)gridDim.x * blockDim.x)
    a.dX[(size_t)a.v0 * K + i] += static_cast<const float*>(a.H0)[i];
}

rgnn_status launch_transpose_w(int prec, int R, int K, int N, const float* W, float* Wt, cudaStream_t s) {
  const int64_t n = (int64_t)R * K * N;
  RGNN_LAUNCH(k_transpose_w, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s, R, K, N, W, Wt,
              prec == RGNN_BF16 ? 1 : 0);
  return RGNN_OK;
}

static unsigned warp_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, 148 * 16)); }

template <int K>
static rgnn_status dx_walk(bool rgat, const DxArgs& a, cudaStream_t s) {
  {
    Phase ph("dx_src", s);
    if (a.num_items > 0) {
      if (a.h_bf16) {
        if (rgat) RGNN_LAUNCH((k_dx_walk<K, true, __nv_bfloat16>), warp_grid(a.num_items), 256, 0, s, a);
        else RGNN_LAUNCH((k_dx_walk<K, false, __nv_bfloat16>), warp_grid(a.num_items), 256, 0, s, a);
      } else {
        if (rgat) RGNN_LAUNCH((k_dx_walk<K, true, float>), warp_grid(a.num_items), 256, 0, s, a);
        else RGNN_LAUNCH((k_dx_walk<K, false, float>), warp_grid(a.num_items), 256, 0, s, a);
      }
    }
    if (a.num_split > 0)
      RGNN_LAUNCH((k_dx_merge<K>), (unsigned)std::min<int64_t>(a.num_split, 148 * 8), 256, 0, s, a);
  }
  Phase ph("dx_dst", s);
  if (rgat) {
    if (a.num_ditems > 0) RGNN_LAUNCH((k_dx_dst_rgat<K>), warp_grid(a.num_ditems), 256, 0, s, a);
    if (a.num_dsplit > 0)
      RGNN_LAUNCH((k_dx_dst_merge<K>), (unsigned)std::min<int64_t>(a.num_dsplit, 148 * 8), 256, 0, s, a);
  } else if (a.H0 && a.V_own > 0) {
    const int64_t n = a.V_own * K;
    RGNN_LAUNCH((k_dx_self<K>), (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s, a);
  }
  return RGNN_OK;
}

// H is fp32 on both paths: rounding G or H to bf16 loses too much where the source sums cancel
// (measured against the oracle: 2-4% of rms(dX) at single elements, above reading O19's bf16 bound).
// dX must be zeroed by the caller (sources without out-edges keep 0).
rgnn_status launch_dx_walk(int K, bool rgat, const DxArgs& a, cudaStream_t s) {
  switch (K) {
    case 32: return dx_walk<32>(rgat, a, s);
    case 64: return dx_walk<64>(rgat, a, s);
    case 128: return dx_walk<128>(rgat, a, s);
    default: return set_error(RGNN_E_UNSUPPORTED, "d_in=%d not in {32,64,128}", K);
  }
}

}  // namespace rgnn
