// traverse.cu -- destination walks over CSR-by-dst (DESIGN.md Sec. 6 "a3", "a4").
//
// Forward (fused score + edge softmax + aggregate, no atomics):
//   The paper's edge loop is rewritten as a dst-node loop over incoming edges
//   (graph-semantic loop transform, Sec. 3.3.3, Sec. 3.4.2),
//   per-dst loads are hoisted out of the edge loop, and exp / sum /
//   divide of Listing 1's edge_softmax are fused with the
//   attention score and the alpha-weighted aggregation into one
//   pass with an online (running max) softmax -- exact in real arithmetic
//   (reading O5).  RGAT score: pre_e = s_src[p] + x_dst . U[r]  (the second
//   term computed once per (dst, relation) run of the row) where
//   s_src[p] = A[r,0].Z[p] came from the GEMM epilogue and U[r] = W_r A[r,1]
//   (linear-operator fusion, Sec. 3.4.1).
// One warp per work item (a row or a <= cap-edge chunk of a long row).  A Z
// row is read by L = N*sizeof(T)/16 lanes with 16-byte loads; the warp's
// G = 32/L lane groups take interleaved edges, each keeps its own online
// state, and the states are merged in a fixed shuffle tree: deterministic.
// Split rows write unnormalised partial states; k_merge combines them in slot
// order.
//
// Backward (RGAT): per edge recompute s_e and alpha_e = exp(s_e - lse_v),
//   dalpha_e = G_v . Z[p],  S_v = G_v . Y_v,
//   dpre_e = alpha_e (dalpha_e - S_v) leaky'(pre_e),
//   dZ[p] = alpha_e G_v + dpre_e A[r,0]   (stored in (etype,dst) order), dpre[p].
#include <math_constants.h>

#include "kernels.cuh"

namespace rgnn {

__device__ __forceinline__ float leaky(float x, float slope) { return x > 0.f ? x : slope * x; }

#ifndef RGNN_WALK_UNR
#define RGNN_WALK_UNR 4
#endif
#ifndef RGNN_WALK_UNR_NARROW
#define RGNN_WALK_UNR_NARROW 2  // rows narrower than 8 lanes' 16-byte slices (G >= 4 groups per warp)
#endif
template <typename T, int K, int N>
struct WalkShape {
  static constexpr int EPL = 16 / sizeof(T);  // features per lane (one 16-byte load)
  static constexpr int L = N / EPL;           // lanes per Z row
  static constexpr int G = 32 / L;            // edge groups per warp
  static constexpr int UNR = G >= 4 ? RGNN_WALK_UNR_NARROW : RGNN_WALK_UNR;  // edges per group per step
  static constexpr int B = G * UNR;           // edges per warp step (<= 32)
  static constexpr int KPL = K / L;           // x_dst features per lane
  static_assert(L >= 1 && L <= 32 && B <= 32, "shape");
  static_assert(K % L == 0, "K must be a multiple of the lane group");
};

// KPL consecutive features -> fp32 registers, 16-byte loads when the slice allows it.
template <int KPL, typename T>
__device__ __forceinline__ void load_slice(const T* p, float* out) {
  constexpr int V = 16 / sizeof(T);
  if constexpr (KPL % V == 0) {
#pragma unroll
    for (int i = 0; i < KPL; i += V) Vec16<T>{ldg16(p + i)}.to_float(out + i);
  } else {
#pragma unroll
    for (int i = 0; i < KPL; ++i) out[i] = to_f(p[i]);
  }
}

// x . U[r] over this lane's KPL features (U fp32, float4 loads when possible).
template <int KPL, bool SM = false>
__device__ __forceinline__ float dot_u(const float* xv, const float* Ur) {
  float d = 0.f;
  if constexpr (KPL % 4 == 0) {
#pragma unroll
    for (int i = 0; i < KPL; i += 4) {
      const float4 u = SM ? *reinterpret_cast<const float4*>(Ur + i) : __ldg(reinterpret_cast<const float4*>(Ur + i));
      d = fmaf(xv[i], u.x, d); d = fmaf(xv[i + 1], u.y, d); d = fmaf(xv[i + 2], u.z, d); d = fmaf(xv[i + 3], u.w, d);
    }
  } else {
#pragma unroll
    for (int i = 0; i < KPL; ++i) d = fmaf(xv[i], SM ? Ur[i] : __ldg(Ur + i), d);
  }
  return d;
}

// pre_u = s_src_u + x_dst . U[r_u] for the UNR edges of a lane group (same expression as the
// backward's pre).  CACHE: the slots of a row come grouped by relation ((etype, dst) positions
// in ascending order) and x_dst . U[r] depends only on (dst, r), so it is recomputed only when
// some group's relation changes (warp-uniform vote: no divergence) -- chosen for graphs with
// long (etype, dst) runs.  Otherwise one dot per edge, UNR independent chains.
template <int K, int L, int KPL, int UNR, bool CACHE, bool USM = false>
__device__ __forceinline__ void dst_scores(const float* xv, const float* U, int l, const int* rr, const float* ssv,
                                           int& cr, float& cd, float* sc) {
  if constexpr (CACHE) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (__any_sync(0xffffffffu, rr[u] != cr)) {
        float d = dot_u<KPL, USM>(xv, U + (size_t)rr[u] * K + l * KPL);
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        cd = d;
        cr = rr[u];
      }
      sc[u] = ssv[u] + cd;
    }
  } else {
#pragma unroll
    for (int u = 0; u < UNR; ++u) sc[u] = dot_u<KPL, USM>(xv, U + (size_t)rr[u] * K + l * KPL);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
#pragma unroll
      for (int o = L / 2; o > 0; o >>= 1) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
      sc[u] = ssv[u] + sc[u];
    }
  }
}

// Packed fp32x2 FMA / MUL (Blackwell FFMA2 / FMUL2): the same per-element rounding as fmaf / *,
// so results are bit-identical to the scalar loops, at half the instructions.
#ifndef RGNN_WALK_FFMA2
#define RGNN_WALK_FFMA2 0  // measured r02: FFMA2 on, ogbn-mag walk 1.82 -> 2.13 ms (register pressure); AM / wikikg2 unchanged
#endif
template <int EPL>
__device__ __forceinline__ void fma_acc(float* acc, float e, const float* z) {
  if constexpr (EPL % 2 == 0 && RGNN_WALK_FFMA2) {
#pragma unroll
    for (int i = 0; i < EPL; i += 2) {
      uint64_t a, b, c, d;
      asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(e), "f"(e));
      asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(z[i]), "f"(z[i + 1]));
      asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(acc[i]), "f"(acc[i + 1]));
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
      asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(d));
    }
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = fmaf(e, z[i], acc[i]);
  }
}
template <int EPL>
__device__ __forceinline__ void mul_acc(float* acc, float f) {
  if constexpr (EPL % 2 == 0 && RGNN_WALK_FFMA2) {
#pragma unroll
    for (int i = 0; i < EPL; i += 2) {
      uint64_t a, c, d;
      asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(f), "f"(f));
      asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(acc[i]), "f"(acc[i + 1]));
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(c), "l"(a));
      asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(d));
    }
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] *= f;
  }
}

// A finished 16-byte slice of Y row `row` (local): the owned rows, and -- peer-memory gather -- the
// same slice of every peer's Y_full, stored from the walk's epilogue (the transfer overlaps the
// rest of the walk; NVLink stores on a multi-GPU box).
#ifndef RGNN_PEER_STORES
#define RGNN_PEER_STORES 1  // 0: build without the fused peer stores (A/B of their cost on one GPU)
#endif
template <int N>
__device__ __forceinline__ void put_y(const AggArgs& a, int64_t row, int col, uint4 v) {
  stg16(a.Y + (size_t)row * N + col, v);
  if (RGNN_PEER_STORES)
    for (int p = 0; p < a.npeer; ++p) stg16(a.peer_y[p] + (size_t)(a.v0 + row) * N + col, v);
}
// writers into peer memory fence their stores before the kernel ends (the barrier that follows
// releases them to the peers)
__device__ __forceinline__ void peer_fence(const AggArgs& a) {
  if (a.npeer) __threadfence_system();
}

#ifndef RGNN_NARROW_EMPTY
#define RGNN_NARROW_EMPTY 1  // 1: the narrow pass writes the empty rows (Y = 0 / self term, lse = -inf); 0: k_empty_rows
                             // (measured r02: mag walk 1.83 -> 1.90 ms, AM 0.62 -> 0.67 ms with 0)
#endif
// Narrow rows (deg <= a.narrow, never split): one lane group (L lanes, one 16-byte slice of a
// Z row each) per row, G consecutive row ids per warp step, UN edges per group step and one
// online state per row -- no cross-group merge, so short rows cost a quarter (d = 64 bf16) or
// half (d = 128) of a warp instead of a whole warp plus a shuffle tree.  Rows are visited in id
// order, so empty rows (Y = 0, or the RGCN self term, lse = -inf) are written here too, with
// coalesced stores.  Which walk a row takes depends only on its degree: a dst-range shard walks
// every row exactly as one GPU does (pin P14).
// The three dependent loads of a row (row_ptr -> slot indices -> Z rows / s_src) are software
// pipelined across the warp's row groups: while row group i is reduced, the slot indices of
// group i+1 and the row bounds of group i+2 are already in flight.
template <typename T, int K, int N, bool RGAT>
__device__ __forceinline__ void narrow_rows_pipe(const AggArgs& a, int64_t warp0, int64_t nwarps, int lane) {
  using S = WalkShape<T, K, N>;
  constexpr int EPL = S::EPL, L = S::L, G = S::G, KPL = S::KPL;
  constexpr int UN = L < 4 ? L : 4;  // edges per group step
  const T* Z = static_cast<const T*>(a.Z);
  const T* X = static_cast<const T*>(a.X);
  const int g = lane / L, l = lane % L;
  const unsigned gmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (g * L));
  const int64_t ngroups = (a.V_own + G - 1) / G;
  // row bounds of this group's row in row group rg (q1 < q0 marks "no narrow row here")
  auto bounds = [&](int64_t rg, int& q0, int& q1) {
    const int64_t row = rg * G + g;
    q0 = 0; q1 = -1;
    if (rg < ngroups && row < a.V_own) {
      q0 = a.row_ptr[row]; q1 = a.row_ptr[row + 1];
      if (q1 - q0 > a.narrow) q1 = -1;  // a wide row: walked from the item list
    }
  };
  // slot indices of the first step (lanes l < UN): position / Z row, relation (RGAT) or 1/c (RGCN)
  auto slots = [&](int q0, int q1, int& p, int& r, float& sc) {
    const int q = q0 + l;
    const bool ok = l < UN && q < q1;
    p = ok ? a.pos[q] : 0;
    r = (RGAT && ok) ? a.et_slot[q] : 0;
    sc = RGAT ? 0.f : ((ok && a.slot_scale) ? a.slot_scale[q] : 1.f);
  };
  int q0c, q1c, q0n, q1n;  // current / next row group bounds
  bounds(warp0, q0c, q1c);
  bounds(warp0 + nwarps, q0n, q1n);
  int pc, rc;
  float sc_c;
  slots(q0c, q1c, pc, rc, sc_c);
  for (int64_t rg = warp0; rg < ngroups; rg += nwarps) {
    const int64_t row = rg * G + g;
    const int q0 = q0c, q1 = q1c;
    int myp = pc, myr = rc;
    float mys = sc_c;
    // stage C of this group: its first step's Z rows and source scores ...
    uint4 zr[UN];
    float sc[UN];
    int rr[UN];
    bool val[UN];
    float ssrc = 0.f;
    if constexpr (RGAT) ssrc = (l < UN && q0 + l < q1) ? a.s_src[myp] : 0.f;
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int p = __shfl_sync(gmask, myp, u, L);
      rr[u] = __shfl_sync(gmask, myr, u, L);
      val[u] = q0 + u < q1;
      zr[u] = val[u] ? ldg16(Z + (size_t)p * N + l * EPL) : make_uint4(0, 0, 0, 0);
    }
    // ... stage B of the next group (its slot indices) and stage A of the one after (its bounds)
    slots(q0n, q1n, pc, rc, sc_c);
    q0c = q0n; q1c = q1n;
    bounds(rg + 2 * nwarps, q0n, q1n);
    if (row >= a.V_own || q1 < q0) continue;  // no row, or a wide row (the whole group together)
    if (!RGNN_NARROW_EMPTY && q1 == q0) continue;  // empty rows: k_empty_rows
    if constexpr (RGAT) mys = ssrc;
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    float m = -CUDART_INF_F, lsum = 0.f;
    float xv[KPL];
    if constexpr (RGAT) {
      if (q1 > q0) load_slice<KPL>(X + (a.v0 + row) * (int64_t)K + l * KPL, xv);
    }
    for (int base = q0; base < q1; base += UN) {
      if (base > q0) {  // later steps of a row longer than UN: loads issued here
        const int q = base + l;
        const bool ok = l < UN && q < q1;
        myp = ok ? a.pos[q] : 0;
        if constexpr (RGAT) {
          myr = ok ? a.et_slot[q] : 0;
          mys = ok ? a.s_src[myp] : 0.f;
        } else {
          mys = (ok && a.slot_scale) ? a.slot_scale[q] : 1.f;
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int p = __shfl_sync(gmask, myp, u, L);
          rr[u] = __shfl_sync(gmask, myr, u, L);
          val[u] = base + u < q1;
          zr[u] = val[u] ? ldg16(Z + (size_t)p * N + l * EPL) : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) sc[u] = __shfl_sync(gmask, mys, u, L);
      if constexpr (RGAT) {
        float d[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) d[u] = dot_u<KPL>(xv, a.U + (size_t)rr[u] * K + l * KPL);
#pragma unroll
        for (int u = 0; u < UN; ++u) {
#pragma unroll
          for (int o = L / 2; o > 0; o >>= 1) d[u] += __shfl_xor_sync(gmask, d[u], o);
          sc[u] = val[u] ? leaky(sc[u] + d[u], a.slope) : -CUDART_INF_F;
        }
        float mnew = m;
#pragma unroll
        for (int u = 0; u < UN; ++u) mnew = fmaxf(mnew, sc[u]);
        const float corr = __expf(m - mnew);  // m = -inf -> 0 (mnew is finite: edge base is valid)
        lsum *= corr;
        mul_acc<EPL>(acc, corr);
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const float e = val[u] ? __expf(sc[u] - mnew) : 0.f;
          lsum += e;
          float zf[EPL];
          Vec16<T>{zr[u]}.to_float(zf);
          fma_acc<EPL>(acc, e, zf);
        }
        m = mnew;
      } else {
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          float zf[EPL];
          Vec16<T>{zr[u]}.to_float(zf);
          fma_acc<EPL>(acc, sc[u], zf);  // invalid slots: z = 0
        }
      }
    }
    if constexpr (RGAT) {
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] *= inv;
      if (l == 0) a.lse[row] = lsum > 0.f ? m + __logf(lsum) : -CUDART_INF_F;
    } else if (a.Z0) {
      float z0[EPL];
      Vec16<T>{ldg16(static_cast<const T*>(a.Z0) + (size_t)row * N + l * EPL)}.to_float(z0);
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] += z0[i];
    }
#pragma unroll
    for (int i = 0; i < EPL; i += 4)
      put_y<N>(a, row, l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]), __float_as_uint(acc[i + 2]),
                              __float_as_uint(acc[i + 3])));
  }
}

#ifndef RGNN_NARROW_UN
#define RGNN_NARROW_UN 4  // RGAT narrow walk: edges per lane-group step (8 measured slower: AM 0.59 -> 0.73 ms)
#endif
// The same walk without the cross-row-group pipeline (measured faster for RGAT, whose per-row
// x_dst slice and per-edge U dot make the pipelined version spill or lose a resident block:
// AM 0.354 vs 0.402 ms; RGCN gains from the pipeline: wikikg2 walk 1.00 -> 0.77 ms).
template <typename T, int K, int N, bool RGAT, bool USM = false>
__device__ __forceinline__ void narrow_rows(const AggArgs& a, int64_t warp0, int64_t nwarps, int lane,
                                            const float* Uw) {
  using S = WalkShape<T, K, N>;
  constexpr int EPL = S::EPL, L = S::L, G = S::G, KPL = S::KPL;
  constexpr int UN = L < RGNN_NARROW_UN ? L : RGNN_NARROW_UN;  // edges per group step
  const T* Z = static_cast<const T*>(a.Z);
  const T* X = static_cast<const T*>(a.X);
  const int g = lane / L, l = lane % L;
  const unsigned gmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (g * L));
  const int64_t ngroups = (a.V_own + G - 1) / G;
  // the next row group's bounds are loaded one iteration ahead (one dependent load off the chain)
  int nq0 = 0, nq1 = 0;
  if (warp0 * G + g < a.V_own) { nq0 = a.row_ptr[warp0 * G + g]; nq1 = a.row_ptr[warp0 * G + g + 1]; }
  for (int64_t rg = warp0; rg < ngroups; rg += nwarps) {
    const int64_t row = rg * G + g;
    const int q0 = nq0, q1 = nq1;
    const int64_t nrow = (rg + nwarps) * G + g;
    if (nrow < a.V_own) { nq0 = a.row_ptr[nrow]; nq1 = a.row_ptr[nrow + 1]; }
    if (row >= a.V_own) continue;  // the whole group leaves together
    if (q1 - q0 > a.narrow) continue;  // a wide row: walked from the item list
    if (!RGNN_NARROW_EMPTY && q1 == q0) continue;  // empty rows: k_empty_rows
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    float m = -CUDART_INF_F, lsum = 0.f;
    float xv[KPL];
    if constexpr (RGAT) {
      if (q1 > q0) load_slice<KPL>(X + (a.v0 + row) * (int64_t)K + l * KPL, xv);
    }
    for (int base = q0; base < q1; base += UN) {
      const int q = base + l;
      const bool ok = l < UN && q < q1;
      const int myp = ok ? a.pos[q] : 0;
      int myr = 0;
      float mys;
      if constexpr (RGAT) {
        myr = ok ? a.et_slot[q] : 0;
        mys = ok ? a.s_src[myp] : 0.f;
      } else {
        mys = (ok && a.slot_scale) ? a.slot_scale[q] : 1.f;
      }
      uint4 zr[UN];
      float sc[UN];
      int rr[UN];
      bool val[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) {  // all Z-row loads of the step first
        const int p = __shfl_sync(gmask, myp, u, L);
        rr[u] = __shfl_sync(gmask, myr, u, L);
        sc[u] = __shfl_sync(gmask, mys, u, L);
        val[u] = base + u < q1;
        zr[u] = val[u] ? ldg16(Z + (size_t)p * N + l * EPL) : make_uint4(0, 0, 0, 0);
      }
      if constexpr (RGAT) {
        float d[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) d[u] = dot_u<KPL, USM>(xv, Uw + (size_t)rr[u] * K + l * KPL);
#pragma unroll
        for (int u = 0; u < UN; ++u) {
#pragma unroll
          for (int o = L / 2; o > 0; o >>= 1) d[u] += __shfl_xor_sync(gmask, d[u], o);
          sc[u] = val[u] ? leaky(sc[u] + d[u], a.slope) : -CUDART_INF_F;
        }
        float mnew = m;
#pragma unroll
        for (int u = 0; u < UN; ++u) mnew = fmaxf(mnew, sc[u]);
        const float corr = __expf(m - mnew);
        lsum *= corr;
        mul_acc<EPL>(acc, corr);
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const float e = val[u] ? __expf(sc[u] - mnew) : 0.f;
          lsum += e;
          float zf[EPL];
          Vec16<T>{zr[u]}.to_float(zf);
          fma_acc<EPL>(acc, e, zf);
        }
        m = mnew;
      } else {
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          float zf[EPL];
          Vec16<T>{zr[u]}.to_float(zf);
          fma_acc<EPL>(acc, sc[u], zf);
        }
      }
    }
    if constexpr (RGAT) {
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] *= inv;
      if (l == 0) a.lse[row] = lsum > 0.f ? m + __logf(lsum) : -CUDART_INF_F;
    } else if (a.Z0) {
      float z0[EPL];
      Vec16<T>{ldg16(static_cast<const T*>(a.Z0) + (size_t)row * N + l * EPL)}.to_float(z0);
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] += z0[i];
    }
#pragma unroll
    for (int i = 0; i < EPL; i += 4)
      put_y<N>(a, row, l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]), __float_as_uint(acc[i + 2]),
                              __float_as_uint(acc[i + 3])));
  }
}

// resident blocks: RGAT 4 (64 registers, simple walk), RGCN 3 (80 registers, pipelined walk; 4
// spilled ~150 B at d = 64)
#ifndef RGNN_NARROW_MINB_RGAT
#define RGNN_NARROW_MINB_RGAT 4
#endif
// USM: the fused attention vectors U[r] (R x K fp32) staged in shared memory (dynamic, sized R*K*4 at launch)
#ifndef RGNN_WALK_USMEM
#define RGNN_WALK_USMEM 1  // measured r02: AM walk 0.618 -> 0.595 ms, ogbn-mag 1.815 -> 1.792 ms
#endif
template <typename T, int K, int N, bool RGAT, bool USM = false>
#ifndef RGNN_NARROW_MINB_RGCN
#define RGNN_NARROW_MINB_RGCN 4  // measured r02 end, wikikg2 walk: 3 / 4 / 5 / 6 blocks 0.861 / 0.783 / 0.829 / 0.832 ms
#endif
__global__ void __launch_bounds__(256, RGAT ? RGNN_NARROW_MINB_RGAT : RGNN_NARROW_MINB_RGCN) k_aggregate_narrow(AggArgs a) {
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  extern __shared__ float4 su4[];
  const float* Uw = a.U;
  if constexpr (RGAT && USM) {
    float* su = reinterpret_cast<float*>(su4);
    for (int i = threadIdx.x; i < a.R * K / 4; i += blockDim.x) su4[i] = __ldg(reinterpret_cast<const float4*>(a.U) + i);
    __syncthreads();
    Uw = su;
  }
  if constexpr (RGAT) narrow_rows<T, K, N, RGAT, USM>(a, w0, nw, threadIdx.x & 31, Uw);
  else narrow_rows_pipe<T, K, N, RGAT>(a, w0, nw, threadIdx.x & 31);
  peer_fence(a);
}

// 4 resident blocks (64 registers): measured r01 on ogbn-mag d=128, the walk is
// latency bound and 32 warps / SM beat 24 warps with fewer spills (1.85 vs 2.43 ms)
#ifndef RGNN_AGG_MINB
#define RGNN_AGG_MINB 4
#endif
#ifndef RGNN_AGG_MINB128
#define RGNN_AGG_MINB128 3  // d_out = 128 (measured r02 end: ogbn-mag wide walk 1.808 -> 1.768 ms with 3; at d_out = 64
                            // AM 0.594 -> 0.628 ms, so 4 stays there)
#endif
#ifndef RGNN_AGG_PREFETCH
#define RGNN_AGG_PREFETCH 1
#endif
#ifndef RGNN_RING
#define RGNN_RING 4  // cp.async ring depth of the RGCN walk (steps of Z rows in flight + 1)
#endif
template <typename T, int K, int N, bool RGAT, bool CACHE>
__global__ void __launch_bounds__(256, N >= 128 ? RGNN_AGG_MINB128 : RGNN_AGG_MINB) k_aggregate(AggArgs a) {
  using S = WalkShape<T, K, N>;
  constexpr int EPL = S::EPL, L = S::L, G = S::G, UNR = S::UNR, B = S::B, KPL = S::KPL;
  const T* Z = static_cast<const T*>(a.Z);
  const T* X = static_cast<const T*>(a.X);

  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  Item nit = warp0 < a.num_items ? a.items[warp0] : Item{0, 0, 0, -1};
  for (int64_t w = warp0; w < a.num_items; w += nwarps) {
    const Item it = nit;
    if (w + nwarps < a.num_items) nit = a.items[w + nwarps];  // next item's descriptor in flight
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    float m = -CUDART_INF_F, lsum = 0.f;
    float xv[KPL];
    int cr = -1;     // relation of the cached dst score (per lane group)
    float cd = 0.f;  // x_dst . U[cr]
    if constexpr (RGAT) {
      if (it.q1 > it.q0) load_slice<KPL>(X + (a.v0 + it.row) * (int64_t)K + l * KPL, xv);
    }
    // slot indices are loaded one step ahead of their use
    int nq = it.q0 + lane;
    bool nok = lane < B && nq < it.q1;
    int np = nok ? a.pos[nq] : 0;
    int nr = nok ? a.et_slot[nq] : 0;
    for (int base = it.q0; base < it.q1; base += B) {
      const bool ok = nok;
      const int myp = np;
      const int myr = nr;
      float mys = 0.f;
      if constexpr (RGAT) mys = ok ? a.s_src[myp] : 0.f;
      else mys = (ok && a.slot_scale) ? a.slot_scale[base + lane] : 1.f;  // compact RGCN: 1/c per slot
      nq = base + B + lane;
      nok = lane < B && nq < it.q1;
      np = nok ? a.pos[nq] : 0;
      nr = nok ? a.et_slot[nq] : 0;
      uint4 zr[UNR];
      float sc[UNR], ssv[UNR];
      int rr[UNR];
      bool val[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {  // all Z-row loads of the step first
        const int j = u * G + g;
        const int p = __shfl_sync(0xffffffffu, myp, j);
        rr[u] = __shfl_sync(0xffffffffu, myr, j);
        ssv[u] = __shfl_sync(0xffffffffu, mys, j);
        val[u] = base + j < it.q1;
        zr[u] = val[u] ? ldg16(Z + (size_t)p * N + l * EPL) : make_uint4(0, 0, 0, 0);
      }
#if RGNN_AGG_PREFETCH
      // L2 prefetch of the Z rows (and s_src) RGNN_AGG_PREFETCH steps ahead: no registers are
      // held for them (one 128-byte line per instruction)
      {
        int pq = np;
        bool pok = nok;
        if constexpr (RGNN_AGG_PREFETCH > 1) {
          const int q2 = base + RGNN_AGG_PREFETCH * B + lane;
          pok = lane < B && q2 < it.q1;
          pq = pok ? a.pos[q2] : 0;
        }
        if (pok) {
          const char* zp = reinterpret_cast<const char*>(Z + (size_t)pq * N);
#pragma unroll
          for (int o = 0; o < N * (int)sizeof(T); o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(zp + o));
          if constexpr (RGAT) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.s_src + pq));
        }
      }
#endif
      if constexpr (RGAT) dst_scores<K, L, KPL, UNR, CACHE>(xv, a.U, l, rr, ssv, cr, cd, sc);
      else {
#pragma unroll
        for (int u = 0; u < UNR; ++u) sc[u] = ssv[u];  // edge weight (1 when Z rows are pre-scaled)
      }
      if constexpr (RGAT) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) sc[u] = val[u] ? leaky(sc[u], a.slope) : -CUDART_INF_F;
        float mnew = m;
#pragma unroll
        for (int u = 0; u < UNR; ++u) mnew = fmaxf(mnew, sc[u]);
        if (mnew != -CUDART_INF_F) {
          const float corr = __expf(m - mnew);  // m = -inf -> 0
          lsum *= corr;
          mul_acc<EPL>(acc, corr);
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            const float e = val[u] ? __expf(sc[u] - mnew) : 0.f;
            lsum += e;
            float zf[EPL];
            Vec16<T>{zr[u]}.to_float(zf);
            fma_acc<EPL>(acc, e, zf);
          }
          m = mnew;
        }
      } else {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          float zf[EPL];
          Vec16<T>{zr[u]}.to_float(zf);
          fma_acc<EPL>(acc, sc[u], zf);  // fma(1, z, acc) == acc + z
        }
      }
    }
    // merge the G group states (fixed xor tree)
#pragma unroll
    for (int o = L; o < 32; o <<= 1) {
      if constexpr (RGAT) {
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
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      }
    }
    if (g == 0) {
      if (it.part < 0) {
            if constexpr (RGAT) {
          const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] *= inv;
          if (l == 0) a.lse[it.row] = lsum > 0.f ? m + __logf(lsum) : -CUDART_INF_F;
        } else if (a.Z0) {
          float z0[EPL];
          Vec16<T>{ldg16(static_cast<const T*>(a.Z0) + (size_t)it.row * N + l * EPL)}.to_float(z0);
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] += z0[i];
        }
#pragma unroll
        for (int i = 0; i < EPL; i += 4) put_y<N>(a, it.row, l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]),
                                                                 __float_as_uint(acc[i + 2]), __float_as_uint(acc[i + 3])));
      } else {
        float* pp = a.part + (size_t)it.part * (N + 4);
#pragma unroll
        for (int i = 0; i < EPL; i += 4) stg16(pp + l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]),
                                                                           __float_as_uint(acc[i + 2]), __float_as_uint(acc[i + 3])));
        if (l == 0) { pp[N] = m; pp[N + 1] = lsum; }
      }
    }
  }
  peer_fence(a);
}

// Same computation as k_aggregate with a per-warp cp.async ring: the Z-row
// slices (each lane copies exactly the 16-byte slices it will reduce) and the
// s_src of RING-1 steps ahead are in flight as asynchronous copies into shared
// memory -- no registers held -- while the current step is reduced.  The warp's
// items form one continuous stream of B-edge steps, so short rows do not drain
// the pipeline.  Results are bit-identical to k_aggregate (same per-group edge
// assignment, same arithmetic order).
// BULK: each Z row (N * sizeof(T) bytes, contiguous in the ring: lanes g*L .. g*L+L-1 of a (slot, u)
// entry hold one row) arrives by one 1-D TMA bulk copy issued by the edge's lane, completing on the slot's
// mbarrier (expect_tx = the step's row bytes), instead of L 16-byte cp.async per row: one instruction per
// row (tools/bulk_gather_bench.cu: random 256-byte rows at 6.9 TB/s, as many as register-held loads).
template <typename T, int K, int N, bool RGAT, int RING, bool CACHE, bool BULK = false>
#ifndef RGNN_RING_MINB
#define RGNN_RING_MINB 4  // measured r02 end, wikikg2: minimum 1 / 4 / 5 blocks 0.845 / 0.782 / 0.784 ms
#endif
__global__ void __launch_bounds__(256, RGNN_RING_MINB) k_aggregate_ring(AggArgs a) {
  using S = WalkShape<T, K, N>;
  constexpr int EPL = S::EPL, L = S::L, G = S::G, UNR = S::UNR, B = S::B, KPL = S::KPL;
  constexpr int ROWB = N * (int)sizeof(T);
  extern __shared__ uint4 ring_smem[];
  __shared__ uint64_t zbar[8][RING];  // BULK: per warp and slot
  const T* Z = static_cast<const T*>(a.Z);
  const T* X = static_cast<const T*>(a.X);
  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L, wib = threadIdx.x >> 5;
  uint4* zring = ring_smem + (size_t)wib * RING * UNR * 32;                          // [RING][UNR][32 lanes]
  float* sring = reinterpret_cast<float*>(ring_smem + (size_t)(blockDim.x >> 5) * RING * UNR * 32) +
                 (size_t)wib * RING * 32 * 2;                                          // [RING][32] s_src, [RING][32] r
  int* rring = reinterpret_cast<int*>(sring + RING * 32);
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  // producer cursor (RING-1 steps ahead of the consumer)
  int64_t pw = warp0;
  Item pit = pw < a.num_items ? a.items[pw] : Item{0, 0, 0, -1};
  int pbase = pit.q0;
  // (pos, et) of the producer's next step, one step ahead of its copies
  int np = 0, nr = 0;
  auto load_idx = [&]() {
    const int q = pbase + lane;
    const bool ok = pw < a.num_items && lane < B && q < pit.q1;
    np = ok ? a.pos[q] : 0;
    nr = ok ? a.et_slot[q] : 0;
  };
  auto advance_producer = [&]() {
    pbase += B;
    if (pbase >= pit.q1) {
      pw += nwarps;
      if (pw < a.num_items) { pit = a.items[pw]; pbase = pit.q0; }
    }
  };
  if constexpr (BULK) {
    if (lane < RING) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(
                                      &zbar[wib][lane])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  int pslot = 0;
  auto produce = [&]() {  // issue the copies of the producer's current step into ring slot pslot
    if (pw < a.num_items) {
      const int myp = np, myr = nr;
      const int q = pbase + lane;
      const bool ok = lane < B && q < pit.q1;
      if constexpr (BULK) {
        const int nvalid = min(B, pit.q1 - pbase);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the slot's generic reads before the refill
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(
                           &zbar[wib][pslot])), "r"(nvalid * ROWB)
                       : "memory");
        __syncwarp();
        if (ok) {  // lane j = u * G + g copies the row of edge j to entry (pslot, u), lanes g*L ..
          const int u = lane / G, gg = lane % G;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(zring + ((size_t)pslot * UNR + u) * 32 + gg * L)),
                       "l"(Z + (size_t)myp * N), "r"(ROWB), "r"((uint32_t)__cvta_generic_to_shared(&zbar[wib][pslot]))
                       : "memory");
        }
      } else {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int j = u * G + g;
          const int p = __shfl_sync(0xffffffffu, myp, j);
          if (pbase + j < pit.q1)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(
                             zring + ((size_t)pslot * UNR + u) * 32 + lane)),
                         "l"(Z + (size_t)p * N + l * EPL)
                         : "memory");
        }
      }
      if (ok && (RGAT || a.slot_scale))  // RGAT: s_src of the Z row; compact RGCN: 1/c of the slot
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(
                         sring + pslot * 32 + lane)),
                     "l"(RGAT ? a.s_src + myp : a.slot_scale + q)
                     : "memory");
      if (lane < B) rring[pslot * 32 + lane] = myr;
      advance_producer();
      load_idx();
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    pslot = pslot + 1 == RING ? 0 : pslot + 1;
  };

  load_idx();
#pragma unroll
  for (int i = 0; i < RING - 1; ++i) produce();

  int cslot = 0;
  uint32_t cuse = 0;  // BULK: steps consumed (mbarrier phase of the slot = (cuse / RING) & 1)
  for (int64_t w = warp0; w < a.num_items; w += nwarps) {
    const Item it = a.items[w];
    float acc[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) acc[i] = 0.f;
    float m = -CUDART_INF_F, lsum = 0.f;
    float xv[KPL];
    int cr = -1;
    float cd = 0.f;
    if constexpr (RGAT) load_slice<KPL>(X + (a.v0 + it.row) * (int64_t)K + l * KPL, xv);
    for (int base = it.q0; base < it.q1; base += B) {
      produce();  // keeps RING-1 steps in flight
      asm volatile("cp.async.wait_group %0;" ::"n"(RING - 1) : "memory");
      if constexpr (BULK) {
        uint32_t done = 0;
        const uint32_t ph = (cuse / RING) & 1;
        while (!done)
          asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done)
                       : "r"((uint32_t)__cvta_generic_to_shared(&zbar[wib][cslot])), "r"(ph)
                       : "memory");
        ++cuse;
      }
      __syncwarp();
      uint4 zr[UNR];
      float sc[UNR], ssv[UNR];
      int rr[UNR];
      bool val[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int j = u * G + g;
        val[u] = base + j < it.q1;
        zr[u] = val[u] ? zring[((size_t)cslot * UNR + u) * 32 + lane] : make_uint4(0, 0, 0, 0);
        if constexpr (RGAT) {
          rr[u] = rring[cslot * 32 + j];
          ssv[u] = sring[cslot * 32 + j];
        } else {
          sc[u] = (a.slot_scale && val[u]) ? sring[cslot * 32 + j] : 1.f;  // stale slots never multiply
        }
      }
      if constexpr (RGAT) dst_scores<K, L, KPL, UNR, CACHE>(xv, a.U, l, rr, ssv, cr, cd, sc);
      __syncwarp();  // the slot may be refilled by the next produce()
      cslot = cslot + 1 == RING ? 0 : cslot + 1;
      if constexpr (RGAT) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) sc[u] = val[u] ? leaky(sc[u], a.slope) : -CUDART_INF_F;
        float mnew = m;
#pragma unroll
        for (int u = 0; u < UNR; ++u) mnew = fmaxf(mnew, sc[u]);
        if (mnew != -CUDART_INF_F) {
          const float corr = __expf(m - mnew);
          lsum *= corr;
          mul_acc<EPL>(acc, corr);
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            const float e = val[u] ? __expf(sc[u] - mnew) : 0.f;
            lsum += e;
            float zf[EPL];
            Vec16<T>{zr[u]}.to_float(zf);
            fma_acc<EPL>(acc, e, zf);
          }
          m = mnew;
        }
      } else {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          float zf[EPL];
          Vec16<T>{zr[u]}.to_float(zf);
          fma_acc<EPL>(acc, sc[u], zf);  // fma(1, z, acc) == acc + z
        }
      }
    }
#pragma unroll
    for (int o = L; o < 32; o <<= 1) {
      if constexpr (RGAT) {
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
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      }
    }
    if (g == 0) {
      if (it.part < 0) {
            if constexpr (RGAT) {
          const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] *= inv;
          if (l == 0) a.lse[it.row] = lsum > 0.f ? m + __logf(lsum) : -CUDART_INF_F;
        } else if (a.Z0) {
          float z0[EPL];
          Vec16<T>{ldg16(static_cast<const T*>(a.Z0) + (size_t)it.row * N + l * EPL)}.to_float(z0);
#pragma unroll
          for (int i = 0; i < EPL; ++i) acc[i] += z0[i];
        }
#pragma unroll
        for (int i = 0; i < EPL; i += 4) put_y<N>(a, it.row, l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]),
                                                                 __float_as_uint(acc[i + 2]), __float_as_uint(acc[i + 3])));
      } else {
        float* pp = a.part + (size_t)it.part * (N + 4);
#pragma unroll
        for (int i = 0; i < EPL; i += 4) stg16(pp + l * EPL + i, make_uint4(__float_as_uint(acc[i]), __float_as_uint(acc[i + 1]),
                                                                           __float_as_uint(acc[i + 2]), __float_as_uint(acc[i + 3])));
        if (l == 0) { pp[N] = m; pp[N + 1] = lsum; }
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  peer_fence(a);
}

// Combine the partial states of each split row: one block per split row, warp w
// merges parts w, w+16, ... (4 per step), then warp 0 merges the 16 warp states
// in warp order.  Fixed assignment and order: deterministic.
template <typename T, int N, bool RGAT>
__global__ void __launch_bounds__(512) k_merge(AggArgs a) {
  constexpr int PER = (N + 31) / 32, NW = 16, U = 4;
  __shared__ float s_st[NW][N + 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const SplitRow sr = a.split_rows[blockIdx.x];
  float acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  float m = -CUDART_INF_F, lsum = 0.f;
  for (int k0 = warp; k0 < sr.nparts; k0 += NW * U) {
    float mk[U], lk[U], ak[U][PER];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * NW;
      const bool ok = k < sr.nparts;
      const float* pp = a.part + (size_t)(sr.part0 + (ok ? k : 0)) * (N + 4);
      mk[u] = ok && RGAT ? pp[N] : -CUDART_INF_F;
      lk[u] = ok && RGAT ? pp[N + 1] : 0.f;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int n = lane + 32 * i;
        ak[u][i] = (ok && n < N) ? pp[n] : 0.f;
      }
    }
    if constexpr (RGAT) {
      float mn = m;
#pragma unroll
      for (int u = 0; u < U; ++u) mn = fmaxf(mn, mk[u]);
      if (mn != -CUDART_INF_F) {
        const float c = __expf(m - mn);
        lsum *= c;
#pragma unroll
        for (int i = 0; i < PER; ++i) acc[i] *= c;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float cu = mk[u] == -CUDART_INF_F ? 0.f : __expf(mk[u] - mn);
          lsum = fmaf(lk[u], cu, lsum);
#pragma unroll
          for (int i = 0; i < PER; ++i) acc[i] = fmaf(ak[u][i], cu, acc[i]);
        }
        m = mn;
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < PER; ++i) acc[i] += ak[u][i];
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int n = lane + 32 * i;
    if (n < N) s_st[warp][n] = acc[i];
  }
  if (lane == 0) { s_st[warp][N] = m; s_st[warp][N + 1] = lsum; }
  __syncthreads();
  if (warp != 0) return;
  m = -CUDART_INF_F; lsum = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  for (int w = 0; w < NW; ++w) {
    if constexpr (RGAT) {
      const float mw = s_st[w][N], lw = s_st[w][N + 1];
      const float mn = fmaxf(m, mw);
      if (mn == -CUDART_INF_F) continue;
      const float c1 = __expf(m - mn), c2 = mw == -CUDART_INF_F ? 0.f : __expf(mw - mn);
      lsum = lsum * c1 + lw * c2;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int n = lane + 32 * i;
        if (n < N) acc[i] = acc[i] * c1 + s_st[w][n] * c2;
      }
      m = mn;
    } else {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int n = lane + 32 * i;
        if (n < N) acc[i] += s_st[w][n];
      }
    }
  }
  float* y = a.Y + (size_t)sr.row * N;
  if constexpr (RGAT) {
    const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
    if (lane == 0) a.lse[sr.row] = lsum > 0.f ? m + __logf(lsum) : -CUDART_INF_F;
#pragma unroll
    for (int i = 0; i < PER; ++i) acc[i] *= inv;
  } else if (a.Z0) {
    const T* z0 = static_cast<const T*>(a.Z0) + (size_t)sr.row * N;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int n = lane + 32 * i;
      if (n < N) acc[i] += to_f(z0[n]);
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int n = lane + 32 * i;
    if (n < N) {
      y[n] = acc[i];
      for (int p = 0; p < a.npeer; ++p) a.peer_y[p][(size_t)(a.v0 + sr.row) * N + n] = acc[i];
    }
  }
  peer_fence(a);
}

template <typename T, int K, int N>
__global__ void __launch_bounds__(256) k_bwd_rgat(BwdArgs a) {
  using S = WalkShape<T, K, N>;
  constexpr int EPL = S::EPL, L = S::L, G = S::G, UNR = S::UNR, B = S::B, KPL = S::KPL;
  const T* Z = static_cast<const T*>(a.Z);
  const T* X = static_cast<const T*>(a.X);
  T* dZ = static_cast<T*>(a.dZ);
  const int lane = threadIdx.x & 31, g = lane / L, l = lane % L;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp0; w < a.num_items; w += nwarps) {
    const Item it = a.items[w];
    if (it.q1 <= it.q0) continue;
    float gv[EPL], yv[EPL], xv[KPL];
    {
      const float* gp = a.dY + (size_t)it.row * N + l * EPL;
      const float* yp = a.Y + (size_t)it.row * N + l * EPL;
#pragma unroll
      for (int i = 0; i < EPL; ++i) { gv[i] = gp[i]; yv[i] = yp[i]; }
    }
    load_slice<KPL>(X + (a.v0 + it.row) * (int64_t)K + l * KPL, xv);
    float Sv = 0.f;
#pragma unroll
    for (int i = 0; i < EPL; ++i) Sv = fmaf(gv[i], yv[i], Sv);
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) Sv += __shfl_xor_sync(0xffffffffu, Sv, o);
    const float lse = a.lse[it.row];
    for (int base = it.q0; base < it.q1; base += B) {
      const int q = base + lane;
      const bool ok = lane < B && q < it.q1;
      const int myp = ok ? a.pos[q] : 0;
      const int myz = ok ? (a.zrow ? a.zrow[q] : myp) : 0;  // row of Z / s_src (compact: (etype, src) row)
      const int myr = ok ? a.et_slot[q] : 0;
      const float mys = ok ? a.s_src[myz] : 0.f;
      uint4 zr[UNR];
      float sc[UNR], da[UNR], sv[UNR];
      int pp[UNR], rr[UNR];
      bool val[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int j = u * G + g;
        pp[u] = __shfl_sync(0xffffffffu, myp, j);
        rr[u] = __shfl_sync(0xffffffffu, myr, j);
        const int zz = __shfl_sync(0xffffffffu, myz, j);
        const float ss = __shfl_sync(0xffffffffu, mys, j);
        val[u] = base + j < it.q1;
        zr[u] = val[u] ? ldg16(Z + (size_t)zz * N + l * EPL) : make_uint4(0, 0, 0, 0);
        sc[u] = dot_u<KPL>(xv, a.U + (size_t)rr[u] * K + l * KPL);
        sv[u] = ss;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        float zf[EPL];
        Vec16<T>{zr[u]}.to_float(zf);
        float d = 0.f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) d = fmaf(gv[i], zf[i], d);
        da[u] = d;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
          da[u] += __shfl_xor_sync(0xffffffffu, da[u], o);
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (!val[u]) continue;
        const float pre = sv[u] + sc[u];  // s_src + x_dst . U[r], as in the forward walk
        const float alpha = __expf(leaky(pre, a.slope) - lse);
        const float dpre = alpha * (da[u] - Sv) * (pre > 0.f ? 1.f : a.slope);
        const float* A0 = a.A + (size_t)rr[u] * 2 * N + l * EPL;
        float o[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) o[i] = fmaf(alpha, gv[i], dpre * __ldg(A0 + i));
        Vec16<T> v;
        v.from_float(o);
        stg16(dZ + (size_t)pp[u] * N + l * EPL, v.raw);
        if (l == 0) {
          a.dpre[pp[u]] = dpre;
          if (a.ad) a.ad[pp[u]] = make_float2(alpha, dpre);
        }
      }
    }
  }
}

// Rows without in-edges: Y_v = 0 (RGCN: the self-loop row X_v W0 if present), lse_v = -inf.
template <typename T, int N>
__global__ void __launch_bounds__(256) k_empty_rows(AggArgs a) {
  constexpr int NCH = N / 4;  // float4 chunks per Y row
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.num_empty * NCH;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / NCH;
    const int c = (int)(i - k * NCH);
    const int row = a.empty_rows[k];
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.Z0) {
      const T* z = static_cast<const T*>(a.Z0) + (size_t)row * N + c * 4;
      v = make_float4(to_f(z[0]), to_f(z[1]), to_f(z[2]), to_f(z[3]));
    }
    reinterpret_cast<float4*>(a.Y + (size_t)row * N)[c] = v;
    for (int p = 0; p < a.npeer; ++p) reinterpret_cast<float4*>(a.peer_y[p] + (size_t)(a.v0 + row) * N)[c] = v;
    if (a.lse && c == 0) a.lse[row] = -CUDART_INF_F;
  }
  peer_fence(a);
}

static unsigned warps_grid(int64_t items) {
  int64_t blocks = (items + 7) / 8;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 16));
}

template <typename T, int K, int N>
static rgnn_status aggregate(bool rgat, const AggArgs& a_in, cudaStream_t s) {
  AggArgs a = a_in;
  // narrow pass: only when a row group is narrower than the warp (G >= 2); it also writes the
  // empty rows, and the item walk then covers the wide rows only
  static const bool no_narrow = getenv("RGNN_NO_NARROW") != nullptr;
  const bool narrow = a.row_ptr && a.V_own > 0 && WalkShape<T, K, N>::G >= 2 && !no_narrow;
  if (narrow) {
    a.items = a.witems; a.num_items = a.num_witems;
    if (RGNN_NARROW_EMPTY) a.num_empty = 0;  // the narrow pass writes the empty rows too
  } else {
    a.row_ptr = nullptr;
  }
  constexpr int G = WalkShape<T, K, N>::G;
  if (narrow) {  // the narrow rows (and the empty ones) first, one lane group per row
    const size_t ub = (size_t)a.R * K * sizeof(float);
    const bool usm = RGNN_WALK_USMEM && rgat && a.R > 0 && ub <= 48 * 1024;
    auto kn = !rgat ? k_aggregate_narrow<T, K, N, false> : usm ? k_aggregate_narrow<T, K, N, true, true>
                                                               : k_aggregate_narrow<T, K, N, true>;
    RGNN_LAUNCH(kn, warps_grid((a.V_own + G - 1) / G), 256, usm ? ub : 0, s, a);
  }
  const int64_t work = a.num_items;
  if (a.num_empty > 0) {
    const int64_t n = a.num_empty * (N / 4);
    RGNN_LAUNCH((k_empty_rows<T, N>), (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s, a);
  }
  if (work > 0) {
    static const bool no_ring = getenv("RGNN_WALK_NO_RING") != nullptr;
    static const bool force_ring = getenv("RGNN_WALK_RING") != nullptr;
    // measured r01: with 4 resident blocks the plain walk wins for RGAT at every width (AM d=64
    // 0.805 vs 0.836 ms); the ring still wins for RGCN at d_out = 64 (wikikg2 1.00 vs 1.26 ms)
    const bool ring = !no_ring && ((N <= 64 && !rgat) || force_ring);
    if (ring) {
      constexpr int RING = RGNN_RING, UNR = WalkShape<T, K, N>::UNR;
      const size_t smem = 8 * (RING * UNR * 32 * sizeof(uint4) + RING * 32 * 2 * sizeof(float));
      static const bool bulk = getenv("RGNN_WALK_BULK") && atoi(getenv("RGNN_WALK_BULK")) != 0;
      auto kern = !rgat ? (bulk ? k_aggregate_ring<T, K, N, false, RING, false, true> : k_aggregate_ring<T, K, N, false, RING, false>)
                  : a.cache_dst ? (bulk ? k_aggregate_ring<T, K, N, true, RING, true, true> : k_aggregate_ring<T, K, N, true, RING, true>)
                                : (bulk ? k_aggregate_ring<T, K, N, true, RING, false, true> : k_aggregate_ring<T, K, N, true, RING, false>);
      RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      RGNN_LAUNCH(kern, warps_grid(work), 256, smem, s, a);
    } else {
      // (U in shared memory here as in the narrow walk measured slower: AM wide walk 0.173 -> 0.190 ms)
      auto kern = !rgat ? k_aggregate<T, K, N, false, false>
                  : a.cache_dst ? k_aggregate<T, K, N, true, true> : k_aggregate<T, K, N, true, false>;
      RGNN_LAUNCH(kern, warps_grid(work), 256, 0, s, a);
    }
  }
  if (a.num_split_rows > 0) {
    if (rgat) RGNN_LAUNCH((k_merge<T, N, true>), (unsigned)a.num_split_rows, 512, 0, s, a);
    else RGNN_LAUNCH((k_merge<T, N, false>), (unsigned)a.num_split_rows, 512, 0, s, a);
  }
  return RGNN_OK;
}

rgnn_status launch_aggregate(int prec, int K, int N, bool rgat, const AggArgs& a, cudaStream_t s) {
  return RGNN_DISPATCH_KN(K, N, [&] {
    return prec == RGNN_BF16 ? aggregate<__nv_bfloat16, kK, kN>(rgat, a, s) : aggregate<float, kK, kN>(rgat, a, s);
  });
}

template <typename T, int K, int N>
static rgnn_status bwd(const BwdArgs& a, cudaStream_t s) {
  if (a.num_items > 0) RGNN_LAUNCH((k_bwd_rgat<T, K, N>), warps_grid(a.num_items), 256, 0, s, a);
  return RGNN_OK;
}

rgnn_status launch_bwd_traverse(int prec, int K, int N, const BwdArgs& a, cudaStream_t s) {
  return RGNN_DISPATCH_KN(K, N, [&] {
    return prec == RGNN_BF16 ? bwd<__nv_bfloat16, kK, kN>(a, s) : bwd<float, kK, kN>(a, s);
  });
}

}  // namespace rgnn
