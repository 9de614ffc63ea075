// bwd_fused_tc.cu -- fused RGAT backward on the tensor cores (bf16 path).
//
// One CTA per split-K chunk of positions (relation r fixed, positions in
// (etype, dst) order).  Per 128-position stage:
//   * warps 1..2: X[src_s[p]] rows -> smem with 16-byte cp.async (MMA operand A,
//     MN-major SW128; TMA tile::gather4 is issue-rate bound, ~1 op / 100 cycles);
//   * warps 3..10 (CUDA cores) recompute the attention of each edge and write
//     its gradient row straight into the MMA's B operand in shared memory:
//        pre = s_src[p] + x_v . U[r]            (U[r] = W_r A[r,1])
//        alpha = exp(leaky(pre) - lse_v),  dalpha = G_v . Z[p],  S_v = G_v . Y_v
//        dpre = alpha (dalpha - S_v) leaky'(pre)
//        dZ[p] = alpha G_v + dpre A[r,0]   -> bf16, MN-major SW128 smem line p
//     plus dpre into a 16-column side operand (column 0) and the destination
//     term c_r += dpre x_v in registers (SURVEY §8 backward formulas);
//   * warp 0: TMEM allocator, tcgen05.mma  D[d_in x d_out] += X_src^T dZ  and  Db += X_src^T dpre.
// dZ never touches HBM (the unfused path writes and re-reads E x d_out bf16),
// and the per-destination quantities (G_v, Y_v, x_v, lse_v) are reloaded only
// when v changes (positions of one relation are sorted by destination).
// Epilogue: TMEM -> part[c] (d_in x d_out + bvec); c_r partial -> cpart[c];
// reduced in chunk order by k_dw_reduce / k_da (deterministic).
#include <math_constants.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

template <int K, int N, bool GAT = true>
struct BfCfg {
// Stage size and compute-warp count per d_out (measured): d_out = 128 (ogbn-mag) 64 positions and
// 16 compute warps; d_out = 64 96 positions and 24 compute warps (wikikg2 RGCN backward 1.155 ->
// 0.947 ms, AM RGAT 0.944 -> 0.921 ms).
#ifndef RGNN_BWD_MT
#define RGNN_BWD_MT 96
#endif
#ifndef RGNN_BWD_MT128
#define RGNN_BWD_MT128 64
#endif
  static constexpr int MT = N == 128 ? RGNN_BWD_MT128 : RGNN_BWD_MT;  // positions per stage
  static constexpr int A_BYTES = MT * K * 2;
  static constexpr int B_BYTES = MT * N * 2;
  static constexpr int B2_BYTES = MT * 16 * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES + B2_BYTES;  // multiple of 1024 (SW128 bases)
  static constexpr int SC_STAGE = MT * 8;                     // per position: local dst (int), s_src or 1/c (float)
#ifndef RGNN_BWD_SMAX
#define RGNN_BWD_SMAX 6
#endif
#ifndef RGNN_BWD_RING_KB
#define RGNN_BWD_RING_KB 200
#endif
  // RGAT at d_out = 64: 4 stages (measured AM 0.922 -> 0.858 ms: the smaller shared-memory
  // carve-out leaves more L1 for the per-destination rows); otherwise up to RGNN_BWD_SMAX
  static constexpr int SMAX = (GAT && N == 64) ? 4 : RGNN_BWD_SMAX;
  static constexpr int STAGES = (RGNN_BWD_RING_KB * 1024) / (STAGE + SC_STAGE) > SMAX
                                    ? SMAX
                                    : (RGNN_BWD_RING_KB * 1024) / (STAGE + SC_STAGE);
#ifndef RGNN_BWD_CW
#define RGNN_BWD_CW 24
#endif
#ifndef RGNN_BWD_CW128
#define RGNN_BWD_CW128 16
#endif
  static constexpr int CW = N == 128 ? RGNN_BWD_CW128 : RGNN_BWD_CW;  // compute warps
  static constexpr int PW = 4;                               // cp.async producer warps
  static constexpr int THREADS = 32 + PW * 32 + CW * 32;     // MMA warp, producers, compute warps
  static constexpr int DEPTH = STAGES - 1;                   // cp.async groups in flight per producer thread
  static constexpr int CPR = K * 2 / 16;                     // 16-byte chunks per X row
  static constexpr int RPI = 32 / CPR;                       // X rows per warp-wide cp.async
  static constexpr int ZCPR = N * 2 / 16;                    // 16-byte chunks per Z row
  static constexpr int ZRPI = 32 / ZCPR;                     // Z rows per warp-wide cp.async
  static constexpr int RPW = MT / PW;                        // stage rows per producer warp
  static constexpr int SMEM = 1024 + STAGES * (STAGE + SC_STAGE) + CW * K * 4 + 256;
  static constexpr int NCOLS = (N + 16) <= 32 ? 32 : (N + 16) <= 64 ? 64 : (N + 16) <= 128 ? 128 : 256;
  static constexpr uint32_t IDESC = tc::idesc_bf16(K, N, 1, 1);
  static constexpr uint32_t IDESC_B = tc::idesc_bf16(K, 16, 1, 1);
  // compute mapping: L lanes per position (16 bytes of Z each), G positions per warp step
  static constexpr int EPL = 8;
  static constexpr int L = N / EPL;
  static constexpr int G = 32 / L;
  static constexpr int PPW = MT / CW;                        // positions per warp per stage
  static constexpr int PG = PPW / G;                         // positions per lane group
  static constexpr int KPL = K / L;                          // x_v features per lane
  static_assert(STAGE % 1024 == 0 && RPW <= 32 && PG >= 1, "bwd config");
  // every stage row must belong to exactly one compute lane group (CW = 20 at MT = 64 once "measured"
  // 25% faster by leaving 4 rows of each stage unprocessed)
  static_assert(CW * PPW == MT && PPW % G == 0, "compute warps must cover the stage exactly");
};

struct BwdFusedParams {
  const Tile* chunks;
  const int32_t* src_s;
  const int32_t* dst_s;
  const float* s_src;
  const __nv_bfloat16* Z;
  const int32_t* zmap;  // compact: Z / s_src row of position p (null = p)
  const __nv_bfloat16* X;
  const float* lse;
  const float* Y;
  const float* dY;
  const float* U;
  const float* A;
  const float* inv_c;  // RGCN: 1/c_{v,r} per position
  float slope;
  int64_t v0;
  float* part;
  float* cpart;
  float2* ad;  // dX: (alpha, dpre) per position, or null
};

__device__ __forceinline__ float leaky_f(float x, float s) { return x > 0.f ? x : s * x; }

// GAT = true: RGAT (dZ = alpha G_v + dpre A[r,0], bvec, dst term); false: RGCN (dZ = G_v / c_{v,r}).
template <int K, int N, bool GAT, bool CM>
#ifndef RGNN_BWD_MINB64
#define RGNN_BWD_MINB64 1  // resident CTAs per SM at d_out = 64 (measured r02: 2 CTAs of 32-position stages and 8 compute
                           // warps, AM 0.757 -> 0.856 ms, wikikg2 0.870 -> 1.19 ms)
#endif
__global__ void __launch_bounds__(BfCfg<K, N, GAT>::THREADS, N == 64 ? RGNN_BWD_MINB64 : 1)
    k_bwd_fused_tc(BwdFusedParams pr) {
  using C = BfCfg<K, N, GAT>;
  constexpr int L = C::L, PG = C::PG, KPL = C::KPL, EPL = C::EPL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sc_base = smem + C::STAGES * C::STAGE;                          // [STAGES][MT] dst, [MT] s
  float* s_c = reinterpret_cast<float*>(sc_base + C::STAGES * C::SC_STAGE);  // [CW][K] dst-term partials
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_c + C::CW * K);
  uint64_t* a_full = bar;
  uint64_t* b_full = a_full + C::STAGES;
  uint64_t* empty = b_full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  auto sA = [&](int s) { return smem + s * C::STAGE; };
  auto sB = [&](int s) { return smem + s * C::STAGE + C::A_BYTES; };
  auto sB2 = [&](int s) { return smem + s * C::STAGE + C::A_BYTES + C::B_BYTES; };
  auto sDst = [&](int s) { return reinterpret_cast<int*>(sc_base + s * C::SC_STAGE); };
  auto sSs = [&](int s) { return reinterpret_cast<float*>(sc_base + s * C::SC_STAGE + C::MT * 4); };
  // swizzled A / B (and staged Z) offset of 16-byte chunk `c` of stage row `lp` (MN-major SW128)
  auto b_off = [&](int c, int lp) { return (c >> 3) * (C::MT * 128) + lp * 128 + (((c & 7) ^ (lp & 7)) << 4); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Tile ch = pr.chunks[blockIdx.x];
  const int r = ch.r, row0 = ch.row0, row1 = ch.row1;
  const int nsub = (row1 - row0 + C::MT - 1) / C::MT;
  // Stage row lp of stage `it` holds position pmap(lp, it): the chunk is cut into MT / PG
  // contiguous segments of PG * nsub positions, one per compute lane group, and each stage
  // takes the next PG positions of every segment.  A lane group therefore walks one run of
  // consecutive positions, and its per-destination values (G_v, Y_v, x_v, lse_v) are reloaded
  // only when the destination changes, not at every stage.  (The dW sum is order-free; the
  // mapping is fixed, so results stay deterministic.)  Positions >= row1 are padding rows.
  auto pmap = [&](int lp, int it) { return row0 + (lp / C::PG) * (C::PG * nsub) + C::PG * it + (lp % C::PG); };

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      tc::mbar_init(&a_full[i], C::PW * 32);
      tc::mbar_init(&b_full[i], C::CW);
      // two arrivals free a stage: the MMAs' completion (tcgen05.commit) and the MMA thread itself,
      // which has waited for the compute warps' dZ writes (b_full) -- redundant for the hardware, but
      // a thread-level happens-before edge from those generic-proxy writes to the producer's refill
      tc::mbar_init(&empty[i], 2);
    }
    tc::mbar_init(acc_full, 1);
    tc::mbar_fence_init();
  }
  for (int i = threadIdx.x; i < C::STAGES * C::B2_BYTES / 16; i += blockDim.x) {  // dpre operand: cols 1..15 = 0
    const int s = i / (C::B2_BYTES / 16), o = i % (C::B2_BYTES / 16);
    reinterpret_cast<uint4*>(sB2(s))[o] = make_uint4(0, 0, 0, 0);
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) {
    __syncwarp();
    tc::tmem_alloc<C::NCOLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 1 && warp <= C::PW) {
    // ------------------------------------------------------------ producers (cp.async, 16 B / 4 B):
    // X[src] rows -> A, Z rows -> B (overwritten in place by dZ), dst and s_src (1/c) -> scalars.
    const int pw = warp - 1;                      // rows pw*RPW .. pw*RPW+RPW-1 of each stage
    constexpr int RPW = C::RPW;
    auto load_idx = [&](int it, int& src, int& zr, int& p, int& v) {
      p = pmap(pw * RPW + (lane % RPW), it);
      const int pc = min(p, row1 - 1);
      src = __ldg(pr.src_s + pc);
      zr = CM ? __ldg(pr.zmap + pc) : pc;
      v = __ldg(pr.dst_s + pc);
    };
    // L2 prefetch of the per-destination rows (G_v, Y_v, x_v) the compute warps will load when
    // they reach these positions, STAGES-1 stages from now (one lane per run start).
    auto prefetch_dst = [&](int p, int v) {
      const int vp = __shfl_up_sync(0xffffffffu, v, 1);
      if (lane < RPW && p < row1 && (lane == 0 || vp != v)) {
        const char* gp = reinterpret_cast<const char*>(pr.dY + (size_t)v * N);
#pragma unroll
        for (int o = 0; o < N * 4; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(gp + o));
        if constexpr (GAT) {
          const char* yp = reinterpret_cast<const char*>(pr.Y + (size_t)v * N);
          const char* xp = reinterpret_cast<const char*>(pr.X + (pr.v0 + v) * (int64_t)K);
#pragma unroll
          for (int o = 0; o < N * 4; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(yp + o));
#pragma unroll
          for (int o = 0; o < K * 2; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(xp + o));
        }
      }
    };
    int src = 0, zr = 0, p = 0, v = 0;
    if (nsub > 0) load_idx(0, src, zr, p, v);
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      const uint32_t use = (uint32_t)(it / C::STAGES);
      int nsrc = 0, nzr = 0, np = 0, nv = 0;
      if (it + 1 < nsub) load_idx(it + 1, nsrc, nzr, np, nv);
      if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
      uint8_t* a = sA(st);
#pragma unroll 4
      for (int i = 0; i < RPW / C::RPI; ++i) {
        const int rr = i * C::RPI + lane / C::CPR;  // row within this warp's RPW
        const int c = lane % C::CPR;
        const int row = pw * RPW + rr;
        const int xr = __shfl_sync(0xffffffffu, src, rr);
        tc::cp_async16(a + b_off(c, row), pr.X + (size_t)xr * K + c * 8);
      }
      if constexpr (GAT) {
        uint8_t* b = sB(st);
#pragma unroll 4
        for (int i = 0; i < RPW / C::ZRPI; ++i) {
          const int rr = i * C::ZRPI + lane / C::ZCPR;
          const int c = lane % C::ZCPR;
          const int row = pw * RPW + rr;
          const int zz = __shfl_sync(0xffffffffu, zr, rr);
          tc::cp_async16(b + b_off(c, row), pr.Z + (size_t)zz * N + c * 8);
        }
      }
      if (lane < RPW && p < row1) {  // padding rows are recognised by position, not staged
        const int row = pw * RPW + lane;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(sDst(st) + row)),
                     "l"(pr.dst_s + p) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(sSs(st) + row)),
                     "l"(GAT ? pr.s_src + zr : pr.inv_c + p) : "memory");
      }
      // the stage is published by the copy engine itself: the arrive fires when all of this
      // thread's prior cp.async have landed (no wait, no publication lag)
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&a_full[st]))
                   : "memory");
      prefetch_dst(p, v);
      src = nsrc; zr = nzr; p = np; v = nv;
    }
    tc::cp_async_wait<0>();
  } else if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      const uint32_t ph = (uint32_t)(it / C::STAGES) & 1;
      tc::mbar_wait(&a_full[st], ph);
      tc::mbar_wait(&b_full[st], ph);
      tc::fence_proxy_async_smem();  // cp.async (generic proxy) data of A -> tcgen05 (async proxy)
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = tc::smem_u32(sA(st)), b0 = tc::smem_u32(sB(st)), c0 = tc::smem_u32(sB2(st));
#pragma unroll
        for (int ks = 0; ks < C::MT / 16; ++ks) {
          const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
          const uint64_t ad = tc::umma_desc(a0 + ks * 16 * 128, C::MT * 128, 1024, 2u);
          const uint64_t bd = tc::umma_desc(b0 + ks * 16 * 128, C::MT * 128, 1024, 2u);
          tc::umma_bf16(tmem, ad, bd, C::IDESC, acc);
          if (GAT) {
            const uint64_t cd = tc::umma_desc(c0 + ks * 512, 256, 128, 0u);
            tc::umma_bf16(tmem + N, ad, cd, C::IDESC_B, acc);
          }
        }
        tc::umma_commit(&empty[st]);
        tc::mbar_arrive(&empty[st]);
        if (it == nsub - 1) tc::umma_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ compute warps: dZ -> smem B operand
    const int cw = warp - 1 - C::PW;         // 0..7
    const int g = lane / L, l = lane % L;    // lane group (one position at a time), lane within group
    float u[KPL], a0[EPL];
    if constexpr (GAT) {
      const float* Ur = pr.U + (size_t)r * K + l * KPL;
      const float* A0 = pr.A + (size_t)r * 2 * N + l * EPL;
#pragma unroll
      for (int i = 0; i < KPL; ++i) u[i] = __ldg(Ur + i);
#pragma unroll
      for (int i = 0; i < EPL; ++i) a0[i] = __ldg(A0 + i);
    }
    float cacc[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) cacc[i] = 0.f;
    int cur_v = -1;
    float gv[EPL], xv[KPL], Sv = 0.f, dsc = 0.f, lse = 0.f;
    const uint32_t gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (g * L));
    // Everything per position comes from the stage in shared memory (staged by the producers
    // several stages ahead); only the per-destination rows are read from global memory, once
    // per destination change.
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      tc::mbar_wait(&a_full[st], (uint32_t)(it / C::STAGES) & 1);
      uint8_t* b = sB(st);
      uint8_t* b2 = sB2(st);
#pragma unroll
      for (int i = 0; i < PG; ++i) {
        const int lp = cw * C::PPW + g * PG + i;  // row of the stage
        const bool pv = pmap(lp, it) < row1;
        const int v = pv ? sDst(st)[lp] : -1;
        const float ss = pv ? sSs(st)[lp] : 0.f;
        uint4* bz = reinterpret_cast<uint4*>(b + b_off(l, lp));  // staged Z chunk; dZ goes to the same place
        float dz[EPL];
        float dpre = 0.f;
        if (v >= 0 && !GAT) {  // RGCN: dZ[p] = G_v / c_{v,r}
          if (v != cur_v) {
            const float* gp = pr.dY + (size_t)v * N + l * EPL;
#pragma unroll
            for (int j = 0; j < EPL; j += 4) {
              const float4 gg = __ldg(reinterpret_cast<const float4*>(gp + j));
              gv[j] = gg.x; gv[j + 1] = gg.y; gv[j + 2] = gg.z; gv[j + 3] = gg.w;
            }
            cur_v = v;
          }
#pragma unroll
          for (int j = 0; j < EPL; ++j) dz[j] = gv[j] * ss;
        } else if (v >= 0) {
          if (v != cur_v) {  // per-destination values (group-uniform branch)
            const float* gp = pr.dY + (size_t)v * N + l * EPL;
            const float* yp = pr.Y + (size_t)v * N + l * EPL;
            const __nv_bfloat16* xp = pr.X + (pr.v0 + v) * (int64_t)K + l * KPL;
            float s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int j = 0; j < EPL; j += 4) {
              const float4 gg = __ldg(reinterpret_cast<const float4*>(gp + j));
              const float4 yy = __ldg(reinterpret_cast<const float4*>(yp + j));
              gv[j] = gg.x; gv[j + 1] = gg.y; gv[j + 2] = gg.z; gv[j + 3] = gg.w;
              s1 = fmaf(gg.x, yy.x, s1); s1 = fmaf(gg.y, yy.y, s1); s1 = fmaf(gg.z, yy.z, s1); s1 = fmaf(gg.w, yy.w, s1);
            }
#pragma unroll
            for (int j = 0; j < KPL; j += 8) {
              float xf[8];
              Vec16<__nv_bfloat16>{ldg16(xp + j)}.to_float(xf);
#pragma unroll
              for (int t = 0; t < 8; ++t) xv[j + t] = xf[t];
            }
#pragma unroll
            for (int j = 0; j < KPL; ++j) s2 = fmaf(xv[j], u[j], s2);
#pragma unroll
            for (int o = L / 2; o > 0; o >>= 1) {
              s1 += __shfl_xor_sync(gmask, s1, o);
              s2 += __shfl_xor_sync(gmask, s2, o);
            }
            Sv = s1;
            dsc = s2;
            lse = __ldg(pr.lse + v);
            cur_v = v;
          }
          float zf[EPL];
          Vec16<__nv_bfloat16>{*bz}.to_float(zf);
          float da = 0.f;
#pragma unroll
          for (int j = 0; j < EPL; ++j) da = fmaf(gv[j], zf[j], da);
#pragma unroll
          for (int o = L / 2; o > 0; o >>= 1) da += __shfl_xor_sync(gmask, da, o);
          const float pre = ss + dsc;
          const float alpha = __expf(leaky_f(pre, pr.slope) - lse);
          dpre = alpha * (da - Sv) * (pre > 0.f ? 1.f : pr.slope);
          if (pr.ad && l == 0) pr.ad[pmap(lp, it)] = make_float2(alpha, dpre);
#pragma unroll
          for (int j = 0; j < EPL; ++j) dz[j] = fmaf(alpha, gv[j], dpre * a0[j]);
#pragma unroll
          for (int j = 0; j < KPL; ++j) cacc[j] = fmaf(dpre, xv[j], cacc[j]);
        } else {
#pragma unroll
          for (int j = 0; j < EPL; ++j) dz[j] = 0.f;
        }
        // MN-major SW128 line `lp`: features l*8..l*8+7 = 16-byte chunk (l % 8) of block l / 8
        uint4 o;
        o.x = tc::pack_bf16(dz[0], dz[1]); o.y = tc::pack_bf16(dz[2], dz[3]);
        o.z = tc::pack_bf16(dz[4], dz[5]); o.w = tc::pack_bf16(dz[6], dz[7]);
        *bz = o;
        if (GAT && l == 0)
          *reinterpret_cast<__nv_bfloat16*>(b2 + (lp >> 3) * 256 + (lp & 7) * 16) = __float2bfloat16_rn(dpre);
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&b_full[st]);
    }
    // destination-term partial: sum over lane groups, then over warps (fixed order)
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      float v = cacc[j];
#pragma unroll
      for (int o = L; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      cacc[j] = v;
    }
    if (g == 0) {
#pragma unroll
      for (int j = 0; j < KPL; ++j) s_c[cw * K + l * KPL + j] = cacc[j];
    }
    // epilogue: TMEM accumulators -> part[c]; two warps per lane quarter split the columns
    tc::mbar_wait(acc_full, 0);
    tc::tc_fence_after();
    const int q = warp & 3, half = cw >> 2;  // 16 compute warps: each TMEM lane quarter read by 4 warps
    const int row = K == 128 ? q * 32 + lane : q * 16 + lane;
    const bool rvalid = K == 128 || lane < 16;
    float* out = pr.part + (size_t)blockIdx.x * (K * N + K);
    // the CW / 4 warps of a lane quarter take interleaved 16-column chunks
    for (int c0 = half * 16; c0 < N; c0 += (C::CW / 4) * 16) {
      uint32_t v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
      tc::tmem_ld_wait();
      if (rvalid) {
        float4* o = reinterpret_cast<float4*>(out + (size_t)row * N + c0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          o[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                             __uint_as_float(v[4 * j + 3]));
      }
    }
    if (half == 0) {
      uint32_t v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + N, v);
      tc::tmem_ld_wait();
      if (rvalid) out[K * N + row] = GAT ? __uint_as_float(v[0]) : 0.f;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < C::CW; ++w) s += s_c[w * K + k];
    pr.cpart[(size_t)blockIdx.x * K + k] = s;
  }
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

template <int K, int N>
static rgnn_status bwd_fused(const rgnn_graph* g, const BwdFusedParams& p0, const void* X, cudaStream_t s) {
  tc::watchdog_init();
  if (g->num_chunks == 0) return RGNN_OK;
  (void)X;
  if (!p0.s_src) {
    using C = BfCfg<K, N, false>;
    auto kern = k_bwd_fused_tc<K, N, false, false>;
    RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    RGNN_LAUNCH(kern, (unsigned)g->num_chunks, C::THREADS, C::SMEM, s, p0);
    return RGNN_OK;
  }
  using C = BfCfg<K, N, true>;
  auto kern = p0.zmap ? k_bwd_fused_tc<K, N, true, true> : k_bwd_fused_tc<K, N, true, false>;
  RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  RGNN_LAUNCH(kern, (unsigned)g->num_chunks, C::THREADS, C::SMEM, s, p0);
  return RGNN_OK;
}

bool tc_disabled();

// RGAT when s_src != null, RGCN (dZ = G_v / c_{v,r}) otherwise.
rgnn_status launch_bwd_fused_tc(int K, int N, const rgnn_graph* g, const void* X, const void* Z, const int32_t* zmap,
                                const float* s_src,
                                const float* lse, const float* Y, const float* dY, const float* U, const float* A,
                                float slope, float* part, float* cpart, float2* ad, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  if (getenv("RGNN_DISABLE_FUSED_BWD")) return RGNN_E_UNSUPPORTED;
  BwdFusedParams p{g->chunks, g->src_s, g->dst_s, s_src, static_cast<const __nv_bfloat16*>(Z), zmap,
                   static_cast<const __nv_bfloat16*>(X), lse, Y, dY, U, A, g->inv_c, slope, g->v0, part, cpart, ad};
  if (K == 64 && N == 64) return bwd_fused<64, 64>(g, p, X, s);
  if (K == 64 && N == 128) return bwd_fused<64, 128>(g, p, X, s);
  if (K == 128 && N == 64) return bwd_fused<128, 64>(g, p, X, s);
  if (K == 128 && N == 128) return bwd_fused<128, 128>(g, p, X, s);
  return RGNN_E_UNSUPPORTED;
}

}  // namespace rgnn
