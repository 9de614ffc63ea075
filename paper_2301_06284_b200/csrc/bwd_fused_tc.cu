// bwd_fused_tc.cu -- fused backward on the tensor cores (bf16 path).
//
// One CTA per split-K chunk of positions (one relation r, positions in
// (etype, dst) order).  Per 128-position stage:
//   * warps 1..2 gather X[src_s[p]] rows with 16-byte cp.async into shared
//     memory (128B-swizzled lines, one per position);
//   * RGAT: warp 0 recomputes the messages on the tensor cores,
//       Z_tile = X_tile . W_r                 (tcgen05, K-major view of the tile)
//     into one of two TMEM buffers -- the same smem bytes are the MN-major A
//     operand of the dW MMA below, so Z never has to come from HBM (NEXT-4:
//     the unfused design re-reads E x d_out bf16 Z, 5.4 GB on ogbn-mag);
//   * warps 3..18 (CUDA cores) drain Z into the stage's B operand (bf16,
//     MN-major SW128) and then, per edge, in place:
//        pre = s_src[p] + x_v . U[r]          (U[r] = W_r A[r,1])
//        alpha = exp(leaky(pre) - lse_v),  dalpha = G_v . z_p,  S_v = G_v . Y_v
//        dpre = alpha (dalpha - S_v) leaky'(pre)
//        dZ[p] = alpha G_v + dpre A[r,0]                          (RGAT)
//        dZ[p] = G_v / c_{v,r}                                    (RGCN)
//     accumulating dA[r,0] += dpre z_p and c_r += dpre x_v in registers;
//     per-destination values (G_v, Y_v, x_v, lse_v) are reloaded only when v
//     changes (positions of one relation are sorted by destination);
//   * warp 0: D[d_in x d_out] += X_src^T dZ   (tcgen05, MN-major operands).
// Epilogue: TMEM -> part[c] (d_in x d_out); c_r -> cpart[c]; sum dpre z -> apart[c];
// reduced in chunk order by k_dw_reduce / k_da (deterministic).
#include <math_constants.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

template <int K, int N, bool GAT>
struct BfCfg {
  static constexpr int MT = 128;                             // positions per stage
  static constexpr int A_BYTES = MT * K * 2;                 // X_src rows
  static constexpr int B_BYTES = MT * N * 2;                 // Z, then dZ, in place
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int W_BYTES = GAT ? N * K * 2 : 0;        // W_r^T (K-major B of the Z MMA)
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int ST_FIT = (SMEM_MAX - 1024 - 256 - W_BYTES) / STAGE;
  static constexpr int STAGES = ST_FIT > 6 ? 6 : ST_FIT;
  static_assert(STAGES >= 3, "the Z lookahead needs three stages");
  static constexpr int DEPTH = STAGES - 2;                   // cp.async stages in flight before publishing
  static constexpr int CW = 16;                              // compute warps
  static constexpr int PW = 2;                               // cp.async producer warps
  static constexpr int THREADS = 32 + PW * 32 + CW * 32;
  static constexpr int CPR = K * 2 / 16;                     // 16-byte chunks per X row
  static constexpr int RPI = 32 / CPR;                       // X rows per warp-wide cp.async
  static constexpr int SMEM = 1024 + STAGES * STAGE + W_BYTES + 256;
  static constexpr int ZCOL = N;                             // Z accumulators at [N, 3N)
  static constexpr int TCOLS = GAT ? 3 * N : N;
  static constexpr int NCOLS = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC_DW = tc::idesc_bf16(K, N, 1, 1);   // M = d_in, both MN-major
  static constexpr uint32_t IDESC_Z = tc::idesc_bf16(128, N, 0, 0);  // M = positions, both K-major
  // compute mapping: L lanes per position (16 bytes of a Z / dZ row each), G positions per warp step
  static constexpr int EPL = 8;
  static constexpr int L = N / EPL;
  static constexpr int G = 32 / L;
  static constexpr int PPW = MT / CW;                        // positions per warp per stage (8)
  static constexpr int PG = PPW / G;                         // positions per lane group
  static constexpr int KPL = K / L;                          // x_v features per lane
  static_assert(CW * K * 4 + CW * N * 4 <= STAGE, "epilogue scratch aliases stage 0");
};

struct BwdFusedParams {
  const Tile* chunks;
  const int32_t* src_s;
  const int32_t* dst_s;
  const float* s_src;
  const __nv_bfloat16* X;
  const float* W;      // fp32 master [R, K, N] (RGAT: rounded to bf16 into smem)
  const float* lse;
  const float* Y;
  const float* dY;
  const float* U;
  const float* A;
  const float* inv_c;  // RGCN: 1/c_{v,r} per position
  float slope;
  int64_t v0;
  float* part;         // [chunks, K*N + K]
  float* cpart;        // [chunks, K]   c_r partials
  float* apart;        // [chunks, N]   sum dpre z partials (dA[r,0])
};

__device__ __forceinline__ float leaky_f(float x, float s) { return x > 0.f ? x : s * x; }

// byte offset of 16-byte chunk `c` (features 8c..8c+7) of line `row` in a 128B-swizzled
// tile of `mt` lines (feature blocks of 64 at mt*128 bytes)
__device__ __forceinline__ int sw_off(int row, int c, int mt) {
  return (c >> 3) * (mt * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4);
}

// GAT = true: RGAT (dZ = alpha G_v + dpre A[r,0], dA, dst term, Z recomputed); false: RGCN.
template <int K, int N, bool GAT>
__global__ void __launch_bounds__(BfCfg<K, N, GAT>::THREADS, 1) k_bwd_fused_tc(BwdFusedParams pr) {
  using C = BfCfg<K, N, GAT>;
  constexpr int L = C::L, PG = C::PG, KPL = C::KPL, EPL = C::EPL, MT = C::MT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem + C::STAGES * C::STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sW + C::W_BYTES);
  uint64_t* a_full = bar;
  uint64_t* b_full = a_full + C::STAGES;
  uint64_t* empty = b_full + C::STAGES;
  uint64_t* z_full = empty + C::STAGES;
  uint64_t* z_free = z_full + 2;
  uint64_t* acc_full = z_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  auto sA = [&](int s) { return smem + s * C::STAGE; };
  auto sB = [&](int s) { return smem + s * C::STAGE + C::A_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Tile ch = pr.chunks[blockIdx.x];
  const int r = ch.r, row0 = ch.row0, row1 = ch.row1;
  const int nsub = (row1 - row0 + MT - 1) / MT;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      tc::mbar_init(&a_full[i], C::PW * 32);
      tc::mbar_init(&b_full[i], C::CW);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(&z_full[i], 1); tc::mbar_init(&z_free[i], C::CW); }
    tc::mbar_init(acc_full, 1);
    tc::mbar_fence_init();
  }
  if constexpr (GAT) {  // W_r^T as a K-major SW128 operand: line n (output feature), features k (bf16 RNE)
    const float* Wr = pr.W + (size_t)r * K * N;
    for (int i = threadIdx.x; i < N * (K / 8); i += blockDim.x) {
      const int n = i / (K / 8), c = i % (K / 8);
      float w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = __ldg(Wr + (size_t)(c * 8 + j) * N + n);
      uint4 o;
      o.x = tc::pack_bf16(w[0], w[1]); o.y = tc::pack_bf16(w[2], w[3]);
      o.z = tc::pack_bf16(w[4], w[5]); o.w = tc::pack_bf16(w[6], w[7]);
      *reinterpret_cast<uint4*>(sW + sw_off(n, c, N)) = o;
    }
    tc::fence_proxy_async_smem();
  }
  if (warp == 0) {
    __syncwarp();
    tc::tmem_alloc<C::NCOLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 1 && warp <= C::PW) {
    // ------------------------------------------------------------ producers: X_src rows by cp.async
    const int pw = warp - 1;  // rows pw*64 .. pw*64+63 of each stage
    auto load_idx = [&](int it, int* out) {
      const int p0 = row0 + it * MT + pw * 64;
      out[0] = __ldg(pr.src_s + min(p0 + lane, row1 - 1));
      out[1] = __ldg(pr.src_s + min(p0 + 32 + lane, row1 - 1));
    };
    int idx[2] = {0, 0};
    if (nsub > 0) load_idx(0, idx);
    int pub = 0;
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      const uint32_t use = (uint32_t)(it / C::STAGES);
      int nidx[2] = {0, 0};
      if (it + 1 < nsub) load_idx(it + 1, nidx);
      if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
      uint8_t* a = sA(st);
#pragma unroll 4
      for (int i = 0; i < 64 / C::RPI; ++i) {
        const int rr = i * C::RPI + lane / C::CPR;  // row within this warp's 64
        const int c = lane % C::CPR;
        const int row = pw * 64 + rr;
        const int xr = __shfl_sync(0xffffffffu, rr < 32 ? idx[0] : idx[1], rr & 31);
        tc::cp_async16(a + sw_off(row, c, MT), pr.X + (size_t)xr * K + c * 8);
      }
      tc::cp_async_commit();
      if (it - pub >= C::DEPTH) {
        tc::cp_async_wait<C::DEPTH>();
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&a_full[pub % C::STAGES]);
        ++pub;
      }
      idx[0] = nidx[0];
      idx[1] = nidx[1];
    }
    tc::cp_async_wait<0>();
    tc::fence_proxy_async_smem();
    for (; pub < nsub; ++pub) tc::mbar_arrive(&a_full[pub % C::STAGES]);
  } else if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    auto issue_z = [&](int it) {  // Z_tile = X_tile . W_r into TMEM buffer it & 1
      const int st = it % C::STAGES, zb = it & 1;
      tc::mbar_wait(&a_full[st], (uint32_t)(it / C::STAGES) & 1);
      if (it >= 2) tc::mbar_wait(&z_free[zb], (uint32_t)((it >> 1) - 1) & 1);
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = tc::smem_u32(sA(st)), w0 = tc::smem_u32(sW);
#pragma unroll
        for (int ks = 0; ks < K / 16; ++ks) {
          const int kb = (ks * 32) / 128, off = (ks * 32) % 128;
          const uint64_t ad = tc::umma_desc(a0 + kb * MT * 128 + off, 16, 1024, 2u);
          const uint64_t wd = tc::umma_desc(w0 + kb * N * 128 + off, 16, 1024, 2u);
          tc::umma_bf16(tmem + C::ZCOL + zb * N, ad, wd, C::IDESC_Z, ks > 0 ? 1u : 0u);
        }
        tc::umma_commit(&z_full[zb]);
      }
      __syncwarp();
    };
    if (GAT && nsub > 0) issue_z(0);
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      if (GAT && it + 1 < nsub) issue_z(it + 1);  // one stage ahead (the producer publishes STAGES-2 deep)
      if constexpr (!GAT) tc::mbar_wait(&a_full[st], (uint32_t)(it / C::STAGES) & 1);
      tc::mbar_wait(&b_full[st], (uint32_t)(it / C::STAGES) & 1);
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = tc::smem_u32(sA(st)), b0 = tc::smem_u32(sB(st));
#pragma unroll
        for (int ks = 0; ks < MT / 16; ++ks) {
          const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
          const uint64_t ad = tc::umma_desc(a0 + ks * 16 * 128, MT * 128, 1024, 2u);
          const uint64_t bd = tc::umma_desc(b0 + ks * 16 * 128, MT * 128, 1024, 2u);
          tc::umma_bf16(tmem, ad, bd, C::IDESC_DW, acc);
        }
        tc::umma_commit(&empty[st]);
        if (it == nsub - 1) tc::umma_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ compute warps
    const int cw = warp - 1 - C::PW;         // 0..15
    const int q = warp & 3, wq = cw >> 2;    // TMEM lane quarter / column quarter for the Z drain
    const int g = lane / L, l = lane % L;    // lane group (one position at a time), lane within group
    float u[KPL], a0[EPL];
    if constexpr (GAT) {
#pragma unroll
      for (int i = 0; i < KPL; ++i) u[i] = __ldg(pr.U + (size_t)r * K + l * KPL + i);
#pragma unroll
      for (int i = 0; i < EPL; ++i) a0[i] = __ldg(pr.A + (size_t)r * 2 * N + l * EPL + i);
    }
    float cacc[KPL], aacc[EPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) cacc[i] = 0.f;
#pragma unroll
    for (int i = 0; i < EPL; ++i) aacc[i] = 0.f;
    int cur_v = -1;
    float gv[EPL], xv[KPL], Sv = 0.f, dsc = 0.f, lse = 0.f;
    const uint32_t gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (g * L));
    // dst and s_src (RGAT) / 1/c (RGCN) of the warp's positions, loaded one stage ahead
    auto load_pos = [&](int it, int& v, float& sv) {
      const int pl = row0 + it * MT + cw * C::PPW + (lane % C::PPW);
      const bool okl = lane < C::PPW && pl < row1;
      v = okl ? __ldg(pr.dst_s + pl) : -1;
      sv = okl ? __ldg((GAT ? pr.s_src : pr.inv_c) + pl) : 0.f;
    };
    int nv = -1;
    float ns = 0.f;
    if (nsub > 0) load_pos(0, nv, ns);
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      const uint32_t use = (uint32_t)(it / C::STAGES);
      const int myv = nv;
      const float mys = ns;
      if (it + 1 < nsub) load_pos(it + 1, nv, ns);
      if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);  // the stage's B buffer is free
      uint8_t* b = sB(st);
      if constexpr (GAT) {
        // drain Z (TMEM, fp32) -> bf16 lines of the B buffer; quarter q, columns [wq*N/4, (wq+1)*N/4)
        const int zb = it & 1;
        tc::mbar_wait(&z_full[zb], (uint32_t)(it >> 1) & 1);
        tc::tc_fence_after();
        const int row = q * 32 + lane;
#pragma unroll
        for (int c0 = wq * (N / 4); c0 < (wq + 1) * (N / 4); c0 += 16) {
          uint32_t v[16];
          tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + C::ZCOL + zb * N + c0, v);
          tc::tmem_ld_wait();
          uint4 w0, w1;
          w0.x = tc::pack_bf16(__uint_as_float(v[0]), __uint_as_float(v[1]));
          w0.y = tc::pack_bf16(__uint_as_float(v[2]), __uint_as_float(v[3]));
          w0.z = tc::pack_bf16(__uint_as_float(v[4]), __uint_as_float(v[5]));
          w0.w = tc::pack_bf16(__uint_as_float(v[6]), __uint_as_float(v[7]));
          w1.x = tc::pack_bf16(__uint_as_float(v[8]), __uint_as_float(v[9]));
          w1.y = tc::pack_bf16(__uint_as_float(v[10]), __uint_as_float(v[11]));
          w1.z = tc::pack_bf16(__uint_as_float(v[12]), __uint_as_float(v[13]));
          w1.w = tc::pack_bf16(__uint_as_float(v[14]), __uint_as_float(v[15]));
          *reinterpret_cast<uint4*>(b + sw_off(row, c0 / 8, MT)) = w0;
          *reinterpret_cast<uint4*>(b + sw_off(row, c0 / 8 + 1, MT)) = w1;
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&z_free[zb]);
        tc::named_bar(2, C::CW * 32);  // every Z line of the stage is in shared memory
      }
#pragma unroll
      for (int i = 0; i < PG; ++i) {
        const int lp = cw * C::PPW + g * PG + i;  // line of the stage (0..127)
        const int src_lane = g * PG + i;
        const int v = __shfl_sync(0xffffffffu, myv, src_lane);
        const float ss = __shfl_sync(0xffffffffu, mys, src_lane);
        uint4* slot = reinterpret_cast<uint4*>(b + sw_off(lp, l, MT));  // this lane's 8 features of line lp
        float dz[EPL];
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
          Vec16<__nv_bfloat16>{*slot}.to_float(zf);
          float da = 0.f;
#pragma unroll
          for (int j = 0; j < EPL; ++j) da = fmaf(gv[j], zf[j], da);
#pragma unroll
          for (int o = L / 2; o > 0; o >>= 1) da += __shfl_xor_sync(gmask, da, o);
          const float pre = ss + dsc;
          const float alpha = __expf(leaky_f(pre, pr.slope) - lse);
          const float dpre = alpha * (da - Sv) * (pre > 0.f ? 1.f : pr.slope);
#pragma unroll
          for (int j = 0; j < EPL; ++j) {
            dz[j] = fmaf(alpha, gv[j], dpre * a0[j]);
            aacc[j] = fmaf(dpre, zf[j], aacc[j]);
          }
#pragma unroll
          for (int j = 0; j < KPL; ++j) cacc[j] = fmaf(dpre, xv[j], cacc[j]);
        } else {
#pragma unroll
          for (int j = 0; j < EPL; ++j) dz[j] = 0.f;
        }
        uint4 o;
        o.x = tc::pack_bf16(dz[0], dz[1]); o.y = tc::pack_bf16(dz[2], dz[3]);
        o.z = tc::pack_bf16(dz[4], dz[5]); o.w = tc::pack_bf16(dz[6], dz[7]);
        *slot = o;
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&b_full[st]);
    }
    // per-warp partials: sum the G lane groups (fixed xor tree)
#pragma unroll
    for (int o = L; o < 32; o <<= 1) {
#pragma unroll
      for (int j = 0; j < KPL; ++j) cacc[j] += __shfl_xor_sync(0xffffffffu, cacc[j], o);
#pragma unroll
      for (int j = 0; j < EPL; ++j) aacc[j] += __shfl_xor_sync(0xffffffffu, aacc[j], o);
    }
    // epilogue: every MMA has completed, so stage 0 is free for the cross-warp scratch
    tc::mbar_wait(acc_full, 0);
    tc::tc_fence_after();
    float* s_c = reinterpret_cast<float*>(smem);  // [CW][K]
    float* s_a = s_c + C::CW * K;                 // [CW][N]
    if (g == 0) {
#pragma unroll
      for (int j = 0; j < KPL; ++j) s_c[cw * K + l * KPL + j] = cacc[j];
#pragma unroll
      for (int j = 0; j < EPL; ++j) s_a[cw * N + l * EPL + j] = aacc[j];
    }
    const int row = K == 128 ? q * 32 + lane : q * 16 + lane;  // UMMA M=64 uses lanes 0-15 of each quarter
    const bool rvalid = K == 128 || lane < 16;
    float* out = pr.part + (size_t)blockIdx.x * (K * N + K);
    constexpr int CQ = N / 4;
#pragma unroll
    for (int c0 = wq * CQ; c0 < (wq + 1) * CQ; c0 += 16) {
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
    if (wq == 0 && rvalid) out[K * N + row] = 0.f;  // bvec slot unused on this path (dA[r,0] comes from apart)
  }
  tc::tc_fence_before();
  __syncthreads();
  {
    const float* s_c = reinterpret_cast<const float*>(smem);
    const float* s_a = s_c + C::CW * K;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < C::CW; ++w) s += s_c[w * K + k];
      pr.cpart[(size_t)blockIdx.x * K + k] = s;
    }
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < C::CW; ++w) s += s_a[w * N + n];
      pr.apart[(size_t)blockIdx.x * N + n] = s;
    }
  }
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

template <int K, int N, bool GAT>
static rgnn_status bwd_fused(const rgnn_graph* g, const BwdFusedParams& p0, cudaStream_t s) {
  using C = BfCfg<K, N, GAT>;
  if (g->num_chunks == 0) return RGNN_OK;
  auto kern = k_bwd_fused_tc<K, N, GAT>;
  RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  RGNN_LAUNCH(kern, (unsigned)g->num_chunks, C::THREADS, C::SMEM, s, p0);
  return RGNN_OK;
}

bool tc_disabled();

// RGAT when s_src != null, RGCN (dZ = G_v / c_{v,r}) otherwise.
rgnn_status launch_bwd_fused_tc(int K, int N, const rgnn_graph* g, const void* X, const float* W, const float* s_src,
                                const float* lse, const float* Y, const float* dY, const float* U, const float* A,
                                float slope, float* part, float* cpart, float* apart, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  if (getenv("RGNN_DISABLE_FUSED_BWD")) return RGNN_E_UNSUPPORTED;
  BwdFusedParams p{g->chunks, g->src_s, g->dst_s, s_src, static_cast<const __nv_bfloat16*>(X), W, lse, Y, dY, U, A,
                   g->inv_c, slope, g->v0, part, cpart, apart};
  const bool gat = s_src != nullptr;
#define RGNN_BF(KK, NN)                                                               \
  if (K == KK && N == NN) return gat ? bwd_fused<KK, NN, true>(g, p, s) : bwd_fused<KK, NN, false>(g, p, s);
  RGNN_BF(64, 64)
  RGNN_BF(64, 128)
  RGNN_BF(128, 64)
  RGNN_BF(128, 128)
#undef RGNN_BF
  return RGNN_E_UNSUPPORTED;
}

}  // namespace rgnn
