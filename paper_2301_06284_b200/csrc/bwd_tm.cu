// bwd_tm.cu -- RGAT backward on the tensor cores with the messages recomputed in TMEM (bf16 layer).
//
// Per 128-position stage of one dW chunk (relation r fixed, positions in (etype, dst) order):
//   * warps 1..4 (producers): X[src_s[p]] rows -> shared memory by 16-byte cp.async (one layout
//     read two ways: K-major A of Z = X_src W_r, MN-major A of dW_r = X_src^T dZ), and per position
//     dst_s[p], the source score s_src of its Z row and lse[dst] (4-byte cp.async); a later stage's
//     X rows are prefetched to L2;
//   * warp 0: Z_tile = X_src . W_r into TMEM (two buffers, tcgen05.mma kind::f16, W_r^T resident in
//     shared memory), then, once the compute warps have written the stage's gradient rows,
//     D += X_src^T dZ and Db += X_src^T dpre;
//   * warps 5..20 (compute: two groups of 8 warps taking alternate stages, so one group's loads
//     overlap the other's arithmetic).  Per stage a group first finds the stage's destination runs
//     (equal dst_s, contiguous) and reads, once per run and coalesced, G_v = dY_v (kept as a bf16
//     row in shared memory), S_v = G_v . Y_v and the destination score x_v . U[r] (U[r] = W_r A[r,1],
//     P:706-708); then one TMEM lane = one position per thread, two warps per lane quarter splitting
//     the columns:
//        pre = s_src + x_v . U[r],  alpha = exp(leaky(pre) - lse_v)      (Listing 1)
//        dalpha = G_v . Z_p  (Z_p from TMEM, G_v from the run row),  dpre = alpha (dalpha - S_v) leaky'(pre)
//        dZ_p = alpha G_v -> bf16 -> MN-major SW128 smem line (the dW MMA's B operand)
//     (SURVEY §8 backward formulas, §3.5).  The score's source term of dW,
//     (sum_p dpre_p x_src(p)) (x) A[r,0] = Db (x) A[r,0], is added by k_dw_reduce.
// The message rows are never read from HBM: Z = X_src W_r is the MMA the forward's typed GEMM issued
// (P:300-305), so the backward reads the X_src rows plus one G / Y / x row triple per run.  The
// destination term c_r = sum_p dpre_p x_dst(p) is summed by k_dst_term from dpre (measured r02: summing it
// per run inside this kernel, after each stage's per-position pass, made the backward 0.33 ms slower on
// ogbn-mag against 0.20 ms for k_dst_term); part is reduced in chunk order by k_dw_reduce (deterministic).
#include <math_constants.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

template <int K, int N>
struct TmCfg {
  static constexpr int MT = 128;                 // positions per stage = TMEM lanes
  static constexpr int A_BYTES = MT * K * 2;     // X_src stage
  static constexpr int SC_BYTES = MT * 4 * 3;    // dst, s_src, lse
  static constexpr int B_BYTES = MT * N * 2;     // dZ (MN-major SW128)
  static constexpr int B2_BYTES = MT * 16 * 2;   // dpre column operand
  static constexpr int DZ_BYTES = B_BYTES + B2_BYTES;
#ifndef RGNN_TM_DZB
#define RGNN_TM_DZB 2  // dZ operand buffers: 2 (one per group) or 1 (shared; one more X stage fits: measured
                       // mag 2.84 vs 2.57 ms with 2)
#endif
  static constexpr int DZB = RGNN_TM_DZB;
  static constexpr int W_BYTES = N * K * 2;      // W_r^T, K-major SW128
  static constexpr int GSEL_BYTES = N == 64 ? 16384 : 7168;  // bf16 run rows per buffer (runs past CAP read dY directly)
  static constexpr int CAP = GSEL_BYTES / (N * 2);
  static constexpr int RUNTAB = MT * 4 * 4;      // per buffer: run of each position; S, dst score, dst per run
#ifndef RGNN_TM_SMAX
#define RGNN_TM_SMAX 6
#endif
#ifndef RGNN_TM_RPF
#define RGNN_TM_RPF 2  // run rows (dY, Y, x of each run head) of stage it + RPF prefetched to L2 when stage it is
                       // issued (0: off)
#endif
#ifndef RGNN_TM_EARLY
#define RGNN_TM_EARLY 0  // 1: build the group's next run table and request its first run rows before this stage's
                        // per-position pass (measured r02: 2.49 -> 3.05 ms on ogbn-mag)
#endif
#ifndef RGNN_TM_XPF
#define RGNN_TM_XPF 2  // X rows of stage it + STAGES + XPF - 1 prefetched to L2 when stage it is issued (0: off)
#endif
  static constexpr int FIXED = 1024 + W_BYTES + DZB * DZ_BYTES + 2 * GSEL_BYTES + 2 * RUNTAB + 2 * 2 * MT * 4 + K * 4 + 256;
  static constexpr int ST_FIT = (227 * 1024 - FIXED) / (A_BYTES + SC_BYTES);
  static constexpr int STAGES = ST_FIT > RGNN_TM_SMAX ? RGNN_TM_SMAX : ST_FIT;
  static constexpr int SMEM = FIXED + STAGES * (A_BYTES + SC_BYTES);
#ifndef RGNN_TM_PW
#define RGNN_TM_PW 4  // producer warps (the first four stage the per-position scalars; 8 measured slower: 2.50 -> 2.69 ms,
                      // the compute warps lose registers at 800 threads)
#endif
#ifndef RGNN_TM_CW
#define RGNN_TM_CW 16  // compute warps: two groups of CW / 2 (16: two warps per lane quarter splitting the columns;
                       // 8, one warp per quarter over all columns, measured 2.48 -> 2.99 ms)
#endif
  static constexpr int PW = RGNN_TM_PW, CW = RGNN_TM_CW;  // producers, two compute groups of CW / 2 warps
  static constexpr int WPG = CW / 2;             // warps per compute group
  static constexpr int HPQ = WPG / 4;            // warps per TMEM lane quarter in a group (column parts)
  static constexpr int THREADS = 32 * (1 + PW + CW);
  static constexpr int ZOFF = N + 32;            // TMEM: [0,N) dW, [N,N+16) Db, Z buffers at ZOFF, ZOFF+N
  static constexpr int NCOLS = ZOFF + 2 * N <= 256 ? 256 : 512;
  static constexpr int NH = N / HPQ;             // columns per compute warp
  static constexpr int CPR = K * 2 / 16;         // 16-byte chunks per X row
  static constexpr int RPI = 32 / CPR;           // X rows per warp-wide cp.async
  static constexpr int LPR = N / 4;              // per-run pass: lanes per G row (4 floats each)
  static constexpr int RUNS_PI = 32 / LPR;       // runs per warp iteration
  static constexpr uint32_t IDESC_Z = tc::idesc_bf16(128, N, 0, 0);
  static constexpr uint32_t IDESC_W = tc::idesc_bf16(K, N, 1, 1);
  static constexpr uint32_t IDESC_B = tc::idesc_bf16(K, 16, 1, 1);
  static_assert(STAGES >= 3 && SMEM <= 227 * 1024, "bwd_tm shared memory");
  static_assert(NH % 16 == 0, "compute halves take 16-column TMEM loads");
};

struct BwdTmParams {
  const Tile* chunks;
  const int32_t* src_s;
  const int32_t* dst_s;
  const int32_t* zmap;  // compact: s_src row of position p (null = p)
  const float* s_src;
  const float* U;       // [R, K]
  const float* lse;
  const __nv_bfloat16* X;
  int64_t v0;
  const __nv_bfloat16* Wt;  // [R, N, K]
  const float* Y;
  const float* dY;
  float slope;
  float* part;
  float* dpre;
  float2* ad;
};

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// KPL consecutive bf16 -> fp32 (KPL in {2, 4, 8}: one 4-, 8- or 16-byte load)
template <int KPL>
__device__ __forceinline__ void load_bf16(const __nv_bfloat16* p, float* out) {
  if constexpr (KPL == 8) {
    Vec16<__nv_bfloat16>{ldg16(p)}.to_float(out);
  } else if constexpr (KPL == 4) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
  } else {
    const uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(p));
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
    out[0] = a.x; out[1] = a.y;
  }
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(dst)), "l"(src) : "memory");
}

// RGNN_TM_TRACE=1 builds: clock64 stamps of the pipeline events of one CTA (lane 0 of the recording warp;
// slots per stage: 0-2 producer, 3-5 and 14 MMA, 6-13 compute group), read by the launcher (tools/tm_trace.py)
#ifndef RGNN_TM_TRACE
#define RGNN_TM_TRACE 0
#endif
#if RGNN_TM_TRACE
__device__ long long g_tm_trace[256 * 16];
#define TMT(it, slot)                                                                                     \
  do {                                                                                                    \
    if (blockIdx.x == 300 && lane == 0 && (it) < 256) g_tm_trace[(it) * 16 + (slot)] = clock64() - t_start; \
  } while (0)
#else
#define TMT(it, slot) \
  do {                \
  } while (0)
#endif

template <int K, int N>
__global__ void __launch_bounds__(TmCfg<K, N>::THREADS, 1) k_bwd_rgat_tm(BwdTmParams pr) {
#if RGNN_TM_TRACE
  const long long t_start = clock64();
#endif
  using C = TmCfg<K, N>;
  constexpr int MT = C::MT;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself (the compiler keeps shared-space accesses)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;
  uint8_t* sDZ = sW + C::W_BYTES;                      // [2][B | B2]
  uint8_t* sAst = sDZ + C::DZB * C::DZ_BYTES;          // [STAGES][A]
  uint8_t* sGs = sAst + C::STAGES * C::A_BYTES;        // [2][CAP][N] bf16 run rows
  uint8_t* sSc = sGs + 2 * C::GSEL_BYTES;              // [STAGES][dst | pre | lse]
  uint8_t* sRt = sSc + C::STAGES * C::SC_BYTES;        // [2][run of position | S of run | dst of run]
  float* sT = reinterpret_cast<float*>(sRt + 2 * C::RUNTAB);  // [2 buf][2 half][MT] partial dots
  float* sU = sT + 2 * 2 * MT;                                // U[r] (fp32)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sU + K);
  uint64_t* a_full = bar;
  uint64_t* empty = a_full + C::STAGES;
  uint64_t* zfull = empty + C::STAGES;
  uint64_t* zempty = zfull + 2;
  uint64_t* bfull = zempty + 2;
  uint64_t* dzempty = bfull + 2;
  uint64_t* idx_full = dzempty + 2;
  uint64_t* acc_full = idx_full + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  auto sA = [&](int s) { return sAst + s * C::A_BYTES; };
  auto sB = [&](int b) { return sDZ + (C::DZB == 1 ? 0 : b) * C::DZ_BYTES; };
  auto sB2 = [&](int b) { return sDZ + (C::DZB == 1 ? 0 : b) * C::DZ_BYTES + C::B_BYTES; };
  auto sG = [&](int b) { return reinterpret_cast<__nv_bfloat16*>(sGs + b * C::GSEL_BYTES); };
  auto sDst = [&](int s) { return reinterpret_cast<int*>(sSc + s * C::SC_BYTES); };
  auto sSs = [&](int s) { return reinterpret_cast<float*>(sSc + s * C::SC_BYTES + MT * 4); };
  auto sLse = [&](int s) { return reinterpret_cast<float*>(sSc + s * C::SC_BYTES + MT * 8); };
  auto sRun = [&](int b) { return reinterpret_cast<int*>(sRt + b * C::RUNTAB); };
  auto sS = [&](int b) { return reinterpret_cast<float*>(sRt + b * C::RUNTAB + MT * 4); };
  auto sHv = [&](int b) { return reinterpret_cast<int*>(sRt + b * C::RUNTAB + MT * 8); };
  auto sDs = [&](int b) { return reinterpret_cast<float*>(sRt + b * C::RUNTAB + MT * 12); };
  // 16-byte chunk c of line `row` in a 128B-swizzled tile of `rows` lines per 64-element block
  auto swz = [&](int c, int row, int rows) { return (c >> 3) * (rows * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Tile ch = pr.chunks[blockIdx.x];
  const int r = ch.r, row0 = ch.row0, row1 = ch.row1;
  const int nsub = (row1 - row0 + MT - 1) / MT;

  // W_r^T (K-major SW128 B operand of the Z MMA), once per CTA
  for (int i = threadIdx.x; i < N * (K / 8); i += blockDim.x) {
    const int n = i / (K / 8), c = i % (K / 8);
    tc::cp_async16(sW + swz(c, n, N), pr.Wt + ((size_t)r * N + n) * K + c * 8);
  }
  tc::cp_async_commit();
  for (int k = threadIdx.x; k < K; k += blockDim.x) sU[k] = __ldg(pr.U + (size_t)r * K + k);
  for (int i = threadIdx.x; i < C::DZB * C::B2_BYTES / 16; i += blockDim.x) {  // dpre operand: cols 2..15 = 0
    const int b = i / (C::B2_BYTES / 16), o = i % (C::B2_BYTES / 16);
    reinterpret_cast<uint4*>(sB2(b))[o] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      tc::mbar_init(&a_full[i], C::PW * 32);
      tc::mbar_init(&empty[i], 1);
      tc::mbar_init(&idx_full[i], 4 * 32);  // producer warps 0..3 stage the destinations
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&zfull[i], 1);
      tc::mbar_init(&zempty[i], C::CW / 2);  // buffer i is used by compute group i only
      tc::mbar_init(&bfull[i], C::CW / 2);
      tc::mbar_init(&dzempty[i], 1);
    }
    tc::mbar_init(acc_full, 1);
    tc::mbar_fence_init();
  }
  tc::cp_async_wait<0>();
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
    // ------------------------------------------------------------ producers
    // warps 0..3 of the producers stage the per-position scalars (one position per thread); all PW warps
    // copy X rows, MT / PW rows each (more warps issue a stage's copies sooner)
    constexpr int RWX = MT / C::PW;  // X rows per producer warp
    const int pw = warp - 1, lp = pw * 32 + lane;
    const bool spos = pw < 4;        // this warp stages scalars
    auto load_idx = [&](int it, int& v, int& p, int& zr) {
      p = row0 + it * MT + lp;
      const int pc = min(p, row1 - 1);
      v = __ldg(pr.dst_s + pc);
      zr = pr.zmap ? __ldg(pr.zmap + pc) : pc;
    };
    auto load_src = [&](int it) {  // lanes < RWX: source row of X row pw * RWX + lane of stage it
      const int q = min(row0 + it * MT + pw * RWX + (lane % RWX), row1 - 1);  // padding rows re-read a valid row
      return __ldg(pr.src_s + q);
    };
    int src = 0, v = 0, p = 0, zr = 0;
    if (nsub > 0) {
      src = load_src(0);
      if (spos) load_idx(0, v, p, zr);
    }
    // the indices the prefetches need are loaded one iteration before they are used (a prefetch that
    // waits for its own index load costs the producer a memory latency per stage)
    constexpr int XA = C::STAGES + RGNN_TM_XPF - 1;  // X rows prefetched XA stages ahead
    auto pf_src = [&](int it) {
      const int q = row0 + it * MT + pw * RWX + (lane % RWX);
      return (lane < RWX && q < row1) ? __ldg(pr.src_s + q) : -1;
    };
    auto pf_dst = [&](int it) { const int q = row0 + it * MT + lp; return (spos && q < row1) ? __ldg(pr.dst_s + q) : -1; };
    int xs = RGNN_TM_XPF > 0 ? pf_src(XA) : -1;
    int rv = RGNN_TM_RPF > 0 ? pf_dst(RGNN_TM_RPF) : -1;
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      const uint32_t use = (uint32_t)(it / C::STAGES);
      int nsrc = 0, nv = 0, np = 0, nzr = 0;
      if (it + 1 < nsub) {
        nsrc = load_src(it + 1);
        if (spos) load_idx(it + 1, nv, np, nzr);
      }
      const int xs_n = RGNN_TM_XPF > 0 ? pf_src(it + 1 + XA) : -1;
      const int rv_n = RGNN_TM_RPF > 0 ? pf_dst(it + 1 + RGNN_TM_RPF) : -1;
      if (RGNN_TM_XPF > 0 && xs >= 0) {  // L2 prefetch of a later stage's X rows (the ring is only STAGES deep)
        const char* xp = reinterpret_cast<const char*>(pr.X + (size_t)xs * K);
#pragma unroll
        for (int o = 0; o < K * 2; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(xp + o));
      }
      if (pw == 0) TMT(it, 0);
      if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
      if (pw == 0) TMT(it, 1);
      if (spos) {
        // the stage's destinations go out first (plain stores + idx_full): the compute group finds the
        // stage's runs and reads their rows while the X rows are still in flight
        sDst(st)[lp] = p < row1 ? v : -1;
        tc::mbar_arrive(&idx_full[st]);
        if (p < row1) {
          cp_async4(sSs(st) + lp, pr.s_src + zr);
          cp_async4(sLse(st) + lp, pr.lse + v);
        }
      }
      uint8_t* a = sA(st);
#pragma unroll
      for (int i = 0; i < RWX / C::RPI; ++i) {  // all row indices first, then the copies back to back
        const int rr = i * C::RPI + lane / C::CPR;
        const int c = lane % C::CPR;
        const int xr = __shfl_sync(0xffffffffu, src, rr);
        tc::cp_async16(a + swz(c, pw * RWX + rr, MT), pr.X + (size_t)xr * K + c * 8);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&a_full[st])) : "memory");
      if (pw == 0) TMT(it, 2);
      // L2 prefetch of the per-destination rows (dY, Y, x of each run head) of stage it + RGNN_TM_RPF, so
      // that they have arrived when a compute group reads them (it does so as soon as a stage is issued)
      if (RGNN_TM_RPF > 0 && spos) {
        const int vf = rv;
        const int vfp = __shfl_up_sync(0xffffffffu, vf, 1);
        if (vf >= 0 && (lane == 0 || vfp != vf)) {
          const char* gp = reinterpret_cast<const char*>(pr.dY + (size_t)vf * N);
          const char* yp = reinterpret_cast<const char*>(pr.Y + (size_t)vf * N);
          const char* xp = reinterpret_cast<const char*>(pr.X + (pr.v0 + vf) * (int64_t)K);
#pragma unroll
          for (int o = 0; o < N * 4; o += 128) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(gp + o));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(yp + o));
          }
#pragma unroll
          for (int o = 0; o < K * 2; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(xp + o));
        }
      }
      src = nsrc; v = nv; p = np; zr = nzr;
      xs = xs_n; rv = rv_n;
    }
    tc::cp_async_wait<0>();
  } else if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t w0 = tc::smem_u32(sW);
    auto issue_dw = [&](int j) {
      const int bj = j & 1, sj = j % C::STAGES;
      tc::mbar_wait(&bfull[bj], (uint32_t)(j >> 1) & 1);
      TMT(j, 14);
      tc::fence_proxy_async_smem();
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = tc::smem_u32(sA(sj)), b0 = tc::smem_u32(sB(bj)), c0 = tc::smem_u32(sB2(bj));
#pragma unroll
        for (int ks = 0; ks < MT / 16; ++ks) {
          const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
          const uint64_t ad = tc::umma_desc(a0 + ks * 16 * 128, MT * 128, 1024, 2u);
          const uint64_t bd = tc::umma_desc(b0 + ks * 16 * 128, MT * 128, 1024, 2u);
          tc::umma_bf16(tmem, ad, bd, C::IDESC_W, acc);
          const uint64_t cd = tc::umma_desc(c0 + ks * 512, 256, 128, 0u);
          tc::umma_bf16(tmem + N, ad, cd, C::IDESC_B, acc);
        }
        tc::umma_commit(&empty[sj]);
        tc::umma_commit(&dzempty[C::DZB == 1 ? 0 : bj]);
      }
      __syncwarp();
    };
    // (measured: issuing Z and dW MMAs in readiness order by polling both barriers was slower, 2.57 ->
    // 3.33 ms on ogbn-mag; the MMA warp issues Z(it), then the dW of the previous stage)
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES, buf = it & 1;
      tc::mbar_wait(&a_full[st], (uint32_t)(it / C::STAGES) & 1);
      if (it >= 2) tc::mbar_wait(&zempty[buf], (uint32_t)((it - 2) >> 1) & 1);
      tc::fence_proxy_async_smem();  // cp.async (generic proxy) rows -> tcgen05 (async proxy)
      tc::tc_fence_after();
      TMT(it, 3);
      if (lane == 0) {
        const uint32_t a0 = tc::smem_u32(sA(st));
#pragma unroll
        for (int ks = 0; ks < K / 16; ++ks) {
          const int kb = ks / 4, off = (ks % 4) * 32;
          const uint64_t ad = tc::umma_desc(a0 + kb * MT * 128 + off, 16, 1024, 2u);
          const uint64_t bd = tc::umma_desc(w0 + kb * N * 128 + off, 16, 1024, 2u);
          tc::umma_bf16(tmem + C::ZOFF + buf * N, ad, bd, C::IDESC_Z, ks > 0 ? 1u : 0u);
        }
        tc::umma_commit(&zfull[buf]);
        TMT(it, 4);
      }
      __syncwarp();
      if (it >= 1) issue_dw(it - 1);
      TMT(it, 5);
    }
    if (nsub > 0) issue_dw(nsub - 1);
    if (lane == 0) tc::umma_commit(acc_full);
    __syncwarp();
  } else {
    // ------------------------------------------------------------ compute warps
    const int cw = warp - 1 - C::PW;   // 0..15
    const int grp = cw / C::WPG;       // compute group: stages it with it % 2 == grp (TMEM / dZ / run buffer grp)
    const int gw = cw % C::WPG;        // warp within the group
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int h = gw >> 2;             // column part (HPQ warps per lane quarter)
    const int lp = q * 32 + lane;      // stage row (TMEM lane) = position of this thread
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    constexpr int LPR = C::LPR, RPIT = C::RUNS_PI, BATCH = 4, KPL = K / LPR;
    const int sub = lane / LPR, ln = lane % LPR;
    volatile int* sFlag = reinterpret_cast<volatile int*>(tmem_slot + 1);  // per group: next stage staged
    // (1) the stage's destination runs: a run = maximal block of stage rows with one destination (rows of
    // a relation are sorted by destination); every warp of the group derives the same table, warp 0
    // stores it.  Returns the number of runs.
    auto build_table = [&](int it) -> int {
      const int st = it % C::STAGES, buf = it & 1;
      tc::mbar_wait(&idx_full[st], (uint32_t)(it / C::STAGES) & 1);
      int nruns = 0, lastv = -2;
#pragma unroll
      for (int c = 0; c < MT / 32; ++c) {
        const int l2 = c * 32 + lane;
        const bool val = row0 + it * MT + l2 < row1;
        const int v = val ? sDst(st)[l2] : -1;
        int vprev = __shfl_up_sync(0xffffffffu, v, 1);
        if (lane == 0) vprev = lastv;
        const bool head = val && v != vprev;
        const unsigned hb = __ballot_sync(0xffffffffu, head);
        const int j = nruns + __popc(hb & (0xffffffffu >> (31 - lane))) - 1;
        if (gw == 0) {
          sRun(buf)[l2] = j;
          if (head) sHv(buf)[j] = v;
        }
        nruns += __popc(hb);
        lastv = __shfl_sync(0xffffffffu, v, 31);
      }
      return nruns;
    };
    // (2) per run (warps of the group take interleaved runs, NB runs' loads in flight per warp): G_v as a
    // bf16 row (if j < CAP), S_v = G_v . Y_v and the destination score x_v . U[r], read once per run
    auto load_run = [&](int buf, int nruns, int jj, float4& g, float4& y, float* xv) {
      if (jj < nruns) {
        const int v = sHv(buf)[jj];
        g = __ldg(reinterpret_cast<const float4*>(pr.dY + (size_t)v * N) + ln);
        y = __ldg(reinterpret_cast<const float4*>(pr.Y + (size_t)v * N) + ln);
        load_bf16<KPL>(pr.X + (pr.v0 + v) * (int64_t)K + ln * KPL, xv);
      } else {
        g = y = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < KPL; ++i) xv[i] = 0.f;
      }
    };
    auto store_run = [&](int buf, int nruns, int jj, float4 g, float4 y, const float* xv) {
      // G_v as the per-position pass sees it (bf16), so that sum_p alpha_p dalpha_p = S_v holds for the
      // rounded values as it does in exact arithmetic (Y_v = sum_p alpha_p bf16(Z_p))
      g = make_float4(bf16r(g.x), bf16r(g.y), bf16r(g.z), bf16r(g.w));
      float sv = g.x * y.x;
      sv = fmaf(g.y, y.y, sv);
      sv = fmaf(g.z, y.z, sv);
      sv = fmaf(g.w, y.w, sv);
      float dsc = 0.f;
#pragma unroll
      for (int i = 0; i < KPL; ++i) dsc = fmaf(xv[i], sU[ln * KPL + i], dsc);
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) {
        sv += __shfl_xor_sync(0xffffffffu, sv, o);
        dsc += __shfl_xor_sync(0xffffffffu, dsc, o);
      }
      if (jj < nruns) {
        if (ln == 0) {
          sS(buf)[jj] = sv;
          sDs(buf)[jj] = dsc;
        }
        if (jj < C::CAP)
          *reinterpret_cast<uint2*>(sG(buf) + (size_t)jj * N + ln * 4) =
              make_uint2(tc::pack_bf16(g.x, g.y), tc::pack_bf16(g.z, g.w));
      }
    };
    auto runs_from = [&](int buf, int nruns, int j0) {  // runs j0, j0 + 8 RPIT, ... of this warp, BATCH at a time
      for (; j0 < nruns; j0 += C::WPG * RPIT * BATCH) {
        float4 g[BATCH], y[BATCH];
        float xv[BATCH][KPL];
#pragma unroll
        for (int b = 0; b < BATCH; ++b) load_run(buf, nruns, j0 + b * C::WPG * RPIT + sub, g[b], y[b], xv[b]);
#pragma unroll
        for (int b = 0; b < BATCH; ++b) store_run(buf, nruns, j0 + b * C::WPG * RPIT + sub, g[b], y[b], xv[b]);
      }
    };
    auto prep = [&](int it) {  // blocking: the group's previous stage is finished by all its warps first
      tc::named_bar(9 + grp, C::WPG * 32);
      const int nr = build_table(it);
      tc::named_bar(9 + grp, C::WPG * 32);
      runs_from(it & 1, nr, gw * RPIT);
      tc::named_bar(9 + grp, C::WPG * 32);  // run rows and scalars visible to the group
    };
    if (grp < nsub) prep(grp);
    for (int it = grp; it < nsub; it += 2) {
      const int st = it % C::STAGES, buf = it & 1;
      const int p = row0 + it * MT + lp;
      const bool valid = p < row1;
      // (3) per position
      tc::mbar_wait(&a_full[st], (uint32_t)(it / C::STAGES) & 1);  // s_src, lse of the stage
      tc::mbar_wait(&zfull[buf], (uint32_t)(it >> 1) & 1);
      if (gw == 0) TMT(it, 9);
      tc::tc_fence_after();
      const float lse = valid ? sLse(st)[lp] : 0.f;
      const int j = valid ? sRun(buf)[lp] : 0;
      const float S = valid ? sS(buf)[j] : 0.f;
      const float pre = valid ? sSs(st)[lp] + sDs(buf)[j] : 0.f;
      const bool in_smem = j < C::CAP;
      const __nv_bfloat16* grow = sG(buf) + (size_t)(in_smem ? j : 0) * N + h * C::NH;
      const float* gglob = pr.dY + (size_t)(valid && !in_smem ? sDst(st)[lp] : 0) * N + h * C::NH;
      const float alpha = valid ? __expf((pre > 0.f ? pre : pr.slope * pre) - lse) : 0.f;
      // the group's next stage: if its indices are already staged, its run table is built and the first
      // of its run rows are requested now (in flight during this stage's per-position pass)
      const bool nxt = it + 2 < nsub;
      bool early = false;
      int nr2 = 0;
      float4 eg[2], ey[2];
      float ex[2][KPL];
      if (RGNN_TM_EARLY && nxt) {
        if (gw == 0 && lane == 0)
          sFlag[grp] = tc::mbar_try(&idx_full[(it + 2) % C::STAGES], (uint32_t)((it + 2) / C::STAGES) & 1) ? 1 : 0;
        tc::named_bar(9 + grp, C::WPG * 32);  // every warp has read this stage's run entries; the flag is visible
        early = sFlag[grp] != 0;
        if (early) {
          nr2 = build_table(it + 2);
          tc::named_bar(9 + grp, C::WPG * 32);
#pragma unroll
          for (int e = 0; e < 2; ++e) load_run(buf, nr2, gw * RPIT + e * C::WPG * RPIT + sub, eg[e], ey[e], ex[e]);
        }
      }
      if (gw == 0) TMT(it, 10);
      if (C::DZB == 1) {  // one dZ buffer: the dW MMAs of the previous stage (other group) have read it
        if (it >= 1) tc::mbar_wait(&dzempty[0], (uint32_t)(it - 1) & 1);
      } else if (it >= 2) {
        tc::mbar_wait(&dzempty[buf], (uint32_t)((it - 2) >> 1) & 1);
      }
      if (gw == 0) TMT(it, 15);
      uint8_t* b = sB(buf);
      float t = 0.f;
#pragma unroll
      for (int c = 0; c < C::NH; c += 16) {
        uint32_t z[16];
        tc::tmem_ld16(tl + C::ZOFF + buf * N + h * C::NH + c, z);
        float g[16];
        if (in_smem) {
          const uint4 u0 = *reinterpret_cast<const uint4*>(grow + c);
          const uint4 u1 = *reinterpret_cast<const uint4*>(grow + c + 8);
          Vec16<__nv_bfloat16>{u0}.to_float(g);
          Vec16<__nv_bfloat16>{u1}.to_float(g + 8);
        } else {  // a stage with more runs than the run-row buffer holds: the fp32 row, rounded like them
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(gglob + c) + i);
            g[4 * i] = bf16r(f.x);
            g[4 * i + 1] = bf16r(f.y);
            g[4 * i + 2] = bf16r(f.z);
            g[4 * i + 3] = bf16r(f.w);
          }
        }
        tc::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; i += 2) {  // Z rounded as the forward stored it (one cvt per pair):
          const uint32_t zb = tc::pack_bf16(__uint_as_float(z[i]), __uint_as_float(z[i + 1]));
          t = fmaf(g[i], __uint_as_float(zb << 16), t);
          t = fmaf(g[i + 1], __uint_as_float(zb & 0xffff0000u), t);
        }
        // for a destination with one in-edge Y_v = bf16(Z_p), so dalpha - S_v must vanish exactly)
        uint4 o0 = make_uint4(0, 0, 0, 0), o1 = make_uint4(0, 0, 0, 0);
        if (valid) {
          o0 = make_uint4(tc::pack_bf16(alpha * g[0], alpha * g[1]), tc::pack_bf16(alpha * g[2], alpha * g[3]),
                          tc::pack_bf16(alpha * g[4], alpha * g[5]), tc::pack_bf16(alpha * g[6], alpha * g[7]));
          o1 = make_uint4(tc::pack_bf16(alpha * g[8], alpha * g[9]), tc::pack_bf16(alpha * g[10], alpha * g[11]),
                          tc::pack_bf16(alpha * g[12], alpha * g[13]), tc::pack_bf16(alpha * g[14], alpha * g[15]));
        }
        const int ck = (h * C::NH + c) / 8;  // 16-byte chunk of the dZ line
        *reinterpret_cast<uint4*>(b + swz(ck, lp, MT)) = o0;
        *reinterpret_cast<uint4*>(b + swz(ck + 1, lp, MT)) = o1;
      }
      // this stage's Z buffer and run rows are consumed
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&zempty[buf]);
      if (gw == 0) TMT(it, 11);
      // the two halves' partial dots, summed in a fixed order
      if (C::HPQ == 2) {
        sT[(buf * 2 + h) * MT + lp] = t;
        tc::named_bar(1 + grp * 4 + q, 64);
      }
      if (gw == 0) TMT(it, 12);
      const float dot = C::HPQ == 2 ? sT[(buf * 2 + 0) * MT + lp] + sT[(buf * 2 + 1) * MT + lp] : t;
      const float dp = valid ? alpha * (dot - S) * (pre > 0.f ? 1.f : pr.slope) : 0.f;
      if (h == 0) {
        // dpre as hi + lo bf16 (columns 0, 1 of the side operand): Db = X_src^T dpre to ~2^-16
        const float hi = __bfloat162float(__float2bfloat16_rn(dp));
        *reinterpret_cast<uint32_t*>(sB2(buf) + (lp >> 3) * 256 + (lp & 7) * 16) = tc::pack_bf16(hi, dp - hi);
        if (valid) {
          pr.dpre[p] = dp;
          if (pr.ad) pr.ad[p] = make_float2(alpha, dp);
        }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bfull[buf]);
      if (gw == 0) TMT(it, 13);
      if (early) {  // the next stage's run rows (their first loads were in flight during the pass above)
        tc::named_bar(9 + grp, C::WPG * 32);  // every warp is done with this stage's run rows
#pragma unroll
        for (int e = 0; e < 2; ++e) store_run(buf, nr2, gw * RPIT + e * C::WPG * RPIT + sub, eg[e], ey[e], ex[e]);
        runs_from(buf, nr2, gw * RPIT + 2 * C::WPG * RPIT);
        tc::named_bar(9 + grp, C::WPG * 32);
      } else if (nxt) {
        prep(it + 2);
      }
    }
    // epilogue: TMEM accumulators -> part[c]; the four warps of a lane quarter split the columns
    tc::mbar_wait(acc_full, 0);
    tc::tc_fence_after();
    const int row = K == 128 ? q * 32 + lane : q * 16 + lane;  // M = 64: lanes 0..15 of each quarter
    const bool rvalid = K == 128 || lane < 16;
    float* out = pr.part + (size_t)blockIdx.x * (K * N + K);
    for (int c0 = (cw >> 2) * 16; c0 < N; c0 += (C::CW / 4) * 16) {  // the CW / 4 warps of a lane quarter
      uint32_t vv[16];
      tc::tmem_ld16(tl + c0, vv);
      tc::tmem_ld_wait();
      if (rvalid) {
        float4* o = reinterpret_cast<float4*>(out + (size_t)row * N + c0);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          o[jj] = make_float4(__uint_as_float(vv[4 * jj]), __uint_as_float(vv[4 * jj + 1]),
                              __uint_as_float(vv[4 * jj + 2]), __uint_as_float(vv[4 * jj + 3]));
      }
    }
    if (cw < 4) {
      uint32_t vv[16];
      tc::tmem_ld16(tl + N, vv);
      tc::tmem_ld_wait();
      if (rvalid) out[K * N + row] = __uint_as_float(vv[0]) + __uint_as_float(vv[1]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

// W [R, K, N] fp32 -> Wt [R, N, K] bf16 (RNE), the K-major B operand of the Z MMA (same rounding as the
// forward's typed GEMM).
__global__ void k_tm_wt(int R, int K, int N, const float* __restrict__ W, __nv_bfloat16* __restrict__ Wt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)R * K * N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / ((int64_t)K * N));
    const int rem = (int)(i - (int64_t)r * K * N);
    const int n = rem / K, k = rem - n * K;
    Wt[i] = __float2bfloat16_rn(W[((size_t)r * K + k) * N + n]);
  }
}

bool tc_disabled();

bool bwd_tm_enabled(int K, int N, int prec) {
  static const bool off = getenv("RGNN_BWD_V1") != nullptr || getenv("RGNN_DISABLE_FUSED_BWD") != nullptr;
  return prec == RGNN_BF16 && !off && !tc_disabled() && (K == 64 || K == 128) && (N == 64 || N == 128);
}

template <int K, int N>
static rgnn_status bwd_tm(const rgnn_graph* g, const BwdTmParams& p, cudaStream_t s) {
  using C = TmCfg<K, N>;
  auto kern = k_bwd_rgat_tm<K, N>;
  RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  RGNN_LAUNCH(kern, (unsigned)g->num_chunks, C::THREADS, C::SMEM, s, p);
#if RGNN_TM_TRACE
  static long long host[256 * 16];
  cudaStreamSynchronize(s);
  cudaMemcpyFromSymbol(host, g_tm_trace, sizeof(host));
  if (FILE* f = fopen("gpurun_out/tm_trace.txt", "w")) {
    fprintf(f, "STAGES %d chunk300 rows %d\n", C::STAGES, g->num_chunks > 300 ? 0 : -1);
    for (int i = 0; i < 256; ++i) {
      for (int j = 0; j < 16; ++j) fprintf(f, "%lld ", host[i * 16 + j]);
      fprintf(f, "\n");
    }
    fclose(f);
  }
#endif
  return RGNN_OK;
}

rgnn_status launch_bwd_rgat_tm(int K, int N, const rgnn_graph* g, const void* X, const float* W, void* Wt,
                               const int32_t* zmap, const float* s_src, const float* U, const float* lse,
                               const float* Y, const float* dY, float slope, float* part, float* dpre, float2* ad,
                               cudaStream_t s) {
  tc::watchdog_init();
  if (g->num_chunks == 0) return RGNN_OK;
  auto* wt = static_cast<__nv_bfloat16*>(Wt);
  const int64_t nw = (int64_t)g->R * K * N;
  RGNN_LAUNCH(k_tm_wt, (unsigned)std::max<int64_t>(1, std::min<int64_t>((nw + 255) / 256, 4096)), 256, 0, s, g->R, K,
              N, W, wt);
  BwdTmParams p{g->chunks, g->src_s, g->dst_s, zmap, s_src, U, lse, static_cast<const __nv_bfloat16*>(X), g->v0, wt,
                Y, dY, slope, part, dpre, ad};
  if (K == 64 && N == 64) return bwd_tm<64, 64>(g, p, s);
  if (K == 64 && N == 128) return bwd_tm<64, 128>(g, p, s);
  if (K == 128 && N == 64) return bwd_tm<128, 64>(g, p, s);
  if (K == 128 && N == 128) return bwd_tm<128, 128>(g, p, s);
  return RGNN_E_UNSUPPORTED;
}

}  // namespace rgnn
