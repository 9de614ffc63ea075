// gemm_fwd_tf32x3.cu -- typed grouped GEMM of the fp32 layer on the tensor cores (3xTF32).
//
//   Z[p, :] = X[gather(p), :] . W_{r(p)}   for every 128-row tile (r, row0, row1)
//   epilogue: Z *= row_scale[p] (RGCN 1/c), s_src[p] = Z[p] . A[r, 0] (RGAT)
//
// The segment-MM of gemm_tc.cu (gather list P:628-633) with fp32 operands.  tcgen05
// kind::tf32 multiplies 10-bit mantissas, so both operands are split x = hi + lo (hi = tf32(x),
// lo = tf32(x - hi), rounded to nearest) and the tile is accumulated as hi.hi + hi.lo + lo.hi in
// TMEM (fp32): about 3 2^-22 relative per product (same scheme as gemm_dw_tf32.cu).
//
// Shared memory: W_r^T hi and lo stay resident (2 N K 4 bytes: 128 KB at d = 128, reloaded by TMA
// only when the relation changes), so the X tile is staged one 32-feature K-block (a 128-byte
// swizzle line per row) at a time: a stage = 128 rows x 32 features, hi + lo = 32 KB.  The
// producers split while staging, so they load with plain 16-byte loads into registers (the next
// stage's loads are issued before the current stage is written: two stages in flight per thread)
// and store hi and lo into the K-major 128B-swizzled layout.
//
// Persistent, one CTA per SM, 416 threads:
//   warp 0     TMEM allocator, MMA issuer (12 MMAs per K-block), W hi/lo TMA loads
//   warps 1-4  epilogue: tcgen05.ld -> scale, s_src dot, fp32 rows to global
//   warps 5-12 two producer groups; group g fills the stages of iterations g, g+2, ...
// Two TMEM accumulators: tile i+1's MMAs overlap tile i's epilogue.
#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

template <int K, int N>
struct F3Cfg {
  static constexpr int M = 128;
  static constexpr int KB = K / 32;                              // 128-byte K-blocks per row
  static constexpr int A_BYTES = M * 128;                        // one K-block of the tile (hi or lo)
  static constexpr int B_BYTES = N * K * 4;                      // W_r^T (hi or lo)
  static constexpr int FIXED = 1024 + 2 * B_BYTES + 512;
  static constexpr int STAGES_FIT = (227 * 1024 - FIXED) / (2 * A_BYTES);
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr int NG = 2;                                   // producer groups
  static constexpr int SMEM = 1024 + STAGES * 2 * A_BYTES + 2 * B_BYTES + 512;
  static constexpr int THREADS = 32 * (1 + 4 + 4 * NG);
  static constexpr int NCOLS = (2 * N) <= 32 ? 32 : (2 * N) <= 64 ? 64 : (2 * N) <= 128 ? 128 : 256;
  static constexpr uint32_t IDESC = tc::idesc_tf32(128, N);
  static_assert(STAGES >= 2 && SMEM <= 227 * 1024, "3xTF32 GEMM smem");
};

struct F3Params {
  const Tile* tiles;
  int64_t num_tiles, rows, gofs;
  const int32_t* gather;
  const float* X;
  float* Z;
  const float* row_scale;
  const float* A;
  float* s_src;
};

template <int K, int N>
__global__ void __launch_bounds__(F3Cfg<K, N>::THREADS, 1)
    k_gemm_fwd_tf32x3(const __grid_constant__ CUtensorMap whi, const __grid_constant__ CUtensorMap wlo, F3Params pr) {
  using C = F3Cfg<K, N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sBh = smem;
  uint8_t* sBl = sBh + C::B_BYTES;
  uint8_t* sA = sBl + C::B_BYTES;  // stage s: hi at sA + 2 s A_BYTES, lo right after
  uint64_t* bar = reinterpret_cast<uint64_t*>(sA + C::STAGES * 2 * C::A_BYTES);
  uint64_t* full = bar;
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* b_full = acc_empty + 2;
  uint64_t* b_free = b_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = pr.tiles ? pr.num_tiles : (pr.rows + C::M - 1) / C::M;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per, t1 = min(ntiles, t0 + per);
  const int64_t nt = t1 > t0 ? t1 - t0 : 0;
  const int64_t nit = nt * C::KB;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) { tc::mbar_init(&full[i], 4); tc::mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(&acc_full[i], 1); tc::mbar_init(&acc_empty[i], 4); }
    tc::mbar_init(b_full, 1);
    tc::mbar_init(b_free, 1);
    tc::mbar_fence_init();
    tc::tma_prefetch_desc(&whi);
    tc::tma_prefetch_desc(&wlo);
  }
  if (warp == 0) {
    __syncwarp();
    tc::tmem_alloc<C::NCOLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto tile_of = [&](int64_t t, int& r, int& row0, int& row1) {
    if (pr.tiles) { const Tile tl = pr.tiles[t]; r = tl.r; row0 = tl.row0; row1 = tl.row1; }
    else { r = 0; row0 = (int)(t * C::M); row1 = (int)min(pr.rows, (int64_t)row0 + C::M); }
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer + W loads
    int cur_r = -1;
    uint32_t nload = 0, nfree = 0;
    for (int64_t tl = 0; tl < nt; ++tl) {
      int r, row0, row1;
      tile_of(t0 + tl, r, row0, row1);
      if (r != cur_r) {
        if (cur_r >= 0) {  // every MMA reading the old W has completed before TMA overwrites it
          if (lane == 0) tc::umma_commit(b_free);
          tc::mbar_wait(b_free, nfree & 1);
          ++nfree;
        }
        if (lane == 0) {
          tc::mbar_expect_tx(b_full, 2 * C::B_BYTES);
#pragma unroll
          for (int kb = 0; kb < C::KB; ++kb) {
            tc::tma_load_2d(sBh + kb * N * 128, &whi, b_full, kb * 32, r * N);
            tc::tma_load_2d(sBl + kb * N * 128, &wlo, b_full, kb * 32, r * N);
          }
        }
        tc::mbar_wait(b_full, nload & 1);
        ++nload;
        cur_r = r;
      }
      const int acc = (int)(tl & 1);
      if (tl >= 2) tc::mbar_wait(&acc_empty[acc], (uint32_t)((tl >> 1) - 1) & 1);
      tc::tc_fence_after();
      for (int kb = 0; kb < C::KB; ++kb) {
        const int64_t it = tl * C::KB + kb;
        const int st = (int)(it % C::STAGES);
        tc::mbar_wait(&full[st], (uint32_t)(it / C::STAGES) & 1);
        tc::tc_fence_after();
        if (lane == 0) {
          const uint32_t ah = tc::smem_u32(sA + st * 2 * C::A_BYTES), al = ah + C::A_BYTES;
          const uint32_t bh = tc::smem_u32(sBh + kb * N * 128), bl = tc::smem_u32(sBl + kb * N * 128);
          const uint32_t d = tmem + acc * N;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {  // 8 tf32 = 32 bytes per MMA
            const uint64_t dah = tc::umma_desc(ah + ks * 32, 16, 1024, 2u);
            const uint64_t dal = tc::umma_desc(al + ks * 32, 16, 1024, 2u);
            const uint64_t dbh = tc::umma_desc(bh + ks * 32, 16, 1024, 2u);
            const uint64_t dbl = tc::umma_desc(bl + ks * 32, 16, 1024, 2u);
            tc::umma_tf32(d, dah, dbh, C::IDESC, (kb > 0 || ks > 0) ? 1u : 0u);
            tc::umma_tf32(d, dah, dbl, C::IDESC, 1u);
            tc::umma_tf32(d, dal, dbh, C::IDESC, 1u);
          }
          tc::umma_commit(&empty[st]);
          if (kb == C::KB - 1) tc::umma_commit(&acc_full[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp <= 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int row = q * 32 + lane;
    for (int64_t tl = 0; tl < nt; ++tl) {
      int r, row0, row1;
      tile_of(t0 + tl, r, row0, row1);
      const int acc = (int)(tl & 1);
      const int p = row0 + row;
      const bool valid = p < row1;
      const float scale = (pr.row_scale && valid) ? __ldg(pr.row_scale + p) : 1.f;
      const float* a0 = pr.A ? pr.A + (size_t)r * 2 * N : nullptr;
      tc::mbar_wait(&acc_full[acc], (uint32_t)(tl >> 1) & 1);
      tc::tc_fence_after();
      float sdot = 0.f;
      float* zrow = pr.Z + (size_t)p * N;
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * N + c0, v);
        tc::tmem_ld_wait();
        if (a0) {
#pragma unroll
          for (int j = 0; j < 16; ++j) sdot = fmaf(__uint_as_float(v[j]), __ldg(a0 + c0 + j), sdot);
        }
        if (valid) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            stg16(zrow + c0 + j, make_uint4(__float_as_uint(__uint_as_float(v[j]) * scale),
                                            __float_as_uint(__uint_as_float(v[j + 1]) * scale),
                                            __float_as_uint(__uint_as_float(v[j + 2]) * scale),
                                            __float_as_uint(__uint_as_float(v[j + 3]) * scale)));
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[acc]);
      if (pr.s_src && valid) pr.s_src[p] = sdot;
    }
  } else {
    // ---------------------------------------------------------------- producers
    const int pg = (warp - 5) >> 2, wq = (warp - 5) & 3;
    // thread (wq, lane) stages rows 16 j + 4 wq + lane / 8 (j = 0..7), 16-byte chunk lane % 8 of the
    // K-block; lane L holds the X row index of tile row 16 (L % 8) + 4 wq + L / 8
    const int myrow = 16 * (lane & 7) + 4 * wq + (lane >> 3);
    const int chunk = lane & 7;
    auto load_idx = [&](int64_t tl, int& row1_out, int& row0_out) -> int {
      int r, row0, row1;
      tile_of(t0 + tl, r, row0, row1);
      row0_out = row0; row1_out = row1;
      const int p = min(row0 + myrow, row1 - 1);  // rows past row1 re-read a valid row, never stored
      return pr.gather ? __ldg(pr.gather + p) : (int)(pr.gofs + p);
    };
    auto issue = [&](int64_t it, int idx, int row0, int row1, float4* v) {
      const int kb = (int)(it % C::KB);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int rr = 16 * j + 4 * wq + (lane >> 3);
        const int xr = __shfl_sync(0xffffffffu, idx, (lane & ~7) | j);
        v[j] = row0 + rr < row1 ? __ldg(reinterpret_cast<const float4*>(pr.X + (size_t)xr * K + kb * 32) + chunk)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    int64_t itile = -1;
    int idx = 0, row0 = 0, row1 = 0;
    float4 cur[8], nxt[8];
    int64_t it = pg;
    if (it < nit) {
      itile = it / C::KB;
      idx = load_idx(itile, row1, row0);
      issue(it, idx, row0, row1, cur);
    }
    for (; it < nit; it += C::NG) {
      const int64_t in = it + C::NG;
      if (in < nit) {  // the next stage's loads go out before this stage is written
        if (in / C::KB != itile) {
          itile = in / C::KB;
          idx = load_idx(itile, row1, row0);
        }
        issue(in, idx, row0, row1, nxt);
      }
      const int st = (int)(it % C::STAGES);
      const uint32_t use = (uint32_t)(it / C::STAGES);
      if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
      uint8_t* hi = sA + st * 2 * C::A_BYTES;
      uint8_t* lo = hi + C::A_BYTES;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int rr = 16 * j + 4 * wq + (lane >> 3);
        const uint32_t off = (uint32_t)rr * 128u + (uint32_t)((chunk ^ (rr & 7)) << 4);
        const float4 x = cur[j];
        float4 h, l;
        tc::tf32_split(x.x, h.x, l.x); tc::tf32_split(x.y, h.y, l.y);
        tc::tf32_split(x.z, h.z, l.z); tc::tf32_split(x.w, h.w, l.w);
        *reinterpret_cast<float4*>(hi + off) = h;
        *reinterpret_cast<float4*>(lo + off) = l;
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[st]);
#pragma unroll
      for (int j = 0; j < 8; ++j) cur[j] = nxt[j];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

// W [num_w, K, N] -> W^T hi and lo [num_w, N, K] (tc::tf32_split)
__global__ void k_w_split_tf32(int num_w, int K, int N, const float* __restrict__ W, float* __restrict__ hi,
                               float* __restrict__ lo) {
  const int64_t total = (int64_t)num_w * K * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ((int64_t)K * N);
    const int rem = (int)(i - r * K * N), n = rem / K, k = rem - n * K;  // output index (r, n, k)
    float h, l;
    tc::tf32_split(W[(r * K + k) * N + n], h, l);
    hi[i] = h;
    lo[i] = l;
  }
}

template <int K, int N>
static rgnn_status gemm_fwd_tf32x3(const GemmFwdArgs& a, cudaStream_t s) {
  tc::watchdog_init();
  using C = F3Cfg<K, N>;
  const int64_t ntiles = a.tiles ? a.num_tiles : (a.rows + C::M - 1) / C::M;
  if (ntiles == 0) return RGNN_OK;
  if (!a.wt_bf16) return set_error(RGNN_E_INVALID_ARG, "3xTF32 GEMM: no weight workspace");
  float* hi = static_cast<float*>(a.wt_bf16);
  const int64_t nw = (int64_t)a.num_w * K * N;
  float* lo = hi + nw;
  RGNN_LAUNCH(k_w_split_tf32, (unsigned)std::max<int64_t>(1, std::min<int64_t>((nw + 255) / 256, 4096)), 256, 0, s,
              a.num_w, K, N, a.W, hi, lo);
  CUtensorMap mh, ml;
  RGNN_TRY(make_tmap_2d_f32(&mh, hi, K, (uint64_t)a.num_w * N, K * 4, 32, N, 128));
  RGNN_TRY(make_tmap_2d_f32(&ml, lo, K, (uint64_t)a.num_w * N, K * 4, 32, N, 128));
  auto kern = k_gemm_fwd_tf32x3<K, N>;
  RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  int dev, sms;
  RGNN_CUDA_TRY(cudaGetDevice(&dev));
  RGNN_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  F3Params pr{a.tiles, a.num_tiles, a.rows, a.gofs, a.gather, static_cast<const float*>(a.X),
              static_cast<float*>(a.Z), a.row_scale, a.A, a.s_src};
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, sms);
  RGNN_LAUNCH(kern, grid, C::THREADS, C::SMEM, s, mh, ml, pr);
  return RGNN_OK;
}

bool tc_disabled();

rgnn_status launch_gemm_fwd_tf32x3(int K, int N, const GemmFwdArgs& a, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  return RGNN_DISPATCH_KN(K, N, [&] { return gemm_fwd_tf32x3<kK, kN>(a, s); });
}

}  // namespace rgnn
