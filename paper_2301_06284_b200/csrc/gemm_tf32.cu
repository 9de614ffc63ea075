// gemm_tf32.cu -- typed grouped GEMM with fp32 operands on the tensor cores
// (tcgen05.mma kind::tf32, fp32 accumulate in TMEM, fp32 output).
//
//   Z[p, :] = X[gather(p), :] . W_{r(p)}   for every 128-row tile (r, row0, row1)
//
// Same segment-MM structure as gemm_tc.cu (gather list P:628-633),
// for the fp32 GEMMs of the path: the HGT score factors (k, q, k W_{a,r}) and
// the dX run products H = G_v W_r^T.  Operands with bf16 values (X of the bf16
// layer, RNE-rounded weights) are exact in tf32, so those products are exact
// and the accumulation is fp32; fp32 data (G) is truncated to tf32 (10-bit
// mantissa), 4x finer than bf16 (O16 / dX).
//
// Persistent, warp specialised, one CTA per SM, 288 threads:
//   warp 0    TMEM allocator + single-thread MMA issuer (M=128, N=d_out, K-steps of 8)
//   warps 1-4 producers: X rows by 16-byte cp.async into the 128B-swizzled K-major
//             layout; warp 1 also TMA-loads W_r^T (fp32, K-major) into a B ring
//             (2 slots when they fit, else 1), reloaded only when the relation changes
//   warps 5-8 epilogue: tcgen05.ld 32 lanes x 16 columns -> fp32 rows to global
// Two TMEM accumulators: tile i+1's MMAs overlap tile i's epilogue.
#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

template <int K, int N>
struct Tf32Cfg {
  static constexpr int M = 128;
  static constexpr int RB = 128;                            // bytes per row of one swizzle block (32 fp32)
  static constexpr int KBLK = (K * 4) / RB;                 // column blocks
  static constexpr int A_BYTES = M * K * 4;
  static constexpr int B_BYTES = N * K * 4;
  static constexpr int NB = (B_BYTES <= 32 * 1024) ? 2 : 1; // W slots
  static constexpr int STAGES_MAX = (200 * 1024 - NB * B_BYTES) / A_BYTES;
#ifndef RGNN_TF32_SMAX
#define RGNN_TF32_SMAX 6
#endif
  static constexpr int STAGES = STAGES_MAX > RGNN_TF32_SMAX ? RGNN_TF32_SMAX : STAGES_MAX;
  static constexpr int DEPTH = STAGES - 1;
  static constexpr int NCOLS = (2 * N) <= 32 ? 32 : (2 * N) <= 64 ? 64 : (2 * N) <= 128 ? 128 : 256;
  static constexpr int SMEM = 1024 + STAGES * A_BYTES + NB * B_BYTES + 256;
  static constexpr int THREADS = 288;
  static constexpr int CPR = K * 4 / 16;                    // 16-byte chunks per X row
  static constexpr int RPI = CPR >= 32 ? 1 : 32 / CPR;      // X rows per warp-wide cp.async
  static constexpr int CPI = CPR >= 32 ? CPR / 32 : 1;      // cp.async per lane per row (K = 128)
  static constexpr uint32_t IDESC = tc::idesc_tf32(128, N);
  static_assert(STAGES >= 2, "tf32 GEMM smem");
};

struct Tf32Params {
  const Tile* tiles;
  int64_t num_tiles, rows, gofs;
  const int32_t* gather;
  const float* X;
  float* Z;
  int z_bf16;  // store the rows as bf16 (RNE) instead of fp32
};

template <int K, int N>
__global__ void __launch_bounds__(288, 1)
    k_gemm_fwd_tf32(const __grid_constant__ CUtensorMap wmap, Tf32Params pr) {
  using C = Tf32Cfg<K, N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + C::NB * C::B_BYTES);
  uint64_t* a_full = bar;
  uint64_t* a_empty = a_full + C::STAGES;
  uint64_t* b_full = a_empty + C::STAGES;
  uint64_t* b_empty = b_full + 2;
  uint64_t* acc_full = b_empty + 2;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = pr.tiles ? pr.num_tiles : (pr.rows + C::M - 1) / C::M;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per, t1 = min(ntiles, t0 + per);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) { tc::mbar_init(&a_full[i], 128); tc::mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&b_full[i], 1); tc::mbar_init(&b_empty[i], 1);
      tc::mbar_init(&acc_full[i], 1); tc::mbar_init(&acc_empty[i], 4);
    }
    tc::mbar_fence_init();
    tc::tma_prefetch_desc(&wmap);
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
    if (pr.tiles) { Tile tl = pr.tiles[t]; r = tl.r; row0 = tl.row0; row1 = tl.row1; }
    else { r = 0; row0 = (int)(t * C::M); row1 = (int)min(pr.rows, (int64_t)row0 + C::M); }
  };
  auto next_slot = [](int b) { return C::NB == 2 ? (b ^ 1) : 0; };

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer
    int cur_r = -1, bslot = C::NB == 2 ? 1 : 0;
    uint32_t buse[2] = {0, 0};
    int64_t it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      if (r != cur_r) {
        if (cur_r >= 0 && lane == 0) tc::umma_commit(&b_empty[bslot]);  // slot free once its MMAs finish
        bslot = next_slot(bslot);
        tc::mbar_wait(&b_full[bslot], buse[bslot] & 1);
        ++buse[bslot];
        cur_r = r;
      }
      const int stage = (int)(it % C::STAGES);
      const uint32_t use = (uint32_t)(it / C::STAGES);
      const int acc = (int)(it & 1);
      const uint32_t ause = (uint32_t)(it >> 1);
      tc::mbar_wait(&a_full[stage], use & 1);
      if (ause > 0) tc::mbar_wait(&acc_empty[acc], (ause - 1) & 1);
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = tc::smem_u32(sA + stage * C::A_BYTES);
        const uint32_t b0 = tc::smem_u32(sB + bslot * C::B_BYTES);
        const uint32_t d = tmem + acc * N;
#pragma unroll
        for (int ks = 0; ks < K * 4 / 32; ++ks) {  // 8 tf32 = 32 bytes per MMA
          const int kb = (ks * 32) / C::RB, off = (ks * 32) % C::RB;
          const uint64_t ad = tc::umma_desc(a0 + kb * C::M * C::RB + off, 16, 8 * C::RB, 2u);
          const uint64_t bd = tc::umma_desc(b0 + kb * N * C::RB + off, 16, 8 * C::RB, 2u);
          tc::umma_tf32(d, ad, bd, C::IDESC, ks > 0 ? 1u : 0u);
        }
        tc::umma_commit(&a_empty[stage]);
        tc::umma_commit(&acc_full[acc]);
      }
      __syncwarp();
    }
  } else if (warp <= 4) {
    // ---------------------------------------------------------------- producers (warps 1..4)
    const int pw = warp - 1;
    int cur_r = -1, bslot = C::NB == 2 ? 1 : 0;
    uint32_t buse[2] = {0, 0};
    auto load_idx = [&](int64_t t) -> int {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      const int p = min(row0 + pw * 32 + lane, row1 - 1);  // rows past row1 re-read a valid row, never stored
      return pr.gather ? __ldg(pr.gather + p) : (int)(pr.gofs + p);
    };
    int myidx = t0 < t1 ? load_idx(t0) : 0;
    int64_t it = 0, pub = 0;
    auto flush = [&]() {
      tc::cp_async_wait<0>();
      tc::fence_proxy_async_smem();
      for (; pub < it; ++pub) tc::mbar_arrive(&a_full[pub % C::STAGES]);
    };
    for (int64_t t = t0; t < t1; ++t, ++it) {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      const int nidx = t + 1 < t1 ? load_idx(t + 1) : 0;
      if (pw == 0 && r != cur_r) {
        bslot = next_slot(bslot);
        if (buse[bslot] > 0) {
          flush();
          tc::mbar_wait(&b_empty[bslot], (buse[bslot] - 1) & 1);
        }
        ++buse[bslot];
        if (lane == 0) {
          tc::mbar_expect_tx(&b_full[bslot], C::B_BYTES);
#pragma unroll
          for (int kb = 0; kb < C::KBLK; ++kb)
            tc::tma_load_2d(sB + bslot * C::B_BYTES + kb * N * C::RB, &wmap, &b_full[bslot], kb * (C::RB / 4), r * N);
        }
        cur_r = r;
      }
      const int stage = (int)(it % C::STAGES);
      const uint32_t use = (uint32_t)(it / C::STAGES);
      if (use > 0) {
        if (pub < it - C::STAGES + 1) flush();
        tc::mbar_wait(&a_empty[stage], (use - 1) & 1);
      }
      uint8_t* dstA = sA + stage * C::A_BYTES;
#pragma unroll
      for (int i = 0; i < 32 / C::RPI; ++i) {
#pragma unroll
        for (int h = 0; h < C::CPI; ++h) {
          const int rr = i * C::RPI + (C::CPR >= 32 ? 0 : lane / C::CPR);  // row within this warp's 32
          const int c = (C::CPR >= 32 ? h * 32 + lane : lane % C::CPR);    // 16-byte chunk of the row
          const int row = pw * 32 + rr;
          const int xr = __shfl_sync(0xffffffffu, myidx, rr);
          const int cb = c % 8, blk = c / 8;
          tc::cp_async16(dstA + blk * C::M * C::RB + row * C::RB + ((cb ^ (row & 7)) * 16),
                         pr.X + (size_t)xr * K + c * 4);
        }
      }
      tc::cp_async_commit();
      if (it - pub >= C::DEPTH) {
        tc::cp_async_wait<C::DEPTH>();
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&a_full[pub % C::STAGES]);
        ++pub;
      }
      myidx = nidx;
    }
    flush();
  } else {
    // ---------------------------------------------------------------- epilogue (warps 5..8)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int64_t it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      const int acc = (int)(it & 1);
      const int p = row0 + row;
      const bool valid = p < row1;
      tc::mbar_wait(&acc_full[acc], (uint32_t)(it >> 1) & 1);
      tc::tc_fence_after();
      float* zrow = pr.Z + (size_t)p * N;
      __nv_bfloat16* zrow_b = reinterpret_cast<__nv_bfloat16*>(pr.Z) + (size_t)p * N;
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * N + c0, v);
        tc::tmem_ld_wait();
        if (valid) {
          if (pr.z_bf16) {
            uint32_t b[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = tc::pack_bf16(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
            stg16(zrow_b + c0, make_uint4(b[0], b[1], b[2], b[3]));
            stg16(zrow_b + c0 + 8, make_uint4(b[4], b[5], b[6], b[7]));
          } else {
#pragma unroll
            for (int j = 0; j < 16; j += 4) stg16(zrow + c0 + j, make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]));
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[acc]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

bool tc_disabled();

// W [num_w, K, N] fp32 is read as W^T [num_w, N, K] (K-major B operand) from `wt_f32`,
// which the caller fills (launch_transpose_w: RNE-rounded to bf16 values when requested).
template <int K, int N>
static rgnn_status gemm_fwd_tf32(const GemmFwdArgs& a, const float* wt_f32, cudaStream_t s) {
  tc::watchdog_init();
  using C = Tf32Cfg<K, N>;
  const int64_t ntiles = a.tiles ? a.num_tiles : (a.rows + C::M - 1) / C::M;
  if (ntiles == 0) return RGNN_OK;
  CUtensorMap wmap;
  RGNN_TRY(make_tmap_2d_f32(&wmap, wt_f32, K, (uint64_t)a.num_w * N, K * 4, C::RB / 4, N, 128));
  auto kern = k_gemm_fwd_tf32<K, N>;
  RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  int dev, sms;
  RGNN_CUDA_TRY(cudaGetDevice(&dev));
  RGNN_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  Tf32Params pr{a.tiles, a.num_tiles, a.rows, a.gofs, a.gather, static_cast<const float*>(a.X),
                static_cast<float*>(a.Z), a.z_bf16};
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, sms);
  RGNN_LAUNCH(kern, grid, C::THREADS, C::SMEM, s, wmap, pr);
  return RGNN_OK;
}

rgnn_status launch_gemm_fwd_tf32(int K, int N, const GemmFwdArgs& a, const float* wt_f32, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  return RGNN_DISPATCH_KN(K, N, [&] { return gemm_fwd_tf32<kK, kN>(a, wt_f32, s); });
}

}  // namespace rgnn
