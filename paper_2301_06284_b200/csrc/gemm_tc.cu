// gemm_tc.cu -- typed grouped GEMM on the 5th-generation tensor cores (bf16 path).
//
//   Z[p, :] = X[src_s[p], :] . W_{r(p)}      for every 128-row tile (r, row0, row1)
//
// Segment MM (Sec. 2.2): tiles never straddle relations, one
// bf16 copy of W_r per relation (never replicated per edge), X rows
// gathered on load (the GEMM template's gather list) by 16-byte
// cp.async, accumulators in TMEM, epilogue fused: RGAT source score
// s_src[p] = A[r,0] . Z_fp32[p] and RGCN per-row 1/c ("per-row
// scalar ... applied to A tiles"), bf16 Z written through an XOR-swizzled smem
// stage with coalesced 16-byte stores (rows beyond row1 are never written).
//
// Persistent, warp specialised, one CTA per SM:
//   warp 0    TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=d_out,
//             K-steps of 16), commits to the smem-empty / accumulator-full barriers
//   warps 1-4 producers: X rows gathered with 16-byte cp.async straight into the
//             128B-swizzled K-major layout (r4 profile: TMA tile::gather4 issued
//             ~1 op / 100 cycles / SM and starved the MMA), W_r by TMA into a
//             2-slot ring reloaded only when the relation changes
//   warps 5-8 epilogue: tcgen05.ld (32 lanes x 16 columns) -> fp32 math -> bf16
// TMEM holds two accumulators (tile i+1's MMAs overlap tile i's epilogue).
#include <cudaTypedefs.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static rgnn_status make_tmap_2d(CUtensorMapDataType dt, CUtensorMap* map, const void* base, uint64_t cols,
                                uint64_t rows, uint64_t pitch_bytes, uint32_t box_cols, uint32_t box_rows,
                                int swizzle_bytes);
rgnn_status make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                              uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
  return make_tmap_2d(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, map, base, cols, rows, pitch_bytes, box_cols, box_rows,
                      swizzle_bytes);
}
rgnn_status make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                             uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
  return make_tmap_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, map, base, cols, rows, pitch_bytes, box_cols, box_rows,
                      swizzle_bytes);
}
static rgnn_status make_tmap_2d(CUtensorMapDataType dt, CUtensorMap* map, const void* base, uint64_t cols,
                                uint64_t rows, uint64_t pitch_bytes, uint32_t box_cols, uint32_t box_rows,
                                int swizzle_bytes) {
  auto fn = encode_fn();
  if (!fn) return set_error(RGNN_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(RGNN_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RGNN_OK;
}

// W [R, K, N] fp32 -> Wt [R, N, K] bf16 (RNE): the K-major B operand.
__global__ void k_w_to_bf16_t(int R, int K, int N, const float* __restrict__ W, __nv_bfloat16* __restrict__ Wt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)R * K * N;
       i += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(i / ((int64_t)K * N));
    int rem = (int)(i - (int64_t)r * K * N);
    int n = rem / K, k = rem - n * K;
    Wt[i] = __float2bfloat16_rn(W[((size_t)r * K + k) * N + n]);
  }
}

template <int K, int N>
struct FwdCfg {
  static constexpr int M = 128;
  static constexpr int RB = (K * 2 < 128) ? K * 2 : 128;    // bytes per row of one swizzle block
  static constexpr int KBLK = (K * 2) / RB;                 // column blocks
  static constexpr int SWZ = RB;                            // 64 or 128 byte swizzle
  static constexpr uint32_t LAYOUT = RB == 128 ? 2u : 4u;   // UMMA layout type
  static constexpr int A_BYTES = M * K * 2;
  static constexpr int B_BYTES = N * K * 2;
#ifndef RGNN_FWD_RING_KB
#define RGNN_FWD_RING_KB 64  // measured: 64 KB of A stages beats 32, 48, 96, 128 (mag, AM, wikikg2)
#endif
#ifndef RGNN_FWD_MINB64
#define RGNN_FWD_MINB64 3  // resident CTAs per SM at d_in, d_out <= 64, with a 32 KB A ring each (measured r02: AM
                           // 0.228 / 0.169 / 0.147 ms and wikikg2 0.602 / 0.444 / 0.375 ms with 1 / 2 / 3 CTAs per SM)
#endif
  static constexpr int MINB = (K <= 64 && N <= 64) ? RGNN_FWD_MINB64 : 1;
  static constexpr int RING_KB = MINB >= 3 ? 32 : RGNN_FWD_RING_KB;
  static constexpr int STAGES = (RING_KB * 1024) / A_BYTES > 8 ? 8 : (RING_KB * 1024) / A_BYTES;
  static constexpr int DEPTH = STAGES - 1;                  // cp.async groups kept in flight per producer thread
  static constexpr int STG_BYTES = M * N * 2;
  static constexpr int NCOLS = (2 * N) <= 32 ? 32 : (2 * N) <= 64 ? 64 : (2 * N) <= 128 ? 128 : 256;
  static constexpr int SMEM0 = 1024 + STAGES * A_BYTES + 2 * B_BYTES + STG_BYTES + N * 4 + 256;
  // tile descriptors of the CTA's range cached in shared memory (up to TCAP, in what is left of
  // 227 KB per SM): every role reads its next tile without a dependent global load
  static constexpr int TCAP_RAW = (227 * 1024 / MINB - 1024 * (MINB - 1) - SMEM0 - 64) / 16;
  // (measured: AM / wikikg2 d = 64 typed GEMM -7%; at d_in = 128 the global descriptor loads are
  // hidden by the longer tiles and the cache costs 7% on ogbn-mag, so it is off there)
  static constexpr int TCAP = K > 64 ? 0 : (TCAP_RAW > 4096 ? 4096 : (TCAP_RAW < 0 ? 0 : TCAP_RAW));
  static constexpr int SMEM = SMEM0 + TCAP * 16 + 16;
  static constexpr int THREADS = 288;                       // 1 MMA warp, 4 producer warps, 4 epilogue warps
  static constexpr int CPR = K * 2 / 16;                    // 16-byte chunks per X row
  static constexpr int RPI = 32 / CPR;                      // X rows per warp-wide cp.async
  static constexpr uint32_t IDESC = tc::idesc_bf16(128, N, 0, 0);
};

struct TcFwdParams {
  const Tile* tiles;
  int64_t num_tiles, rows, gofs;
  const int32_t* gather;
  const __nv_bfloat16* X;
  __nv_bfloat16* Z;
  const float* row_scale;
  const float* A;
  float* s_src;
  int tcap;  // tile descriptors cached in shared memory (<= FwdCfg::TCAP; the launch sizes the smem)
};

template <int K, int N, bool F32OUT>
__global__ void __launch_bounds__(288, FwdCfg<K, N>::MINB)
    k_gemm_fwd_tc(const __grid_constant__ CUtensorMap wmap, TcFwdParams pr) {
  using C = FwdCfg<K, N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;
  uint8_t* sStg = sB + 2 * C::B_BYTES;
  float* sA0 = reinterpret_cast<float*>(sStg + C::STG_BYTES);  // A[r,0] of the current relation
  uint64_t* bar = reinterpret_cast<uint64_t*>(sA0 + N);
  uint64_t* a_full = bar;
  uint64_t* a_empty = a_full + C::STAGES;
  uint64_t* b_full = a_empty + C::STAGES;
  uint64_t* b_empty = b_full + 2;
  uint64_t* acc_full = b_empty + 2;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  Tile* sTiles = reinterpret_cast<Tile*>(smem + C::SMEM0 - 1024);  // [TCAP], 16-byte aligned

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = pr.tiles ? pr.num_tiles : (pr.rows + C::M - 1) / C::M;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per, t1 = min(ntiles, t0 + per);
  if (C::TCAP > 0 && pr.tiles)
    for (int64_t i = threadIdx.x; i < t1 - t0 && i < (int64_t)pr.tcap; i += blockDim.x) sTiles[i] = pr.tiles[t0 + i];

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
    __syncwarp();  // .sync.aligned: the warp must be converged (thread 0 initialised the barriers)
    tc::tmem_alloc<C::NCOLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto tile_of = [&](int64_t t, int& r, int& row0, int& row1) {
    if (pr.tiles) {
      Tile tl;
      if constexpr (C::TCAP > 0) tl = t - t0 < pr.tcap ? sTiles[t - t0] : pr.tiles[t];
      else tl = pr.tiles[t];
      r = tl.r; row0 = tl.row0; row1 = tl.row1;
    }
    else { r = 0; row0 = (int)(t * C::M); row1 = (int)min(pr.rows, (int64_t)row0 + C::M); }
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer
    int cur_r = -1, bslot = 1;
    uint32_t buse[2] = {0, 0};
    int64_t it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      if (r != cur_r) {
        if (cur_r >= 0 && lane == 0) tc::umma_commit(&b_empty[bslot]);  // old slot free once its MMAs finish
        bslot ^= 1;
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
        for (int ks = 0; ks < K / 16; ++ks) {
          const int kb = (ks * 32) / C::RB, off = (ks * 32) % C::RB;
          const uint64_t ad = tc::umma_desc(a0 + kb * C::M * C::RB + off, 16, 8 * C::RB, C::LAYOUT);
          const uint64_t bd = tc::umma_desc(b0 + kb * N * C::RB + off, 16, 8 * C::RB, C::LAYOUT);
          tc::umma_bf16(d, ad, bd, C::IDESC, ks > 0 ? 1u : 0u);
        }
        tc::umma_commit(&a_empty[stage]);
        tc::umma_commit(&acc_full[acc]);
      }
      __syncwarp();
    }
  } else if (warp <= 4) {
    // ---------------------------------------------------------------- producers (warps 1..4)
    // X rows gathered with 16-byte cp.async straight into the swizzled K-major layout;
    // each thread keeps DEPTH tiles in flight, then publishes a tile with a proxy
    // fence + mbarrier arrive (128 producer threads per tile).  W_r: TMA, warp 1.
    const int pw = warp - 1;
    int cur_r = -1, bslot = 1;
    uint32_t buse[2] = {0, 0};
    auto load_idx = [&](int64_t t) -> int {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      const int p = min(row0 + pw * 32 + lane, row1 - 1);  // rows past row1 re-read a valid row, never stored
      return pr.gather ? __ldg(pr.gather + p) : (int)(pr.gofs + p);
    };
    int myidx = t0 < t1 ? load_idx(t0) : 0;
    int64_t it = 0, pub = 0;  // tiles [0, pub) published by this thread
    auto flush = [&]() {      // publish every pending tile (before any blocking wait: the MMA may need them)
      tc::cp_async_wait<0>();
      tc::fence_proxy_async_smem();
      for (; pub < it; ++pub) tc::mbar_arrive(&a_full[pub % C::STAGES]);
    };
    for (int64_t t = t0; t < t1; ++t, ++it) {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      const int nidx = t + 1 < t1 ? load_idx(t + 1) : 0;
      if (pw == 0 && r != cur_r) {
        bslot ^= 1;
        if (buse[bslot] > 0) {
          flush();
          tc::mbar_wait(&b_empty[bslot], (buse[bslot] - 1) & 1);
        }
        ++buse[bslot];
        if (lane == 0) {
          tc::mbar_expect_tx(&b_full[bslot], C::B_BYTES);
#pragma unroll
          for (int kb = 0; kb < C::KBLK; ++kb)
            tc::tma_load_2d(sB + bslot * C::B_BYTES + kb * N * C::RB, &wmap, &b_full[bslot], kb * (C::RB / 2), r * N);
        }
        cur_r = r;
      }
      const int stage = (int)(it % C::STAGES);
      const uint32_t use = (uint32_t)(it / C::STAGES);
      if (use > 0) {
        if (pub < it - C::STAGES + 1) flush();  // the stage's previous tile must be published before waiting on it
        tc::mbar_wait(&a_empty[stage], (use - 1) & 1);
      }
      uint8_t* dstA = sA + stage * C::A_BYTES;
#pragma unroll
      for (int i = 0; i < 32 / C::RPI; ++i) {
        const int rr = i * C::RPI + lane / C::CPR;  // row within this warp's 32
        const int c = lane % C::CPR;                // 16-byte chunk of the row
        const int row = pw * 32 + rr;
        const int xr = __shfl_sync(0xffffffffu, myidx, rr);
        const int cb = c % (C::RB / 16), blk = c / (C::RB / 16);
        const int phys = C::RB == 128 ? (cb ^ (row & 7)) : (cb ^ ((row >> 1) & 3));
        tc::cp_async16(dstA + blk * C::M * C::RB + row * C::RB + phys * 16, pr.X + (size_t)xr * K + c * 8);
      }
      tc::cp_async_commit();
      if (it - pub >= C::DEPTH) {  // more than DEPTH tiles pending: the oldest has landed
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
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;          // tile row owned by this thread
    const int et = threadIdx.x - 160;       // 0..127
    constexpr int NCH = N / 8;              // 16-byte chunks per Z row
    constexpr int SWM = (NCH < 8 ? NCH : 8) - 1;
    int cur_r = -1;
    int64_t it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      int r, row0, row1;
      tile_of(t, r, row0, row1);
      const int acc = (int)(it & 1);
      const int p = row0 + row;
      const bool valid = p < row1;
      const float scale = (pr.row_scale && valid) ? __ldg(pr.row_scale + p) : 1.f;
      tc::mbar_wait(&acc_full[acc], (uint32_t)(it >> 1) & 1);
      tc::tc_fence_after();
      if (pr.A && r != cur_r)
        for (int n = et; n < N; n += 128) sA0[n] = __ldg(pr.A + (size_t)r * 2 * N + n);
      cur_r = r;
      tc::named_bar(1, 128);  // previous tile's copy-out done; A[r,0] visible
      uint8_t* srow = sStg + row * (N * 2);
      float sdot = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * N + c0, v);
        tc::tmem_ld_wait();
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
        if (pr.A) {
#pragma unroll
          for (int j = 0; j < 16; ++j) sdot = fmaf(f[j], sA0[c0 + j], sdot);
        }
        if constexpr (F32OUT) {  // fp32 rows straight from the accumulator (no staging)
          if (valid) {
            float* zf = reinterpret_cast<float*>(pr.Z) + (size_t)p * N + c0;
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              stg16(zf + j, make_uint4(__float_as_uint(f[j] * scale), __float_as_uint(f[j + 1] * scale),
                                       __float_as_uint(f[j + 2] * scale), __float_as_uint(f[j + 3] * scale)));
          }
          continue;
        }
        uint4 w0, w1;
        w0.x = tc::pack_bf16(f[0] * scale, f[1] * scale); w0.y = tc::pack_bf16(f[2] * scale, f[3] * scale);
        w0.z = tc::pack_bf16(f[4] * scale, f[5] * scale); w0.w = tc::pack_bf16(f[6] * scale, f[7] * scale);
        w1.x = tc::pack_bf16(f[8] * scale, f[9] * scale); w1.y = tc::pack_bf16(f[10] * scale, f[11] * scale);
        w1.z = tc::pack_bf16(f[12] * scale, f[13] * scale); w1.w = tc::pack_bf16(f[14] * scale, f[15] * scale);
        const int ch = c0 / 8;
        *reinterpret_cast<uint4*>(srow + (((ch) ^ (row & SWM)) * 16)) = w0;
        *reinterpret_cast<uint4*>(srow + (((ch + 1) ^ (row & SWM)) * 16)) = w1;
      }
      // accumulator drained: hand it back to the MMA warp
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[acc]);
      if (pr.s_src && valid) pr.s_src[p] = sdot;
      tc::named_bar(1, 128);
      if constexpr (F32OUT) continue;
      // coalesced copy-out of the valid rows (never past row1: the next segment's rows)
      const int nvalid = row1 - row0;
      for (int i = et; i < nvalid * NCH; i += 128) {
        const int rr = i / NCH, ch = i - rr * NCH;
        const uint4 val = *reinterpret_cast<const uint4*>(sStg + rr * (N * 2) + ((ch ^ (rr & SWM)) * 16));
        *reinterpret_cast<uint4*>(pr.Z + (size_t)(row0 + rr) * N + ch * 8) = val;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

template <int K, int N, bool F32OUT>
static rgnn_status gemm_fwd_tc(const GemmFwdArgs& a, cudaStream_t s) {
  tc::watchdog_init();
  using C = FwdCfg<K, N>;
  const int64_t ntiles = a.tiles ? a.num_tiles : (a.rows + C::M - 1) / C::M;
  if (ntiles == 0) return RGNN_OK;
  auto* wt = static_cast<__nv_bfloat16*>(a.wt_bf16);
  const int64_t nw = (int64_t)a.num_w * K * N;
  RGNN_LAUNCH(k_w_to_bf16_t, (unsigned)std::max<int64_t>(1, std::min<int64_t>((nw + 255) / 256, 4096)), 256, 0, s,
              a.num_w, K, N, a.W, wt);
  CUtensorMap wmap;
  RGNN_TRY(make_tmap_2d_bf16(&wmap, wt, K, (uint64_t)a.num_w * N, K * 2, C::RB / 2, N, C::SWZ));
  auto kern = k_gemm_fwd_tc<K, N, F32OUT>;
  RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  int dev, sms;
  RGNN_CUDA_TRY(cudaGetDevice(&dev));
  RGNN_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * C::MINB);
  const int64_t per = (ntiles + grid - 1) / grid;
  const int tcap = a.tiles ? (int)std::min<int64_t>(per, C::TCAP) : 0;
  TcFwdParams pr{a.tiles, a.num_tiles, a.rows, a.gofs, a.gather, static_cast<const __nv_bfloat16*>(a.X),
                 static_cast<__nv_bfloat16*>(a.Z), a.row_scale, a.A, a.s_src, tcap};
  RGNN_LAUNCH(kern, grid, C::THREADS, C::SMEM0 + tcap * 16 + 16, s, wmap, pr);
  return RGNN_OK;
}

bool tc_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RGNN_DISABLE_TCGEN05");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

rgnn_status launch_gemm_fwd_tc(int K, int N, const GemmFwdArgs& a, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  return RGNN_DISPATCH_KN(K, N, [&] { return gemm_fwd_tc<kK, kN, false>(a, s); });
}

// bf16 operands, fp32 output rows (HGT node-typed linears on the bf16 layer)
rgnn_status launch_gemm_fwd_tc_f32out(int K, int N, const GemmFwdArgs& a, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  return RGNN_DISPATCH_KN(K, N, [&] { return gemm_fwd_tc<kK, kN, true>(a, s); });
}

}  // namespace rgnn
