// gemm_dw_tf32.cu -- segmented weight-gradient GEMM of the fp32 layer on the tensor cores (3xTF32).
//
//   part[c] = sum_{p in chunk c} X[g(p)]^T B[p]      (d_in x d_out, fp32)
//   RGAT also: bvec[c] = sum_p dpre[p] X[g(p)]       (for dA[r,0] = b_r W_r)
//
// The same split-K chunks as gemm_dw_tc.cu (dW_r = sum over the relation's edges of
// x_src^T dZ_e), for fp32 operands.  tcgen05 kind::tf32 multiplies 10-bit mantissas, so each operand
// is split x = hi + lo with hi = tf32(x), lo = tf32(x - hi) (round to nearest: |x - hi - lo| <= 2^-22
// |x|), and the product is taken as hi.hi + hi.lo + lo.hi ("3xTF32"; the dropped lo.lo term is below
// 2^-22 |x y|, so a product is good to about 3 2^-22 ~ 7e-7 relative, against 6e-8 for an fp32 FMA).  B[p] is dZ[p] (RGAT walk output) or
// bscale[p] * Bg[bgather[p]] (RGCN: G_dst / c), gathered here, so no dZ is materialised for RGCN.
//
// The reduction runs over positions, so both operands are MN-major (features contiguous, as the
// rows lie in HBM).  tf32 MN-major operands take the SWIZZLE_128B_BASE32B layout: per 32-feature
// block, one 128-byte line per position, the 32-byte chunks of a line XOR-ed with position % 4
// (byte-address bits [5,7) ^= bits [7,9)), 4-position atoms at SBO = 512 B, feature blocks at LBO.
// The producers load rows coalesced (D/4 lanes x 16 bytes per row), split them and store hi and lo
// with 16-byte stores.  RGNN_DW3_KMAJOR=1 selects the first version, which transposed into K-major
// lines instead (a lane per position, scalar stores; measured slower, kept for comparison).
//
// Warp roles (416 threads): warp 0 TMEM allocator + MMA issuer (12 MMAs per 32-position stage,
// +2 for bvec: dpre hi and lo are rows 0 and 1 of a 16-row operand, summed in the epilogue),
// warps 1-12 three producer groups of four warps, group g filling stage g for iterations g, g+3,
// ... (a warp covers a quarter of the features of 32 positions); group 0 then runs the epilogue
// (tcgen05.ld -> fp32 partials).  Partials are reduced in fixed order by k_dw_reduce (deterministic).
#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

template <int K, int N>
struct Dw3Cfg {
  static constexpr int P = 32;                                  // positions per stage
  static constexpr int A_BYTES = K * 128;                       // X^T part: K lines of 32 fp32
  static constexpr int B_BYTES = N * 128;                       // B^T part: N lines
  static constexpr int C_BYTES = 16 * 128;                      // dpre operand (rows 0, 1)
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES + C_BYTES;  // hi, lo, hi, lo, dpre
  static constexpr int NG = 3;                                  // producer groups = stages
  static constexpr int SMEM = 1024 + NG * STAGE + 256;
  static constexpr int THREADS = 32 * (1 + 4 * NG);
  static constexpr int XV = K / 16, BV = N / 16;                // float4 per lane per stage (a quarter)
  static constexpr int NCOLS = (N + 16) <= 32 ? 32 : (N + 16) <= 64 ? 64 : (N + 16) <= 128 ? 128 : 256;
  static constexpr uint32_t IDESC = tc::idesc_tf32(K, N);
  static constexpr uint32_t IDESC_C = tc::idesc_tf32(K, 16);
  static_assert(SMEM <= 227 * 1024, "dW 3xTF32 smem");
};

template <int K, int N, bool BVEC, bool MN>
__global__ void __launch_bounds__(Dw3Cfg<K, N>::THREADS, 1) k_gemm_dw_tf32x3(GemmDwArgs a) {
  using C = Dw3Cfg<K, N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NG * C::STAGE);
  uint64_t* empty = full + C::NG;
  uint64_t* acc_full = empty + C::NG;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  auto sAh = [&](int s) { return smem + s * C::STAGE; };
  auto sAl = [&](int s) { return smem + s * C::STAGE + C::A_BYTES; };
  auto sBh = [&](int s) { return smem + s * C::STAGE + 2 * C::A_BYTES; };
  auto sBl = [&](int s) { return smem + s * C::STAGE + 2 * C::A_BYTES + C::B_BYTES; };
  auto sC = [&](int s) { return smem + s * C::STAGE + 2 * C::A_BYTES + 2 * C::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int row0, row1;
  if (a.chunks) { Tile t = a.chunks[blockIdx.x]; row0 = t.row0; row1 = t.row1; }
  else { row0 = (int)(blockIdx.x * a.chunk_rows); row1 = (int)min(a.rows, (int64_t)row0 + a.chunk_rows); }
  const int nsub = (row1 - row0 + C::P - 1) / C::P;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NG; ++i) { tc::mbar_init(&full[i], 4); tc::mbar_init(&empty[i], 1); }
    tc::mbar_init(acc_full, 1);
    tc::mbar_fence_init();
  }
  if (BVEC) {  // rows 2..15 of the dpre operand stay zero for the whole kernel
    for (int i = threadIdx.x; i < C::NG * 14 * 8; i += blockDim.x) {
      const int s = i / (14 * 8), o = i % (14 * 8);
      reinterpret_cast<uint4*>(sC(s) + 2 * 128)[o] = make_uint4(0, 0, 0, 0);
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

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::NG;
      tc::mbar_wait(&full[st], (uint32_t)(it / C::NG) & 1);
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t ah = tc::smem_u32(sAh(st)), al = tc::smem_u32(sAl(st));
        const uint32_t bh = tc::smem_u32(sBh(st)), bl = tc::smem_u32(sBl(st)), c0 = tc::smem_u32(sC(st));
#pragma unroll
        for (int ks = 0; ks < C::P / 8; ++ks) {  // 8 positions = 32 bytes of each K-major line
          const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
          // MN-major (SWIZZLE_128B_BASE32B): 8 positions = two 4-position atoms of 512 B, 32-feature
          // blocks at LBO = P * 128, atoms at SBO = 512; K-major: 8 positions = 32 bytes of each line
          const uint32_t ko = MN ? ks * 1024 : ks * 32;
          const uint32_t lbo = MN ? C::P * 128 : 16, sbo = MN ? 512 : 1024, lay = MN ? 1u : 2u;
          const uint64_t dah = tc::umma_desc(ah + ko, lbo, sbo, lay);
          const uint64_t dal = tc::umma_desc(al + ko, lbo, sbo, lay);
          const uint64_t dbh = tc::umma_desc(bh + ko, lbo, sbo, lay);
          const uint64_t dbl = tc::umma_desc(bl + ko, lbo, sbo, lay);
          constexpr uint32_t ID = MN ? (C::IDESC | (1u << 15) | (1u << 16)) : C::IDESC;
          tc::umma_tf32(tmem, dah, dbh, ID, acc);
          tc::umma_tf32(tmem, dah, dbl, ID, 1u);
          tc::umma_tf32(tmem, dal, dbh, ID, 1u);
          if (BVEC) {  // dpre operand stays K-major
            const uint64_t dc = tc::umma_desc(c0 + ks * 32, 16, 1024, 2u);
            constexpr uint32_t IDC = MN ? (C::IDESC_C | (1u << 15)) : C::IDESC_C;
            tc::umma_tf32(tmem + N, dah, dc, IDC, acc);
            tc::umma_tf32(tmem + N, dal, dc, IDC, 1u);
          }
        }
        tc::umma_commit(&empty[st]);
        if (it == nsub - 1) tc::umma_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ producers
    const int pg = (warp - 1) >> 2, wq = (warp - 1) & 3;  // group, quarter of the features
    const float* X = static_cast<const float*>(a.X);
    const float* Bz = static_cast<const float*>(a.Bz);
    // position p's X row and B row (-1: past the chunk)
    auto rows_of = [&](int it, int64_t& xr, int64_t& br, float& sc) {
      const int p = row0 + it * C::P + lane;
      if (it >= nsub || p >= row1) { xr = -1; br = -1; sc = 0.f; return; }
      xr = a.gather ? (int64_t)__ldg(a.gather + p) : a.gofs + p;
      br = Bz ? (int64_t)p : (a.bgather ? (int64_t)__ldg(a.bgather + p) : (int64_t)p);
      sc = (Bz || !a.bscale) ? 1.f : __ldg(a.bscale + p);
    };
    int64_t xr, br;
    float sc;
    rows_of(pg, xr, br, sc);
    const uint32_t cpos = (uint32_t)(((lane >> 2) << 4) | ((lane & 3) << 2));  // K-major: unswizzled byte of the lane
    for (int it = pg; it < nsub; it += C::NG) {
      const int st = pg;
      float dp = 0.f;
      if (BVEC && wq == 0) {
        const int p = row0 + it * C::P + lane;
        dp = xr >= 0 ? __ldg(a.dpre + p) : 0.f;
      }
      uint8_t *ah = sAh(st), *al = sAl(st), *bh = sBh(st), *bl = sBl(st);
      if constexpr (MN) {
        // MN-major: warp wq stages positions 8 wq .. 8 wq + 7; a row of D features is D/4 lanes x 16 bytes
        // (coalesced), stored as 128-byte lines per (32-feature block, position), 32-byte chunks swizzled
        // by position % 4 (SWIZZLE_128B_BASE32B)
        constexpr int XL = K / 4, XR = 32 / XL, XI = 8 / XR;  // lanes per X row, rows per load, loads
        constexpr int BL = N / 4, BR = 32 / BL, BI = 8 / BR;
        float4 xv[XI], bv[BI];
        float bsc[BI];
#pragma unroll
        for (int i = 0; i < XI; ++i) {
          const int pp = wq * 8 + i * XR + lane / XL;
          const int64_t r = __shfl_sync(0xffffffffu, xr, pp);
          xv[i] = r >= 0 ? __ldg(reinterpret_cast<const float4*>(X + r * K) + lane % XL) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < BI; ++i) {
          const int pp = wq * 8 + i * BR + lane / BL;
          const int64_t r = __shfl_sync(0xffffffffu, br, pp);
          bsc[i] = __shfl_sync(0xffffffffu, sc, pp);
          const float* brow = Bz ? Bz + r * N : a.Bg + r * N;
          bv[i] = r >= 0 ? __ldg(reinterpret_cast<const float4*>(brow) + lane % BL) : make_float4(0, 0, 0, 0);
        }
        rows_of(it + C::NG, xr, br, sc);  // next iteration's indices, in flight under this one's stores
        const uint32_t use = (uint32_t)(it / C::NG);
        if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
        auto put4 = [&](uint8_t* hi, uint8_t* lo, int pp, int l, float4 x) {
          const uint32_t off = (uint32_t)(l >> 3) * (C::P * 128u) + (uint32_t)pp * 128u +
                               (((uint32_t)(((l & 7) >> 1) ^ (pp & 3))) << 5) + ((uint32_t)(l & 1) << 4);
          float4 h, m;
          tc::tf32_split(x.x, h.x, m.x); tc::tf32_split(x.y, h.y, m.y);
          tc::tf32_split(x.z, h.z, m.z); tc::tf32_split(x.w, h.w, m.w);
          *reinterpret_cast<float4*>(hi + off) = h;
          *reinterpret_cast<float4*>(lo + off) = m;
        };
#pragma unroll
        for (int i = 0; i < XI; ++i) put4(ah, al, wq * 8 + i * XR + lane / XL, lane % XL, xv[i]);
#pragma unroll
        for (int i = 0; i < BI; ++i) {
          const float4 y = bv[i];
          const float c = bsc[i];
          put4(bh, bl, wq * 8 + i * BR + lane / BL, lane % BL, make_float4(y.x * c, y.y * c, y.z * c, y.w * c));
        }
      } else {
      float4 xv[C::XV], bv[C::BV];
      const bool valid = xr >= 0;
#pragma unroll
      for (int j = 0; j < C::XV; ++j)
        xv[j] = valid ? __ldg(reinterpret_cast<const float4*>(X + xr * K + wq * (K / 4)) + j) : make_float4(0, 0, 0, 0);
      const float* brow = Bz ? Bz + br * N : a.Bg + br * N;
#pragma unroll
      for (int j = 0; j < C::BV; ++j)
        bv[j] = valid ? __ldg(reinterpret_cast<const float4*>(brow + wq * (N / 4)) + j) : make_float4(0, 0, 0, 0);
      const float scale = sc;
      rows_of(it + C::NG, xr, br, sc);  // next iteration's indices, in flight under this one's stores
      const uint32_t use = (uint32_t)(it / C::NG);
      if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
      auto put = [&](uint8_t* hi, uint8_t* lo, int r, float v) {
        float h, l;
        tc::tf32_split(v, h, l);
        const uint32_t off = (uint32_t)r * 128u + (cpos ^ ((uint32_t)(r & 7) << 4));
        *reinterpret_cast<float*>(hi + off) = h;
        *reinterpret_cast<float*>(lo + off) = l;
      };
#pragma unroll
      for (int j = 0; j < C::XV; ++j) {
        const int r = wq * (K / 4) + 4 * j;
        put(ah, al, r, xv[j].x); put(ah, al, r + 1, xv[j].y); put(ah, al, r + 2, xv[j].z); put(ah, al, r + 3, xv[j].w);
      }
#pragma unroll
      for (int j = 0; j < C::BV; ++j) {
        const int r = wq * (N / 4) + 4 * j;
        put(bh, bl, r, bv[j].x * scale); put(bh, bl, r + 1, bv[j].y * scale);
        put(bh, bl, r + 2, bv[j].z * scale); put(bh, bl, r + 3, bv[j].w * scale);
      }
      }
      if (BVEC && wq == 0) {  // row 0 = hi, row 1 = lo of dpre
        uint8_t* c = sC(st);
        float h, l;
        tc::tf32_split(dp, h, l);
        *reinterpret_cast<float*>(c + cpos) = h;
        *reinterpret_cast<float*>(c + 128 + (cpos ^ 16u)) = l;
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[st]);
    }
    if (warp <= 4) {
      // ---------------------------------------------------------- epilogue (producer group 0)
      const int q = warp & 3;
      if (nsub > 0) {
        tc::mbar_wait(acc_full, 0);
        tc::tc_fence_after();
      }
      // M=128: row = lane quarter q * 32 + lane; M=64: rows 16q..16q+15 live in lanes 0..15 of quarter q
      const int row = K == 128 ? q * 32 + lane : q * 16 + lane;
      const bool rvalid = K == 128 || lane < 16;
      float* out = a.part + (size_t)blockIdx.x * (K * N + K);
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        if (nsub > 0) {
          tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
          tc::tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0u;
        }
        if (rvalid) {
          float4* o = reinterpret_cast<float4*>(out + (size_t)row * N + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            o[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                               __uint_as_float(v[4 * j + 3]));
        }
      }
      float bv = 0.f;
      if (BVEC && nsub > 0) {
        uint32_t v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + N, v);
        tc::tmem_ld_wait();
        bv = __uint_as_float(v[0]) + __uint_as_float(v[1]);  // dpre hi column + dpre lo column
      }
      if (rvalid) out[K * N + row] = bv;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

template <int K, int N>
static rgnn_status gemm_dw_tf32x3(const GemmDwArgs& a, cudaStream_t s) {
  tc::watchdog_init();
  using C = Dw3Cfg<K, N>;
  if (a.num_chunks == 0) return RGNN_OK;
  if (!a.Bz && !a.Bg) return set_error(RGNN_E_INVALID_ARG, "dW GEMM: no B operand");
  static const bool kmajor = getenv("RGNN_DW3_KMAJOR") && atoi(getenv("RGNN_DW3_KMAJOR")) != 0;
  auto go = [&](auto kern) -> rgnn_status {
    RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    RGNN_LAUNCH(kern, (unsigned)a.num_chunks, C::THREADS, C::SMEM, s, a);
    return RGNN_OK;
  };
  if (a.dpre) return kmajor ? go(k_gemm_dw_tf32x3<K, N, true, false>) : go(k_gemm_dw_tf32x3<K, N, true, true>);
  return kmajor ? go(k_gemm_dw_tf32x3<K, N, false, false>) : go(k_gemm_dw_tf32x3<K, N, false, true>);
}

bool tc_disabled();

rgnn_status launch_gemm_dw_tf32x3(int K, int N, const GemmDwArgs& a, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  if (K == 64 && N == 32) return gemm_dw_tf32x3<64, 32>(a, s);
  if (K == 64 && N == 64) return gemm_dw_tf32x3<64, 64>(a, s);
  if (K == 64 && N == 128) return gemm_dw_tf32x3<64, 128>(a, s);
  if (K == 128 && N == 32) return gemm_dw_tf32x3<128, 32>(a, s);
  if (K == 128 && N == 64) return gemm_dw_tf32x3<128, 64>(a, s);
  if (K == 128 && N == 128) return gemm_dw_tf32x3<128, 128>(a, s);
  return RGNN_E_UNSUPPORTED;  // d_in = 32: UMMA M=32 does not exist for cta_group::1
}

}  // namespace rgnn
