// gemm_dw_tc.cu -- segmented weight-gradient GEMM on the tensor cores (bf16 path).
//
//   part[c] = sum_{p in chunk c} X[src_s[p]]^T dZ[p]        (d_in x d_out, fp32)
//   RGAT also: bvec[c] = sum_p dpre[p] X[src_s[p]]          (for dA[r,0] = b_r W_r)
//
// The reduction runs over edges (positions of one relation), so both operands
// are MN-major: A = X rows gathered by TMA tile::gather4 (each edge row is a
// 128-byte swizzle line, features contiguous), B = dZ rows by a tiled TMA load.
// UMMA M = d_in (64 or 128), N = d_out, one MMA per 16 edges.  dpre enters as
// a second, 16-column B operand (no-swizzle core matrices, column 0 = dpre),
// so bvec is column 0 of a second small TMEM accumulator.  A split-K chunk
// (host table, never straddling relations, ~2 per SM) is one CTA; partials are
// reduced in a fixed order by k_dw_reduce (deterministic).  The paper's GEMM
// template loads with "transpose on the fly"; here the transpose is
// the MN-major operand descriptor, no data movement.
//
// Warp roles: warp 0 TMA producer (+ writes the dpre column), warp 1 TMEM
// allocator + MMA issuer (zeroes dZ rows past the chunk end in the last
// stage), warps 2-5 epilogue (tcgen05.ld -> fp32 partials).
#include "kernels.cuh"
#include "tc_common.cuh"

namespace rgnn {

template <int K, int N>
struct DwCfg {
  static constexpr int MT = 128;                                // edges per stage
  static constexpr int A_BYTES = MT * K * 2;                    // X rows
  static constexpr int RBB = (N * 2 < 128) ? N * 2 : 128;       // dZ swizzle line bytes
  static constexpr int NBLK = (N * 2) / RBB;
  static constexpr uint32_t BLAYOUT = RBB == 128 ? 2u : (RBB == 64 ? 4u : 6u);
  static constexpr int B_BYTES = MT * N * 2;
  static constexpr int B2_BYTES = MT * 16 * 2;                  // dpre column operand
  static constexpr int STAGE = A_BYTES + B_BYTES + B2_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE > 6 ? 6 : (200 * 1024) / STAGE;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256;
  static constexpr int NCOLS = (N + 16) <= 32 ? 32 : (N + 16) <= 64 ? 64 : (N + 16) <= 128 ? 128 : 256;
  static constexpr uint32_t IDESC = tc::idesc_bf16(K, N, 1, 1);
  static constexpr uint32_t IDESC_B = tc::idesc_bf16(K, 16, 1, 1);
};

struct TcDwParams {
  const Tile* chunks;
  int64_t rows, chunk_rows, gofs;
  const int32_t* gather;
  const float* dpre;
  float* part;
};

template <int K, int N, bool BVEC>
__global__ void __launch_bounds__(192, 1)
    k_gemm_dw_tc(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap zmap, TcDwParams pr) {
  using C = DwCfg<K, N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* full = bar;
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  auto sA = [&](int s) { return smem + s * C::STAGE; };
  auto sB = [&](int s) { return smem + s * C::STAGE + C::A_BYTES; };
  auto sB2 = [&](int s) { return smem + s * C::STAGE + C::A_BYTES + C::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int row0, row1;
  if (pr.chunks) { Tile t = pr.chunks[blockIdx.x]; row0 = t.row0; row1 = t.row1; }
  else { row0 = (int)(blockIdx.x * pr.chunk_rows); row1 = (int)min(pr.rows, (int64_t)row0 + pr.chunk_rows); }
  const int nsub = (row1 - row0 + C::MT - 1) / C::MT;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1); }
    tc::mbar_init(acc_full, 1);
    tc::mbar_fence_init();
    tc::tma_prefetch_desc(&xmap);
    tc::tma_prefetch_desc(&zmap);
  }
  if (BVEC) {  // the dpre operand's columns 1..15 stay zero for the whole kernel
    for (int i = threadIdx.x; i < C::STAGES * C::B2_BYTES / 16; i += blockDim.x) {
      const int s = i / (C::B2_BYTES / 16), o = i % (C::B2_BYTES / 16);
      reinterpret_cast<uint4*>(sB2(s))[o] = make_uint4(0, 0, 0, 0);
    }
    tc::fence_proxy_async_smem();
  }
  if (warp == 1) {
    __syncwarp();
    tc::tmem_alloc<C::NCOLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      const uint32_t use = (uint32_t)(it / C::STAGES);
      if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
      const int p0 = row0 + it * C::MT;
      int idx[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int p = min(p0 + 4 * lane + j, row1 - 1);
        idx[j] = pr.gather ? __ldg(pr.gather + p) : (int)(pr.gofs + p);
      }
      if (BVEC) {  // dpre -> column 0 of core matrix (group e/8, row e%8): byte (e/8)*256 + (e%8)*16
        uint8_t* b2 = sB2(st);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int e = 4 * lane + j, p = p0 + e;
          const float v = p < row1 ? __ldg(pr.dpre + p) : 0.f;
          *reinterpret_cast<__nv_bfloat16*>(b2 + (e >> 3) * 256 + (e & 7) * 16) = __float2bfloat16_rn(v);
        }
        tc::fence_proxy_async_smem();
      }
      __syncwarp();
      if (lane == 0) {
        tc::mbar_expect_tx(&full[st], C::A_BYTES + C::B_BYTES);
#pragma unroll
        for (int nb = 0; nb < C::NBLK; ++nb)
          tc::tma_load_2d(sB(st) + nb * C::MT * C::RBB, &zmap, &full[st], nb * (C::RBB / 2), p0);
      }
      __syncwarp();
      uint8_t* a = sA(st);
#pragma unroll
      for (int kb = 0; kb < K / 64; ++kb)
        tc::tma_gather4(a + kb * C::MT * 128 + lane * 4 * 128, &xmap, &full[st], kb * 64, idx[0], idx[1], idx[2],
                        idx[3]);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    for (int it = 0; it < nsub; ++it) {
      const int st = it % C::STAGES;
      tc::mbar_wait(&full[st], (uint32_t)(it / C::STAGES) & 1);
      const int nvalid = min(C::MT, row1 - (row0 + it * C::MT));
      if (nvalid < C::MT) {  // rows past the chunk end belong to the next chunk: zero their dZ lines
        uint8_t* b = sB(st);
        for (int i = lane; i < (C::MT - nvalid) * C::NBLK * (C::RBB / 16); i += 32) {
          const int per = C::RBB / 16;
          const int rr = nvalid + i / (C::NBLK * per), rem = i % (C::NBLK * per);
          const int nb = rem / per, c16 = rem % per;
          reinterpret_cast<uint4*>(b + nb * C::MT * C::RBB + rr * C::RBB)[c16] = make_uint4(0, 0, 0, 0);
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
      }
      tc::tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = tc::smem_u32(sA(st)), b0 = tc::smem_u32(sB(st)), c0 = tc::smem_u32(sB2(st));
#pragma unroll
        for (int ks = 0; ks < C::MT / 16; ++ks) {
          const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
          // A: MN-major SW128, feature blocks of 64 at LBO = MT*128, 8-edge groups at SBO = 1024
          const uint64_t ad = tc::umma_desc(a0 + ks * 16 * 128, C::MT * 128, 1024, 2u);
          const uint64_t bd = tc::umma_desc(b0 + ks * 16 * C::RBB, C::MT * C::RBB, 8 * C::RBB, C::BLAYOUT);
          tc::umma_bf16(tmem, ad, bd, C::IDESC, acc);
          if (BVEC) {
            // no-swizzle MN-major: 8-column blocks at SBO = 128 B, 8-edge groups at LBO = 256 B
            const uint64_t cd = tc::umma_desc(c0 + ks * 512, 256, 128, 0u);
            tc::umma_bf16(tmem + N, ad, cd, C::IDESC_B, acc);
          }
        }
        tc::umma_commit(&empty[st]);
        if (it == nsub - 1) tc::umma_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    tc::mbar_wait(acc_full, 0);
    tc::tc_fence_after();
    // M=128: row = lane quarter q * 32 + lane; M=64: rows 16q..16q+15 live in lanes 0..15 of quarter q
    const int row = K == 128 ? q * 32 + lane : q * 16 + lane;
    const bool rvalid = K == 128 || lane < 16;
    float* out = pr.part + (size_t)blockIdx.x * (K * N + K);
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 16) {
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
    if (BVEC) {
      uint32_t v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + N, v);
      tc::tmem_ld_wait();
      if (rvalid) out[K * N + row] = __uint_as_float(v[0]);
    } else if (rvalid) {
      out[K * N + row] = 0.f;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::NCOLS>(tmem);
  }
}

template <int K, int N>
static rgnn_status gemm_dw_tc(const GemmDwArgs& a, cudaStream_t s) {
  tc::watchdog_init();
  using C = DwCfg<K, N>;
  if (a.num_chunks == 0) return RGNN_OK;
  if (!a.Bz) return RGNN_E_UNSUPPORTED;  // B must be a materialised bf16 dZ
  CUtensorMap xmap, zmap;
  RGNN_TRY(make_tmap_2d_bf16(&xmap, a.X, K, (uint64_t)a.x_rows, K * 2, 64, 1, 128));
  RGNN_TRY(make_tmap_2d_bf16(&zmap, a.Bz, N, (uint64_t)std::max<int64_t>(a.rows, 1), N * 2, C::RBB / 2, C::MT,
                             C::RBB));
  TcDwParams pr{a.chunks, a.rows, a.chunk_rows, a.gofs, a.gather, a.dpre, a.part};
  if (a.dpre) {
    auto kern = k_gemm_dw_tc<K, N, true>;
    RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    RGNN_LAUNCH(kern, (unsigned)a.num_chunks, 192, C::SMEM, s, xmap, zmap, pr);
  } else {
    auto kern = k_gemm_dw_tc<K, N, false>;
    RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    RGNN_LAUNCH(kern, (unsigned)a.num_chunks, 192, C::SMEM, s, xmap, zmap, pr);
  }
  return RGNN_OK;
}

bool tc_disabled();

rgnn_status launch_gemm_dw_tc(int K, int N, const GemmDwArgs& a, cudaStream_t s) {
  if (tc_disabled()) return RGNN_E_UNSUPPORTED;
  if (K == 64 && N == 32) return gemm_dw_tc<64, 32>(a, s);
  if (K == 64 && N == 64) return gemm_dw_tc<64, 64>(a, s);
  if (K == 64 && N == 128) return gemm_dw_tc<64, 128>(a, s);
  if (K == 128 && N == 32) return gemm_dw_tc<128, 32>(a, s);
  if (K == 128 && N == 64) return gemm_dw_tc<128, 64>(a, s);
  if (K == 128 && N == 128) return gemm_dw_tc<128, 128>(a, s);
  return RGNN_E_UNSUPPORTED;  // d_in = 32: UMMA M=32 does not exist for cta_group::1
}

// RGCN: dZ[p] = bf16(inv_c[p] * G[dst_s[p]]) in position order (the B operand of the dW GEMM).
__global__ void k_expand_dz(int64_t E, int N, const int32_t* __restrict__ dst_s, const float* __restrict__ inv_c,
                            const float* __restrict__ G, __nv_bfloat16* __restrict__ dZ) {
  const int nch = N / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E * nch; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / nch;
    const int ch = (int)(i - p * nch);
    const float sc = inv_c ? inv_c[p] : 1.f;
    const float4* g = reinterpret_cast<const float4*>(G + (size_t)(dst_s ? dst_s[p] : p) * N + ch * 8);
    const float4 a = __ldg(g), b = __ldg(g + 1);
    uint4 o;
    o.x = tc::pack_bf16(a.x * sc, a.y * sc); o.y = tc::pack_bf16(a.z * sc, a.w * sc);
    o.z = tc::pack_bf16(b.x * sc, b.y * sc); o.w = tc::pack_bf16(b.z * sc, b.w * sc);
    reinterpret_cast<uint4*>(dZ)[i] = o;
  }
}

rgnn_status launch_expand_dz(int64_t E, int N, const int32_t* dst_s, const float* inv_c, const float* G, void* dZ,
                             cudaStream_t s) {
  if (E == 0) return RGNN_OK;
  const int64_t n = E * (N / 8);
  RGNN_LAUNCH(k_expand_dz, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64), 256, 0, s, E, N, dst_s, inv_c, G,
              static_cast<__nv_bfloat16*>(dZ));
  return RGNN_OK;
}

}  // namespace rgnn
